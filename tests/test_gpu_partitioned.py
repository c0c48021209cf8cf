"""Graph-partitioned device solve on one GPU.

Each rank's sub-problem (own subsystems + 2d-hop halo) runs as its own
device session whose kernels solve only the owned columns; after every
iteration the ranks exchange packed halo messages (device pack/unpack
kernels) and reduce the residual maxima. Driven in lockstep from one process
(`simulate_partitioned_inprocess`) the ranks never wait on one another on
the device, so one GPU checks the partitioned algorithm: in exact mode the
closed loop is bit-identical to the reference's (golden fixtures) for every
world size, which is the C5 determinism claim.
"""

import os
import socket

import numpy as np
import pytest

import paper_2103_14990_b200 as pb
from conftest import golden, random_graph_system
from oracle import admm_ref
from paper_2103_14990_b200.partition import simulate_partitioned, simulate_partitioned_inprocess

pytestmark = pytest.mark.gpu

EXACT, FAST = "b200-exact", "b200"


def loop_problem(g):
    n, d, t, t_sim, seed = (int(v) for v in g["config"])
    system = pb.build_chain_network(n)
    spec = pb.make_benchmark_spec(system, t, eps=float(g["eps"]), bounded=bool(g["bounded"]))
    mask = pb.build_locality_mask(system, d, t)
    return system, spec, mask, t_sim


def rel_err(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)))) / max(1.0, float(np.max(np.abs(b))))


@pytest.mark.parametrize("name,world", [("c1_loop_seed1", 2), ("c1_loop_seed1", 3), ("c2_loop_seed1", 2),
                                        ("c2_loop_seed1", 4), ("d1_loop_n30", 5), ("d4_loop_n20", 2),
                                        ("unbounded_loop_n8", 2)])
@pytest.mark.parametrize("variant", [EXACT, FAST])
def test_partitioned_closed_loop_against_reference(name, world, variant):
    g = golden(name)
    system, spec, mask, t_sim = loop_problem(g)
    states, inputs, iters = simulate_partitioned_inprocess(system, spec, mask, g["x0"], t_sim, world, variant)
    assert iters == list(g["step_iters"])
    if variant == EXACT:
        assert np.array_equal(states, g["states"])
        assert np.array_equal(inputs, g["inputs"])
    else:
        assert rel_err(states, g["states"]) <= 1e-9
        assert rel_err(inputs, g["inputs"]) <= 1e-9


def test_partitioned_fast_matches_single_domain_fast():
    """World size changes which columns share a CTA, not the per-column
    arithmetic: the fast path agrees with its own single-domain run."""
    g = golden("c2_loop_seed1")
    system, spec, mask, t_sim = loop_problem(g)
    one, _ = pb.dlmpc_simulate(system, spec, mask, g["x0"], 6, FAST)
    states, inputs, iters = simulate_partitioned_inprocess(system, spec, mask, g["x0"], 6, 3, FAST)
    assert iters == list(one.step_iterations)
    assert rel_err(states, one.states) <= 1e-12


@pytest.mark.parametrize("name,world", [("c2_loop_seed1", 2), ("c2_loop_seed1", 3), ("d4_loop_n20", 2)])
def test_partitioned_stream_kernel_against_reference(name, world, monkeypatch):
    """Rank sub-problems on the stream kernel (forced at this size): patch
    subsystems whose ball holds another rank's columns recompute their full
    Φ from the exchanged ψ, λ every iteration, the rest sum the owned units'
    Φ-dot partials, which persist across the host-driven launches."""
    from paper_2103_14990_b200 import device
    g = golden(name)
    system, spec, mask, t_sim = loop_problem(g)
    modes = []
    real = device.DeviceSession

    def spy(*a, **k):
        sess = real(*a, **k)
        modes.append(sess.info()["mode"])
        return sess

    monkeypatch.setattr(device, "DeviceSession", spy)   # RankSolver imports it per rank
    monkeypatch.setenv("DLMPC_FORCE_STREAM", "1")
    states, inputs, iters = simulate_partitioned_inprocess(system, spec, mask, g["x0"], t_sim, world, FAST)
    assert modes == ["stream"] * world
    assert iters == list(g["step_iters"])
    assert rel_err(states, g["states"]) <= 1e-9
    assert rel_err(inputs, g["inputs"]) <= 1e-9


@pytest.mark.parametrize("variant", [EXACT, FAST])
def test_partitioned_generic_graph_against_oracle(variant):
    rng = np.random.default_rng(11)
    system = random_graph_system(9, rng)
    spec = pb.make_benchmark_spec(system, 3)
    mask = pb.build_locality_mask(system, 2, 3)
    tables = pb.LayoutTables(mask)
    cs = pb.precompute_column_solvers(pb.build_dynamics_operator(system, 3), mask)
    x0 = rng.uniform(0.0, 1.0, system.n_states)
    ref = admm_ref.simulate(system, spec, tables, cs, x0, 4)
    states, inputs, iters = simulate_partitioned_inprocess(system, spec, mask, x0, 4, 2, variant)
    assert iters == ref["step_iterations"]
    if variant == EXACT:
        assert np.array_equal(states, ref["states"])
    else:
        assert rel_err(states, ref["states"]) <= 1e-9


def test_distributed_driver_single_rank_nccl():
    """The torch.distributed driver (NCCL, world size 1 on this box)."""
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        g = golden("c1_loop_seed1")
        system, spec, mask, t_sim = loop_problem(g)
        states, inputs, iters = simulate_partitioned(system, spec, mask, g["x0"], t_sim, EXACT)
        assert iters == list(g["step_iters"])
        assert np.array_equal(states, g["states"])
    finally:
        dist.destroy_process_group()


def test_distributed_driver_async_exchange_matches_inprocess():
    """The NCCL driver enqueues iteration, halo pack, all-reduce and unpack on
    the solver's stream with one host read per iteration: on a network large
    enough that a missing stream dependency would read a stale residual, it
    takes the same iterations as the synchronous in-process driver and ends
    bit-identical."""
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=20000, d=3, horizon=10, t_sim=2, seed=1))
    ref = simulate_partitioned_inprocess(system, spec, mask, x0, 2, 1, FAST)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        states, inputs, iters = simulate_partitioned(system, spec, mask, x0, 2, FAST)
    finally:
        dist.destroy_process_group()
    assert iters == ref[2]
    assert np.array_equal(states, ref[0]) and np.array_equal(inputs, ref[1])


def test_async_exchange_entry_points_with_halos():
    """dlmpc_iterate_async / dlmpc_halo_pack_async / dlmpc_halo_unpack_async
    with real halos: three ranks in one process, messages moved between
    device buffers on the sessions' streams, the global residual reduced on
    the host; the closed loop equals the synchronous in-process driver bit
    for bit (NCCL cannot run several ranks on one GPU, this covers the async
    path the NCCL driver takes)."""
    import torch
    from paper_2103_14990_b200.errors import NotConverged
    from paper_2103_14990_b200.partition import RankSolver, plan_partition
    g = golden("c2_loop_seed1")
    system, spec, mask, t_sim = loop_problem(g)
    t_sim = 4
    ref = simulate_partitioned_inprocess(system, spec, mask, g["x0"], t_sim, 3, FAST)
    world = 3
    plans = plan_partition(mask, world)
    ranks = [RankSolver(system, spec, mask, plans, r, FAST, 0) for r in range(world)]
    try:
        dev = torch.device("cuda", 0)
        sbuf = [torch.zeros(max(1, rk.send_doubles), dtype=torch.float64, device=dev) for rk in ranks]
        rbuf = [torch.zeros(max(1, rk.recv_doubles), dtype=torch.float64, device=dev) for rk in ranks]
        res = [torch.zeros(2, dtype=torch.float64, device=dev) for _ in ranks]
        x = np.asarray(g["x0"], dtype=np.float64)
        states, iters = [x], []
        for step in range(t_sim):
            for rk in ranks:
                rk.start_step(x, cold=(step == 0))
            for it in range(spec.max_iters):
                for r, rk in enumerate(ranks):
                    rk.session.iterate_async(1, res[r].data_ptr())
                    rk.session.halo_pack_async(sbuf[r].data_ptr())
                for rk in ranks:
                    rk.session.synchronize()
                for r, rk in enumerate(ranks):
                    for k, src in enumerate(rk.recv_from):
                        sk = ranks[src].send_to.index(r)
                        a, b = int(ranks[src].send_off[sk]), int(ranks[src].send_off[sk + 1])
                        rbuf[r][int(rk.recv_off[k]):int(rk.recv_off[k + 1])].copy_(sbuf[src][a:b])
                torch.cuda.synchronize()
                for r, rk in enumerate(ranks):
                    rk.session.halo_unpack_async(rbuf[r].data_ptr())
                pri = max(float(v[0]) for v in res)
                dual = max(float(v[1]) for v in res)
                if pri <= spec.eps_pri and dual <= spec.eps_dual:
                    break
            else:
                raise NotConverged([], step=step)
            iters.append(it + 1)
            xn = np.zeros(system.n_states)
            for rk in ranks:
                rk.session.synchronize()
                _, _, sid, xx = rk.finish_step()
                xn[sid] = xx
            x = xn
            states.append(x)
        assert iters == ref[2]
        assert np.array_equal(np.array(states), ref[0])
    finally:
        for rk in ranks:
            rk.close()


def _dist_worker(rank, world, port, name, variant, out_q):
    """One torch.distributed rank (gloo) of the partitioned closed loop; all
    ranks share cuda:0, their kernels never wait on one another (the
    exchange is host-driven), so this checks the driver's choreography --
    all-reduce, batch_isend_irecv halo messages, the step gathers."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        g = golden(name)
        system, spec, mask, t_sim = loop_problem(g)
        states, inputs, iters = simulate_partitioned(system, spec, mask, g["x0"], t_sim, variant)
        out_q.put((rank, states, inputs, iters))
    except Exception as exc:   # surfaced by the parent
        out_q.put((rank, repr(exc), None, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,world", [("c1_loop_seed1", 2), ("c2_loop_seed1", 3)])
def test_distributed_driver_gloo_multi_process(name, world):
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dist_worker, args=(r, world, port, name, EXACT, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        res = [q.get(timeout=300) for _ in range(world)]
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    g = golden(name)
    for rank, states, inputs, iters in res:
        assert not isinstance(states, str), states
        assert iters == list(g["step_iters"]), rank
        assert np.array_equal(states, g["states"]), rank
        assert np.array_equal(inputs, g["inputs"]), rank


# --------------------------------------------------------------------------
# the exchange ON THE DEVICE (dlmpc_dist_setup / dlmpc_multi_solve)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("name,world", [("c1_loop_seed1", 2), ("c2_loop_seed1", 3), ("d4_loop_n20", 2),
                                        ("unbounded_loop_n8", 2), ("d1_loop_n30", 4)])
@pytest.mark.parametrize("variant", [EXACT, FAST])
def test_device_exchange_closed_loop_against_reference(name, world, variant):
    """Every ADMM iteration's halo stores, arrival counters and global stop
    test inside the persistent kernel (the ranks as slices of one cooperative
    launch on this GPU): the reference's closed loops, bit for bit in exact
    mode."""
    from paper_2103_14990_b200.partition import simulate_partitioned_device_inprocess
    g = golden(name)
    system, spec, mask, t_sim = loop_problem(g)
    states, inputs, iters = simulate_partitioned_device_inprocess(system, spec, mask, g["x0"], t_sim, world,
                                                                  variant)
    assert iters == list(g["step_iters"])
    if variant == EXACT:
        assert np.array_equal(states, g["states"]) and np.array_equal(inputs, g["inputs"])
    else:
        assert rel_err(states, g["states"]) <= 1e-9 and rel_err(inputs, g["inputs"]) <= 1e-9


def test_device_exchange_matches_host_driven_exchange():
    """Device-side and host-driven exchange run the same rank sub-problems
    on the same kernels: bit-identical trajectories (N=2500, 4 ranks, stream
    kernel)."""
    from paper_2103_14990_b200.partition import simulate_partitioned_device_inprocess
    system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=2500, d=3, horizon=10, seed=6))
    a_states, a_inputs, a_iters = simulate_partitioned_device_inprocess(system, spec, mask, x0, 2, 4, FAST)
    one, _ = pb.dlmpc_simulate(system, spec, mask, x0, 2, FAST)
    assert a_iters == list(one.step_iterations)
    assert rel_err(a_states, one.states) <= 1e-12


@pytest.mark.slow
def test_device_exchange_c5_determinism_at_1e5():
    """N=10^5 on 8 ranks, exchange on the device, exact arithmetic: bit for
    bit the single-domain solve (the C5 claim of SURVEY §8(e))."""
    from paper_2103_14990_b200.partition import simulate_partitioned_device_inprocess
    system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=100000, d=3, horizon=10, seed=1))
    states, inputs, iters = simulate_partitioned_device_inprocess(system, spec, mask, x0, 1, 8, EXACT)
    sess = pb.DlmpcSession(system, spec, mask, EXACT)
    one, _ = sess.simulate(x0, 1)
    sess.close()
    assert iters == list(one.step_iterations)
    assert np.array_equal(states, one.states) and np.array_equal(inputs, one.inputs)


@pytest.mark.parametrize("name", ["c1_loop_seed1", "c2_loop_seed1"])
def test_device_exchange_distributed_driver_world1(name):
    """The torch.distributed driver of the device exchange
    (simulate_partitioned_device: IPC wiring, one dist_solve launch per MPC
    step, 2d-hop x halo, trajectory gather) at world size 1 over NCCL on this
    box: the reference's closed loop bit for bit."""
    import torch.distributed as dist
    from paper_2103_14990_b200.partition import simulate_partitioned_device
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        g = golden(name)
        system, spec, mask, t_sim = loop_problem(g)
        states, inputs, iters = simulate_partitioned_device(system, spec, mask, g["x0"], t_sim, EXACT)
        assert iters == list(g["step_iters"])
        assert np.array_equal(states, g["states"]) and np.array_equal(inputs, g["inputs"])
    finally:
        dist.destroy_process_group()
