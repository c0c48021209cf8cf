"""Parity on every configuration the benchmark times.

The bench's numbers are only meaningful if the device solves the reference's
problem on exactly those inputs, so every timed config is pinned here:

* C2  chain N=100, d=3, T=10, 20-step closed loop, for EVERY seed bench.py
      cycles through (1..20): reference fixtures (make_golden.py --c2-seeds).
* C3  the N sweep where the stream kernel takes over (N=3000: reference
      fixture; N=10^4: oracle fixture, make_oracle_golden.py --c3).
* C4  all 24 (d, T) cells at N=1000, step 0, including d=1, where the
      reference does not converge in max_iters (oracle fixtures; the oracle is
      pinned bit for bit to the reference in test_oracle_golden.py).
* C5  1 vs 8 graph-partitioned ranks at N=10^5 (bitwise in exact mode).

`b200-exact` must reproduce the fixtures bit for bit; `b200` (the timed
path) must take the same iteration counts with states within FAST_RTOL
(north_star: 1e-6 relative in FP64; measured ~1e-14).
"""

import os

import numpy as np
import pytest

import paper_2103_14990_b200 as pb
from conftest import GOLDEN, golden

pytestmark = pytest.mark.gpu

EXACT, FAST = "b200-exact", "b200"
FAST_RTOL = 1e-9


def rel_err(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)))) / max(1.0, float(np.max(np.abs(b))))


def have(name):
    return os.path.exists(os.path.join(GOLDEN, name + ".npz"))


def chain(n, d, t, **kw):
    system = pb.build_chain_network(n)
    spec = pb.make_benchmark_spec(system, t, **kw)
    mask = pb.build_locality_mask(system, d, t)
    return system, spec, mask


# --------------------------------------------------------------------------- C2
@pytest.mark.skipif(not have("c2_loops_seeds1_20"), reason="fixture not generated")
@pytest.mark.parametrize("variant", [EXACT, FAST])
def test_c2_every_bench_seed_against_reference(variant):
    """bench.py times seeds 1..max(8, steps) (20 by default): each one's
    per-step iteration list and trajectory against the reference's own
    `run_scenario` (fused schedule, bit-identical to sequential)."""
    g = golden("c2_loops_seeds1_20")
    system, spec, mask = chain(100, 3, 10)
    sess = pb.DlmpcSession(system, spec, mask, variant)
    for seed in range(1, 21):
        traj, _ = sess.simulate(g[f"s{seed}_x0"], 20)
        assert list(traj.step_iterations) == list(g[f"s{seed}_iters"]), seed
        if variant == EXACT:
            assert np.array_equal(traj.states, g[f"s{seed}_states"]), seed
            assert np.array_equal(traj.inputs, g[f"s{seed}_inputs"]), seed
            assert pb.closed_loop_cost(traj) == float(g[f"s{seed}_cost"])
        else:
            assert rel_err(traj.states, g[f"s{seed}_states"]) <= FAST_RTOL, seed
            assert rel_err(traj.inputs, g[f"s{seed}_inputs"]) <= FAST_RTOL, seed
    sess.close()


@pytest.mark.skipif(not have("c2_loops_seeds1_20"), reason="fixture not generated")
def test_c2_bench_device_entry_against_reference():
    """The exact entry point bench.py times (dlmpc_simulate_device: x0 and all
    outputs in device memory, one launch per closed loop) on every seed."""
    import torch
    from bench import N_SUB, T_SIM
    g = golden("c2_loops_seeds1_20")
    system, spec, mask = chain(N_SUB, 3, 10)
    sess = pb.DlmpcSession(system, spec, mask, FAST)
    nx, nu = system.n_states, system.n_inputs
    states = torch.zeros((T_SIM + 1) * nx, dtype=torch.float64, device="cuda:0")
    inputs = torch.zeros(T_SIM * nu, dtype=torch.float64, device="cuda:0")
    iters = torch.zeros(T_SIM, dtype=torch.int32, device="cuda:0")
    status = torch.zeros(8, dtype=torch.int32, device="cuda:0")
    for seed in range(1, 21):
        x0 = torch.tensor(g[f"s{seed}_x0"], dtype=torch.float64, device="cuda:0")
        sess.device.simulate_device(x0.data_ptr(), T_SIM, spec.max_iters, spec.eps_pri, spec.eps_dual,
                                    states.data_ptr(), inputs.data_ptr(), iters.data_ptr(), status.data_ptr())
        sess.device.synchronize()
        assert int(status[0]) == 0
        assert iters.cpu().tolist() == list(g[f"s{seed}_iters"]), seed
        assert rel_err(states.cpu().numpy().reshape(T_SIM + 1, nx), g[f"s{seed}_states"]) <= FAST_RTOL
    sess.close()


# --------------------------------------------------------------------------- C3
C3 = [(3000, "c3_n3000_step0", "reference"), (10000, "c3_n10000_step0_oracle", "oracle")]


@pytest.mark.parametrize("n,name,source", C3)
@pytest.mark.parametrize("variant", [EXACT, FAST])
def test_c3_stream_sizes_against_fixture(n, name, source, variant):
    """The sweep points where the default plan is the stream kernel (the
    timed kernel from N ~ 2,400 at d=3): step-0 iteration count and x1 / u0."""
    if not have(name):
        pytest.skip("fixture not generated")
    g = golden(name)
    system, spec, mask = chain(n, 3, 10)
    sess = pb.DlmpcSession(system, spec, mask, variant)
    if variant == FAST:
        assert sess.device.info()["mode"] == "stream"
    traj, _ = sess.simulate(g["x0"], 1)
    if source == "reference":
        ref_iters, ref_x1, ref_u0 = list(g["step_iters"]), g["states"][1], g["inputs"][0]
    else:
        ref_iters, ref_x1, ref_u0 = [int(g["iterations"])], g["x1"], g["u0"]
    assert list(traj.step_iterations) == ref_iters
    if variant == EXACT:
        assert np.array_equal(traj.states[1], ref_x1)
        assert np.array_equal(traj.inputs[0], ref_u0)
    else:
        assert rel_err(traj.states[1], ref_x1) <= FAST_RTOL
        assert rel_err(traj.inputs[0], ref_u0) <= FAST_RTOL
    sess.close()


# --------------------------------------------------------------------------- C4
C4_CELLS = [(d, t) for t in (5, 10, 20, 30) for d in (1, 2, 3, 4, 5, 6)]


def c4_fixture():
    if not have("c4_n1000_step0_oracle"):
        pytest.skip("fixture not generated")
    return golden("c4_n1000_step0_oracle")


@pytest.mark.parametrize("variant", [EXACT, FAST])
@pytest.mark.parametrize("d,t", C4_CELLS)
def test_c4_cell_against_oracle(d, t, variant):
    """Every cell of the locality/horizon sweep at its timed size N=1000.
    d=1: the reference (oracle) hits max_iters=5000 -- the device must raise
    NotConverged after exactly as many iterations, with the same final
    residual pair (bitwise in exact mode)."""
    g = c4_fixture()
    key = f"d{d}t{t}_"
    if key + "converged" not in g:
        pytest.skip("cell not generated")
    system, spec, mask = chain(1000, d, t)
    sess = pb.DlmpcSession(system, spec, mask, variant)
    x0 = g[key + "x0"]
    if bool(g[key + "converged"]):
        traj, _ = sess.simulate(x0, 1)
        assert traj.step_iterations == [int(g[key + "iterations"])]
        if variant == EXACT:
            assert np.array_equal(traj.states[1], g[key + "x1"])
            assert np.array_equal(traj.inputs[0], g[key + "u0"])
        else:
            assert rel_err(traj.states[1], g[key + "x1"]) <= FAST_RTOL
            assert rel_err(traj.inputs[0], g[key + "u0"]) <= FAST_RTOL
    else:
        with pytest.raises(pb.NotConverged) as exc:
            sess.simulate(x0, 1)
        hist = np.array(exc.value.residual_history)
        assert len(hist) == int(g[key + "history_len"]) == spec.max_iters
        tail = g[key + "history_tail"]
        if variant == EXACT:
            assert np.array_equal(hist[-len(tail):], tail)
            assert np.array_equal(hist[:16], g[key + "history_head"])
        else:
            np.testing.assert_allclose(hist[-len(tail):], tail, rtol=1e-6)
            np.testing.assert_allclose(hist[:16], g[key + "history_head"], rtol=1e-9, atol=1e-15)
    sess.close()


@pytest.mark.parametrize("d,t", [(5, 10), (3, 30), (6, 20), (2, 30)])
def test_gemm1_mrow_schedule_is_bitwise(d, t, monkeypatch):
    """GEMM 1 by whole m-rows (the default for 16-column patch tiles) against
    one (m, n) tile per warp (DLMPC_G1_MROW=0): the same two accumulation
    chains per tile, so Y and every iterate are bit-identical. The cells are
    chosen so the branch fires fully (d=5,T=10: 12 m-tiles < 16 warps) and
    partially (d=3,T=30; d=6,T=20: mr = mt1/NW*NW, rest single tiles)."""
    system, spec, mask = chain(1000, d, t)
    x0 = pb.sample_initial_state(system.partition, np.random.default_rng(1))
    a = pb.DlmpcSession(system, spec, mask, FAST)
    assert a.device.info()["tile_cols"] == 16
    monkeypatch.setenv("DLMPC_G1_MROW", "0")
    b = pb.DlmpcSession(system, spec, mask, FAST)
    monkeypatch.delenv("DLMPC_G1_MROW")
    ta, _ = a.simulate(x0, 1)
    tb, _ = b.simulate(x0, 1)
    assert ta.step_iterations == tb.step_iterations
    assert np.array_equal(ta.states, tb.states) and np.array_equal(ta.inputs, tb.inputs)
    a.close(); b.close()


# --------------------------------------------------------------------------- C5
@pytest.mark.slow
@pytest.mark.parametrize("variant", [EXACT, FAST])
def test_c5_one_vs_eight_ranks_at_1e5(variant):
    """The C5 determinism claim at N=10^5: the graph-partitioned solve over 8
    ranks (in-process lockstep on one GPU, halo messages packed / unpacked by
    device kernels) against the single-domain solve. Exact mode: bitwise;
    fast mode: the same iterations, states within 1e-12 (the stream kernel's
    Φ-dot partial slots follow the unit cut, which the partition moves)."""
    from paper_2103_14990_b200.partition import simulate_partitioned_inprocess
    system, spec, mask = chain(100000, 3, 10)
    x0 = pb.sample_initial_state(system.partition, np.random.default_rng(1))
    sess = pb.DlmpcSession(system, spec, mask, variant)
    one, _ = sess.simulate(x0, 1)
    sess.close()
    states, inputs, iters = simulate_partitioned_inprocess(system, spec, mask, x0, 1, 8, variant)
    assert iters == list(one.step_iterations)
    if variant == EXACT:
        assert np.array_equal(states, one.states) and np.array_equal(inputs, one.inputs)
    else:
        assert rel_err(states, one.states) <= 1e-12


# ------------------------------------------------------------------ divergence
@pytest.mark.parametrize("variant", [EXACT, FAST])
@pytest.mark.parametrize("n,force_stream", [(10, False), (100, False), (2500, True)])
def test_nan_state_is_not_converged(n, force_stream, variant, monkeypatch):
    """A NaN in the measured state makes every residual NaN; np.max
    propagates it, `NaN <= eps` is false and the reference raises
    NotConverged at max_iters with a NaN history (strategies.py:178-183,
    admm.py:339-343). The device maxima must not drop the NaN."""
    if force_stream:
        monkeypatch.setenv("DLMPC_FORCE_STREAM", "1")
    system, spec, mask = chain(n, 3 if n > 10 else 2, 10 if n > 10 else 5, max_iters=6)
    sess = pb.DlmpcSession(system, spec, mask, variant)
    if force_stream and variant == FAST:
        assert sess.device.info()["mode"] == "stream"
    x0 = pb.sample_initial_state(system.partition, np.random.default_rng(2))
    x0[3] = np.nan
    with pytest.raises(pb.NotConverged) as exc:
        sess.simulate(x0, 2)
    hist = np.array(exc.value.residual_history)
    assert len(hist) == 6 and np.all(np.isnan(hist)) and exc.value.step == 0
    sess.close()
