"""Multi-rank paths on CPU with gloo (world size 2).

1. The graph-partitioned ADMM iteration: each rank runs the
   kernel's data flow (layout emulator, exact arithmetic) on its own columns
   and the Φ patch of its rows, exchanges its boundary columns' ψ,λ with the
   neighbour every iteration (dist.send/recv) and all-reduces the residual
   maxima. The partitioned iterates must be bit-identical to the
   single-domain iteration.
2. The bench's replica reduction (sum of iterations, max of times).
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2103_14990_b200 as pb
from paper_2103_14990_b200.devlayout import DeviceLayout
from paper_2103_14990_b200.partition import halo_bytes_per_iteration, plan_partition


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def build(n=12, d=2, t=4):
    system = pb.build_chain_network(n)
    spec = pb.make_benchmark_spec(system, t)
    mask = pb.build_locality_mask(system, d, t)
    op = pb.build_dynamics_operator(system, t)
    classes = pb.build_column_classes(op, mask)
    layout = DeviceLayout(system, spec, mask, classes, exact=True)
    x0 = pb.sample_initial_state(system.partition, np.random.default_rng(7))
    return system, spec, mask, layout, x0


def col_slices(L, subs):
    out = []
    for j in subs:
        c0, cn = int(L.state_start[j]), int(L.state_count[j])
        out.append(slice(c0 * L.s_pad, (c0 + cn) * L.s_pad))
    return out


def partitioned_worker(rank, world, port, iters, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from layout_emulator import LayoutEmulator
    import torch
    system, spec, mask, L, x0 = build()
    plan = plan_partition(mask, world)[rank]
    em = LayoutEmulator(L)
    em.set_x(x0)
    own = list(range(*plan.own))
    own_cols = set(c for j in own for c in range(L.state_start[j], L.state_start[j] + L.state_count[j]))
    hist = []
    for _ in range(iters):
        full_psi, full_lam = em.psi.copy(), em.lam.copy()
        pri, dual = em.iterate()       # computes everything; only own columns are trusted
        # discard non-own columns: keep previous values there until the halo arrives
        mask_own = np.zeros(L.n_cols, dtype=bool)
        mask_own[list(own_cols)] = True
        cell_own = np.repeat(mask_own, L.s_pad)
        em.psi = np.where(cell_own, em.psi, full_psi)
        em.lam = np.where(cell_own, em.lam, full_lam)
        # residual maxima over own columns only, then all-reduce(max)
        own_idx = np.flatnonzero(cell_own)
        loc = torch.tensor([float(np.max(np.abs(em.phi[own_idx] - em.psi[own_idx]))),
                            float(np.max(np.abs(em.psi[own_idx] - em.psi_prev[own_idx])))], dtype=torch.float64)
        dist.all_reduce(loc, op=dist.ReduceOp.MAX)
        hist.append((float(loc[0]), L.rho * float(loc[1])))
        # halo exchange: send own boundary columns, receive the neighbour's
        reqs = []
        for q, subs in plan.send.items():
            buf = torch.from_numpy(np.concatenate([np.concatenate([em.psi[s], em.lam[s]]) for s in col_slices(L, subs)]))
            reqs.append(dist.isend(buf, q))
        for q, subs in plan.recv.items():
            sl = col_slices(L, subs)
            size = sum(2 * (s.stop - s.start) for s in sl)
            buf = torch.zeros(size, dtype=torch.float64)
            dist.recv(buf, q)
            off = 0
            for s in sl:
                w = s.stop - s.start
                em.psi[s] = buf[off:off + w].numpy(); off += w
                em.lam[s] = buf[off:off + w].numpy(); off += w
        for r_ in reqs:
            r_.wait()
    out_q.put((rank, hist, {c: (em.psi[c * L.s_pad:(c + 1) * L.s_pad].copy(),
                                em.lam[c * L.s_pad:(c + 1) * L.s_pad].copy()) for c in own_cols}))
    dist.barrier()
    dist.destroy_process_group()


def test_plan_covers_every_subsystem_once():
    system, spec, mask, L, x0 = build(40, 3, 5)
    for world in (1, 2, 4, 8):
        plans = plan_partition(mask, world)
        owned = np.concatenate([np.arange(*p.own) for p in plans])
        assert np.array_equal(owned, np.arange(40))
        for p in plans:
            for q, subs in p.recv.items():
                assert np.array_equal(plans[q].send[p.rank], subs)
                assert np.all((subs >= plans[q].own[0]) & (subs < plans[q].own[1]))
            # a chain rank only talks to ranks within 2d hops
            assert len(p.recv) <= 2 * 3 * 2
    hb = halo_bytes_per_iteration(plan_partition(mask, 4), mask, L.s_pad)
    assert max(hb) <= 2 * 2 * 3 * 2 * L.s_pad * 2 * 8     # 2d subsystems per side, 2 cols, ψ+λ


def test_partitioned_iteration_matches_single_domain():
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from layout_emulator import LayoutEmulator
    iters, world = 6, 2
    system, spec, mask, L, x0 = build()
    ref = LayoutEmulator(L)
    ref.set_x(x0)
    ref_hist = [ref.iterate() for _ in range(iters)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=partitioned_worker, args=(r, world, port, iters, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, hist, cols in results:
        assert hist == ref_hist, rank
        for c, (psi, lam) in cols.items():
            assert np.array_equal(psi, ref.psi[c * L.s_pad:(c + 1) * L.s_pad])
            assert np.array_equal(lam, ref.lam[c * L.s_pad:(c + 1) * L.s_pad])
    assert sorted(len(c) for _, _, c in results) == [12, 12]


def replica_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    vals = np.array([100.0 * (rank + 1), 3.0 + rank, 50.0, 7.0 - rank])
    out_q.put((rank, bench.reduce_over_ranks(vals, dist)))
    dist.destroy_process_group()


def test_bench_replica_reduction():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=replica_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=30)
    # iterations summed, times maxed over ranks
    for r in (0, 1):
        assert list(res[r]) == [300.0, 4.0, 100.0, 7.0]


def _own_cols(cs, cc, own_local):
    lo, hi = own_local
    return np.arange(int(cs[lo]), int(cs[hi - 1] + cc[hi - 1]))


@pytest.mark.parametrize("n,d,t,world", [(14, 2, 4, 2), (14, 2, 4, 3), (20, 1, 5, 4), (12, 3, 4, 2)])
def test_rank_window_layouts_reproduce_single_domain(n, d, t, world):
    """Each rank's window sub-problem (own + 2d-hop halo, `build_rank_layout`)
    driven on its owned columns only, with halo ψ,λ copied from the owning
    rank after every iteration, reproduces the single-domain iteration bit
    for bit (residual maxima and every owned column)."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from layout_emulator import LayoutEmulator
    from paper_2103_14990_b200.partition import build_rank_layout, halo_cells
    system, spec, mask, L, x0 = build(n, d, t)
    ref = LayoutEmulator(L)
    ref.set_x(x0)
    plans = plan_partition(mask, world)
    ranks = []
    owner_of_col = np.empty(L.n_cols, dtype=np.int64)
    ssid_sub = []
    for p in plans:
        RL, sub_ids, sid, iid, own_local, cs, cc, _, _ = build_rank_layout(system, spec, mask, p, True)
        assert RL.own_sub == own_local
        oc = _own_cols(cs, cc, own_local)
        assert RL.own_cols == (int(oc[0]), int(oc[-1]) + 1)
        owner_of_col[sid[oc]] = len(ranks)
        ssid_sub.append(sub_ids)
        em = LayoutEmulator(RL)
        em.set_x(x0[sid])
        ranks.append((p, RL, em, sid, oc))
    for k in range(8):
        want = ref.iterate()
        pri = dual = 0.0
        for p, RL, em, sid, oc in ranks:
            keep_psi, keep_lam = em.psi.copy(), em.lam.copy()
            em.iterate()
            cell = np.zeros(RL.n_cols, dtype=bool)
            cell[oc] = True
            cell = np.repeat(cell, RL.s_pad)
            em.psi = np.where(cell, em.psi, keep_psi)
            em.lam = np.where(cell, em.lam, keep_lam)
            pri = max(pri, float(np.max(np.abs(em.phi[cell] - em.psi[cell]))))
            dual = max(dual, float(np.max(np.abs(em.psi[cell] - em.psi_prev[cell]))))
        assert (pri, L.rho * dual) == want, k
        # halo refresh: entry-wise messages from every source rank
        for di, (p, RL, em, sid, oc) in enumerate(ranks):
            for si in p.recv:
                _, SL, sem, ssid, _ = ranks[si]
                sc = halo_cells(mask, plans, si, di, SL, np.unique(ssid_sub[si]), "src")
                dc = halo_cells(mask, plans, si, di, RL, np.unique(ssid_sub[di]), "dst")
                assert sc.size == dc.size > 0
                em.psi[dc] = sem.psi[sc]
                em.lam[dc] = sem.lam[sc]
    for p, RL, em, sid, oc in ranks:
        for c in oc:
            g = sid[c]
            w = min(RL.s_pad, L.s_pad)
            assert np.array_equal(em.psi[c * RL.s_pad:c * RL.s_pad + w], ref.psi[g * L.s_pad:g * L.s_pad + w])
            assert np.array_equal(em.lam[c * RL.s_pad:c * RL.s_pad + w], ref.lam[g * L.s_pad:g * L.s_pad + w])


def test_x_halo_lists_cover_every_window():
    """Per MPC step only the 2d-hop halo of the measured state crosses ranks
    (partition.x_halo_lists): what r sends q is exactly what q expects from
    r, and own + received states cover each rank's window."""
    import paper_2103_14990_b200 as pb
    from paper_2103_14990_b200.partition import plan_partition, x_halo_lists
    system = pb.build_chain_network(40)
    mask = pb.build_locality_mask(system, 3, 5)
    st = np.asarray(system.partition.state_ranges).reshape(-1, 2)
    for world in (2, 3, 5):
        plans = plan_partition(mask, world)
        lists = [x_halo_lists(plans, system, r) for r in range(world)]
        for r in range(world):
            send, recv = lists[r]
            for q, ids in send.items():
                assert np.array_equal(ids, lists[q][1][r])
            window = np.concatenate([np.arange(*st[i]) for i in plans[r].need])
            own = np.concatenate([np.arange(*st[i]) for i in range(*plans[r].own)])
            got = np.concatenate([own] + list(recv.values()))
            assert np.array_equal(np.sort(got), np.sort(window))
            assert sum(v.size for v in recv.values()) < system.n_states - own.size or world == 2
