"""Per-rank device time of the graph-partitioned solve, all ranks on one GPU
(driven in lockstep, as simulate_partitioned_inprocess does): the kernel time
each rank would spend on its own GPU per ADMM iteration, the halo bytes it
sends, and the kernel mode of its sub-problem. No multi-GPU timing: this is
the compute side of the scaling estimate (exchange cost not included).
usage: python tools/partition_time.py N world [world ...]"""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2103_14990_b200 as pb
from paper_2103_14990_b200.partition import RankSolver, plan_partition

n = int(sys.argv[1])
worlds = [int(w) for w in sys.argv[2:]] or [2]
system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=n, d=3, horizon=10, t_sim=1, seed=1))
K = 12
for world in worlds:
    t0 = time.time()
    plans = plan_partition(mask, world)
    ranks = [RankSolver(system, spec, mask, plans, r, "b200", 0) for r in range(world)]
    setup = time.time() - t0
    sbuf = [np.zeros(max(1, rk.send_doubles)) for rk in ranks]
    rbuf = [np.zeros(max(1, rk.recv_doubles)) for rk in ranks]
    for rk in ranks:
        rk.start_step(x0, cold=True)
    per = np.zeros((world, K))
    for it in range(K):
        for r, rk in enumerate(ranks):
            rk.iterate()
            per[r, it] = rk.session.last_timing()[0]
        for r, rk in enumerate(ranks):
            rk.pack(sbuf[r].ctypes.data)
        for r, rk in enumerate(ranks):
            for k, src in enumerate(rk.recv_from):
                sk = ranks[src].send_to.index(r)
                a, b = ranks[src].send_off[sk], ranks[src].send_off[sk + 1]
                rbuf[r][rk.recv_off[k]:rk.recv_off[k + 1]] = sbuf[src][a:b]
            rk.unpack(rbuf[r].ctypes.data)
    steady = per[:, 2:]   # after the first (full Φ) iterations
    modes = [rk.session.info()["mode"] for rk in ranks]
    print(f"N={n} world={world} setup {setup:.1f}s modes {sorted(set(modes))} "
          f"rank-max {1e3 * steady.mean(axis=1).max():.1f} us/iter, rank-mean {1e3 * steady.mean():.1f} us/iter, "
          f"halo send max {8 * max(rk.send_doubles for rk in ranks) / 1e3:.1f} KB/iter", flush=True)
    if True:   # per-rank detail
        for r, rk in enumerate(ranks):
            i = rk.session.info()
            print(f"   rank {r}: own {rk.plan.own} {1e3 * steady[r].mean():.1f} us/iter units {i['units']} "
                  f"smem {i['smem_bytes']} n_sub {i['n_sub']}", flush=True)
    for rk in ranks:
        rk.close()
