"""Grid networks (generic graph path, two-phase kernel): step-0 solve timing.
usage: python tools/grid_time.py side [side ...]"""
import json, sys, time
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import numpy as np
import paper_2103_14990_b200 as pb
from conftest import grid_network
for side in [int(a) for a in sys.argv[1:]]:
    t0 = time.perf_counter()
    system = grid_network(side, side)
    spec = pb.make_benchmark_spec(system, 10)
    mask = pb.build_locality_mask(system, 3, 10)
    x0 = pb.sample_initial_state(system.partition, np.random.default_rng(1))
    sess = pb.DlmpcSession(system, spec, mask, "b200")
    setup = time.perf_counter() - t0
    traj, _ = sess.simulate(x0, 1)
    best = min(sess.simulate(x0, 1)[1] for _ in range(2))
    it = int(sum(traj.step_iterations))
    L = sess.layout
    print(json.dumps({"grid": f"{side}x{side}", "n": side * side, "iterations": it, "ms_per_mpc_step": round(best, 3),
                      "us_per_iteration": round(1e3 * best / it, 2), "kernel": sess.device.info()["mode"],
                      "classes": int(L.n_classes), "s_max": int(L.class_s.max()), "n0_max": int(L.class_n0.max()),
                      "setup_s": round(setup, 1)}), flush=True)
    sess.close()
