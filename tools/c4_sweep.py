"""C4: the locality/horizon sweep d = 1..6 x T in {5, 10, 20,
30} at N = 1000, step-0 solve, fast path: device time per iteration, kernel
mode and the class operator size (the longest-vector padding it exercises).
usage: python tools/c4_sweep.py [out.json]"""
import json, sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2103_14990_b200 as pb
rows = []
for t in (5, 10, 20, 30):
    for d in range(1, 7):
        t0 = time.perf_counter()
        try:
            system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=1000, d=d, horizon=t, t_sim=1, seed=1))
            sess = pb.DlmpcSession(system, spec, mask, "b200")
            setup = time.perf_counter() - t0
            traj, _ = sess.simulate(x0, 1)
            best = min(sess.simulate(x0, 1)[1] for _ in range(2))
            it = int(sum(traj.step_iterations))
            L = sess.layout
            info = sess.device.info()
            row = {"d": d, "T": t, "iterations": it, "ms_per_mpc_step": best, "us_per_iteration": 1e3 * best / it,
                   "kernel": info["mode"], "s_max": int(L.class_s.max()), "n0_max": int(L.class_n0.max()),
                   "s_pad": int(L.s_pad), "nnz": int(np.sum(L.col_len)), "setup_s": round(setup, 2)}
            sess.close()
        except Exception as exc:
            row = {"d": d, "T": t, "error": repr(exc)[:200]}
        rows.append(row)
        print(json.dumps(row), flush=True)
if len(sys.argv) > 1:
    json.dump(rows, open(sys.argv[1], "w"), indent=1)
