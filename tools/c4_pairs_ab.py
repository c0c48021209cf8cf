"""A/B of the K-split pairs on C4 cells at N=1000 (step-0 solve, best of 5):
python tools/c4_pairs_ab.py d:T [d:T ...]"""
import os
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

import paper_2103_14990_b200 as pb  # noqa: E402

for arg in sys.argv[1:]:
    d, T = (int(v) for v in arg.split(':'))
    system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=1000, d=d, horizon=T, t_sim=1, seed=1))
    out = {}
    for tag in ("1", "0", "1", "0"):
        os.environ["DLMPC_NO_PAIRS"] = tag
        sess = pb.DlmpcSession(system, spec, mask, "b200")
        ms = min(sess.simulate(x0, 1)[1] for _ in range(5))
        traj, _ = sess.simulate(x0, 1)
        it = sum(traj.step_iterations)
        prev = out.get(tag)
        out[tag] = (min(ms, prev[0]) if prev else ms, it, traj.states.copy())
        sess.close()
    a, b = out["1"], out["0"]
    rel = float(np.max(np.abs(a[2] - b[2])) / max(1.0, np.max(np.abs(a[2]))))
    print(f"N=1000 d={d} T={T} iters {a[1]}/{b[1]}  no pairs {1e3 * a[0] / a[1]:.2f} us/iter  "
          f"pairs {1e3 * b[0] / b[1]:.2f} us/iter  states rel diff {rel:.1e}", flush=True)
