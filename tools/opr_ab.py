"""Stream kernel: operator region sized for every class (DLMPC_OPR_ALL=1) vs
for the classes carrying the work (rare classes read from L2)."""
import os, sys
sys.path.insert(0, '.')
import numpy as np
import paper_2103_14990_b200 as pb
for n in [int(a) for a in sys.argv[1:]]:
    system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=n, d=3, horizon=10, t_sim=1, seed=1))
    res = {}
    for tag in ("1", "0", "1", "0"):
        os.environ["DLMPC_OPR_ALL"] = tag
        sess = pb.DlmpcSession(system, spec, mask, "b200")
        best = min(sess.simulate(x0, 1)[1] for _ in range(3))
        traj, _ = sess.simulate(x0, 1)
        it = sum(traj.step_iterations)
        i = sess.device.info()
        res.setdefault(tag, traj.states[-1])
        print(f"N={n} opr_all={tag} {i['mode']} units={i['units']} smem={i['smem_bytes']} {1e3*best/it:.2f} us/iter", flush=True)
        sess.close()
    print(f"N={n} bitwise equal {np.array_equal(res['0'], res['1'])}")
