"""A/B of a library knob read from the environment at session creation.
usage: python tools/env_ab.py VAR=a,b N:t_sim [N:t_sim ...]
Alternates the two values three times, best of 5 per session; reports
us/iteration, subsystem-iterations/s, and whether the trajectories agree
(bitwise, else the max relative difference) and the iteration counts match."""
import os, sys
sys.path.insert(0, '.')
import numpy as np
import paper_2103_14990_b200 as pb
var, vals = sys.argv[1].split('=')
va, vb = vals.split(',')
for arg in sys.argv[2:]:
    n, t_sim = (int(v) for v in arg.split(':'))
    system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=n, d=3, horizon=10, t_sim=t_sim, seed=1))
    res, best = {}, {}
    for tag in (va, vb, va, vb, va, vb):
        os.environ[var] = tag
        sess = pb.DlmpcSession(system, spec, mask, "b200")
        ms = min(sess.simulate(x0, t_sim)[1] for _ in range(5))
        traj, _ = sess.simulate(x0, t_sim)
        best[tag] = min(best.get(tag, 1e9), ms)
        res.setdefault(tag, (traj.states.copy(), traj.inputs.copy(), list(traj.step_iterations), sess.device.info()["mode"]))
        sess.close()
    it = sum(res[va][2])
    line = f"N={n} t_sim={t_sim} iters={it}"
    for tag in (va, vb):
        line += f" | {var}={tag} ({res[tag][3]}) {1e3*best[tag]/it:.2f} us/iter {n*it/best[tag]*1e-3:.4g} M/s"
    print(line, flush=True)
    same_it = res[va][2] == res[vb][2]
    if all(np.array_equal(a, b) for a, b in zip(res[va][:2], res[vb][:2])):
        print(f"N={n} bitwise equal, iterations equal {same_it}", flush=True)
    else:
        d = max(np.max(np.abs(a - b)) / max(np.max(np.abs(a)), 1e-300) for a, b in zip(res[va][:2], res[vb][:2]))
        print(f"N={n} max rel diff {d:.2e}, iterations equal {same_it}", flush=True)
