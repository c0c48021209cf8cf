"""Step-0 solve time at N=1000 for a few (d, T) cells of the C4 sweep, best
of 5, in a fresh process: python tools/c4_quick.py d:T [d:T ...]"""
import sys
sys.path.insert(0, '.')
import paper_2103_14990_b200 as pb
for arg in sys.argv[1:]:
    d, T = (int(v) for v in arg.split(':'))
    system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=1000, d=d, horizon=T, t_sim=1, seed=1))
    sess = pb.DlmpcSession(system, spec, mask, "b200")
    ms = min(sess.simulate(x0, 1)[1] for _ in range(5))
    traj, _ = sess.simulate(x0, 1)
    it = sum(traj.step_iterations)
    print(f"N=1000 d={d} T={T} iters={it} {1e3 * ms / it:.2f} us/iter mode={sess.device.info()['mode']}", flush=True)
    sess.close()
