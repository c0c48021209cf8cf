"""One chain case for profiling: setup, 2 warm-up solves, 1 measured solve.
usage: python tools/profile_case.py N [d] [T] [variant] [t_sim]"""
import sys, time
sys.path.insert(0, '.')
import paper_2103_14990_b200 as pb
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 3
t = int(sys.argv[3]) if len(sys.argv) > 3 else 10
variant = sys.argv[4] if len(sys.argv) > 4 else "b200"
t_sim = int(sys.argv[5]) if len(sys.argv) > 5 else 1
system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=n, d=d, horizon=t, t_sim=t_sim, seed=1))
t0 = time.time()
sess = pb.DlmpcSession(system, spec, mask, variant)
print("setup", round(time.time() - t0, 2), "s", sess.device.info(), flush=True)
for k in range(3):
    traj, ms = sess.simulate(x0, t_sim)
    it = sum(traj.step_iterations)
    print(f"iters {it} device {ms:.3f} ms  {1e3 * ms / it:.2f} us/iter", flush=True)
