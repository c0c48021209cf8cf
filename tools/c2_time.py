"""Best-of-10 device time of a closed loop (default C2: N=100, 20 steps) in a
fresh process: python tools/c2_time.py [N] [t_sim]"""
import sys
sys.path.insert(0, '.')
import paper_2103_14990_b200 as pb
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
t_sim = int(sys.argv[2]) if len(sys.argv) > 2 else 20
system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=n, d=3, horizon=10, t_sim=t_sim, seed=1))
sess = pb.DlmpcSession(system, spec, mask, "b200")
ms = min(sess.simulate(x0, t_sim)[1] for _ in range(10))
traj, _ = sess.simulate(x0, t_sim)
it = sum(traj.step_iterations)
i = sess.device.info()
print(f"N={n} t_sim={t_sim} iters={it} smem={i['smem_bytes']} {1e3 * ms / it:.2f} us/iter {n * it / ms * 1e-3:.4g} M/s")
