import os, sys
sys.path.insert(0, '.')
import numpy as np
import paper_2103_14990_b200 as pb
system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=100, d=3, horizon=10, t_sim=20, seed=1))
sess = pb.DlmpcSession(system, spec, mask, "b200")
sess.simulate(x0, 20)
sess.device.phase_times(reset=True)
traj, ms = sess.simulate(x0, 20)
it = sum(traj.step_iterations)
pt = sess.device.phase_times(reset=True).astype(np.float64) / it / (1e3 * float(os.environ.get("DLMPC_CLK_GHZ", "1.965")))   # SM cycles -> us
L = sess.layout
print("iters", it, "us/iter", 1e3 * ms / it)
order = np.argsort(-pt[:, 0])
for c in order[:12]:
    print(f"cta {c:3d} phi {pt[c,0]:.2f} stoptest {pt[c,7]:.2f} pro {pt[c,1]:.2f} g1 {pt[c,2]:.2f} g2 {pt[c,3]:.2f} epi {pt[c,4]:.2f} pub {pt[c,5]:.2f} bar {pt[c,6]:.2f}")
print("median phi", np.median(pt[:100, 0]))
