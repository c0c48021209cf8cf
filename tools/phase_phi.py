"""Thread 0's view of the patch Φ stage (timing build, slots 12-15 and 0; locality and horizon from DLMPC_PP_D / DLMPC_PP_T):
DLMPC_LIB=paper_2103_14990_b200/libdlmpc_timing.so python tools/phase_phi.py [N] [t_sim]"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import paper_2103_14990_b200 as pb
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
t_sim = int(sys.argv[2]) if len(sys.argv) > 2 else 20
system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=n, d=int(os.environ.get("DLMPC_PP_D", 3)),
                                                      horizon=int(os.environ.get("DLMPC_PP_T", 10)), t_sim=t_sim, seed=1))
sess = pb.DlmpcSession(system, spec, mask, "b200")
sess.simulate(x0, t_sim)
sess.device.phase_times(reset=True)
traj, ms = sess.simulate(x0, t_sim)
it = sum(traj.step_iterations)
raw = sess.device.phase_times(reset=True).astype(np.float64) / (1e3 * float(os.environ.get("DLMPC_CLK_GHZ", "1.965")))
pt = raw / it
busy = pt[:, 0] + pt[:, 13] > 0
names = {12: "unit start + stash issue", 13: "Φ rows (warp 0)", 14: "residual words landed", 15: "stash landed", 0: "Φ barrier",
         7: "stop test + s_row", 5: "publish + barrier"}
print(f"N={n} {sess.device.info()['grid']} CTAs, {ms / it * 1e3:.2f} us/iter (timing build)")
for k, nm in names.items():
    col = pt[busy, k]
    print(f"  {nm:26s} mean {col.mean():6.3f} us  max {col.max():6.3f}")
