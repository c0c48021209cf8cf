"""Per-phase breakdown of the stream kernel (profiling build).
usage: DLMPC_LIB=paper_2103_14990_b200/libdlmpc_timing.so python tools/phase_profile_stream.py N"""
import os, sys
sys.path.insert(0, '.')
import numpy as np
import paper_2103_14990_b200 as pb
n = int(sys.argv[1])
system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=n, d=3, horizon=10, t_sim=1, seed=1))
sess = pb.DlmpcSession(system, spec, mask, "b200")
sess.simulate(x0, 1)
sess.device.phase_times(reset=True)
traj, ms = sess.simulate(x0, 1)
it = sum(traj.step_iterations)
pt = sess.device.phase_times(reset=True).astype(np.float64) / it / (1e3 * float(os.environ.get("DLMPC_CLK_GHZ", "1.965")))   # SM cycles -> us
names = ["phi loop", "chunks", "tables", "setup+stage", "first K", "publish", "barrier", "flush"]
print(f"N={n} {sess.device.info()} iters {it} device {ms:.3f} ms = {1e3*ms/it:.2f} us/iter")
for k, nm in enumerate(names):
    col = pt[:, k]
    print(f"  {nm:12s} max {col.max():8.2f} us  mean {col.mean():8.2f} us")
for k, nm in zip([12, 9, 10, 13, 14, 15], ["  gemm1", "  gemm2 k", "  wait λ", "  epilogue", "  wait prod", "  row pass"]):
    col = pt[:, k]
    print(f"  {nm:12s} max {col.max():8.2f} us  mean {col.mean():8.2f} us")
tot = pt[:, [0, 1, 2, 3, 4, 5, 7, 9, 10, 12, 13, 14, 15]].sum(axis=1)   # everything but the barrier wait
order = np.argsort(-tot)
print("  slowest CTAs (work us/iter):", ", ".join(f"{c}:{tot[c]:.1f}" for c in order[:6]))
print("  fastest CTAs (work us/iter):", ", ".join(f"{c}:{tot[c]:.1f}" for c in order[-4:]))
print(f"  median work {np.median(tot):.1f} us/iter")
