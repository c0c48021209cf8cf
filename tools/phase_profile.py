"""Per-phase device time breakdown (profiling build of the library).
usage: DLMPC_LIB=paper_2103_14990_b200/libdlmpc_timing.so python tools/phase_profile.py N [t_sim] [twophase]
(locality and horizon from DLMPC_PP_D / DLMPC_PP_T, default d=3, T=10)"""
import os, sys
sys.path.insert(0, '.')
import numpy as np
import paper_2103_14990_b200 as pb
n = int(sys.argv[1]); t_sim = int(sys.argv[2]) if len(sys.argv) > 2 else 1
if len(sys.argv) > 3 and sys.argv[3] == "twophase":
    os.environ["DLMPC_FORCE_TWOPHASE"] = "1"
system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=n, d=int(os.environ.get("DLMPC_PP_D", 3)),
                                                      horizon=int(os.environ.get("DLMPC_PP_T", 10)), t_sim=t_sim, seed=1))
sess = pb.DlmpcSession(system, spec, mask, "b200")
sess.simulate(x0, t_sim)
sess.device.phase_times(reset=True)
traj, ms = sess.simulate(x0, t_sim)
it = sum(traj.step_iterations)
CLK_GHZ = float(os.environ.get('DLMPC_CLK_GHZ', '1.965'))   # timers count SM cycles
raw = sess.device.phase_times(reset=True).astype(np.float64) / (1e3 * CLK_GHZ)
pt = raw / it   # us per iteration per CTA
st = raw[:, 8:12] / t_sim   # us per MPC step per CTA
names = ["phi", "prologue", "gemm1", "gemm2", "epilogue", "publish", "barrier", "wait"]
print(f"N={n} {sess.device.info()} iters {it} device {ms:.3f} ms = {1e3*ms/it:.2f} us/iter")
for k, nm in enumerate(names):
    col = pt[:, k]
    print(f"  {nm:9s} max {col.max():7.2f} us  mean {col.mean():7.2f} us  min {col.min():7.2f}")
print(f"  sum(max) {pt[:, :7].max(axis=0).sum():.2f}  per-CTA total max {pt[:, :7].sum(axis=1).max():.2f}")
tot = pt[:, :8].sum(axis=1)
for b in [int(np.argmax(tot)), int(np.argsort(tot)[len(tot) // 2])]:
    print(f"  CTA {b}: " + " ".join(f"{nm}={pt[b, k]:.2f}" for k, nm in enumerate(names)) + f" total={tot[b]:.2f}")
snames = ["rowdata+bar", "phimeta", "control+plant", "bar"]
print("  per MPC step (us): " + " ".join(f"{nm}={st[:, k].max():.2f}" for k, nm in enumerate(snames))
      + f" total={st.sum(axis=1).max():.2f}  (device {1e3 * ms / t_sim:.2f} per step)")
if os.environ.get("DLMPC_PP_CTAS"):   # per-CTA compute (phases before the publish), slowest first
    comp = pt[:, :5].sum(axis=1)
    order = np.argsort(-comp)
    print("  compute per CTA (us): " + " ".join(f"{b}:{comp[b]:.1f}" for b in order[:12]) + " ... "
          + " ".join(f"{b}:{comp[b]:.1f}" for b in order[-6:]))
    print("  compute quantiles (us): " + " ".join(f"{q}:{np.quantile(comp, q):.1f}" for q in (0, .1, .5, .9, 1)))
    for b in order[:3]:
        print(f"  slow CTA {b}: " + " ".join(f"{nm}={pt[b, k]:.2f}" for k, nm in enumerate(names[:5])))
