"""Quick device-vs-oracle check + timings used during development (not a test)."""
import os, sys, time, numpy as np
sys.path.insert(0, '.')
import paper_2103_14990_b200 as pb
from paper_2103_14990_b200 import sls_core as sc
from oracle import admm_ref
sys.path.insert(0, 'tests')
from conftest import golden

for name in ("c1_loop_seed1", "c2_loop_seed1"):
    g = golden(name)
    n, d, T, tsim, seed = (int(v) for v in g["config"])
    system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=n, d=d, horizon=T, t_sim=tsim, seed=seed))
    for variant in ("b200-exact", "b200"):
        traj, rep = pb.dlmpc_simulate(system, spec, mask, x0, tsim, variant)
        traj, rep = pb.dlmpc_simulate(system, spec, mask, x0, tsim, variant)
        rel = np.max(np.abs(traj.states - g['states'])) / np.max(np.abs(g['states']))
        print(f"{name} {variant}: iters equal {list(traj.step_iterations) == list(g['step_iters'])}, "
              f"states bit-equal {np.array_equal(traj.states, g['states'])}, rel {rel:.2e}, device {rep.scenario['device_ms']:.3f} ms "
              f"= {1e3*rep.scenario['device_ms']/sum(traj.step_iterations):.2f} us/iter", flush=True)

def timing(n, t_sim, force2=False):
    os.environ["DLMPC_FORCE_TWOPHASE"] = "1" if force2 else "0"
    system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=n, d=3, horizon=10, t_sim=t_sim, seed=1))
    sess = pb.DlmpcSession(system, spec, mask, "b200")
    for k in range(2):
        traj, ms = sess.simulate(x0, t_sim)
    it = sum(traj.step_iterations)
    print(f"N={n} {'twophase' if force2 else 'patch'} {sess.device.info()} iters {it} device {ms:.3f} ms = {1e3*ms/it:.2f} us/iter", flush=True)
    sess.close()
    return traj
for n, ts in ((100, 20), (1000, 1), (10000, 1)):
    a = timing(n, ts)
    b = timing(n, ts, True)
    print("   patch vs twophase iters equal", a.step_iterations == b.step_iterations, "max state diff", np.max(np.abs(a.states - b.states)), flush=True)
