"""Closed loops at N sizes without fixtures against the CPU oracle
(oracle/admm_ref.py, test infrastructure): per-step iteration lists equal,
states within 1e-9 relative, and the kernel plan that ran.
usage: python tools/loop_oracle.py T_SIM N [N ...]"""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import paper_2103_14990_b200 as pb
from oracle import admm_ref
t_sim = int(sys.argv[1])
for n in [int(a) for a in sys.argv[2:]]:
    t0 = time.time()
    system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=n, d=3, horizon=10, t_sim=t_sim, seed=1))
    tables = pb.LayoutTables(mask)
    cs = pb.precompute_column_solvers(pb.build_dynamics_operator(system, 10), mask)
    ref = admm_ref.simulate(system, spec, tables, cs, x0, t_sim, workers=os.cpu_count() or 1)
    sess = pb.DlmpcSession(system, spec, mask, "b200")
    traj, _ = sess.simulate(x0, t_sim)
    info = sess.device.info()
    rel = float(np.max(np.abs(traj.states - ref["states"])) / max(1.0, np.max(np.abs(ref["states"]))))
    ok = list(traj.step_iterations) == ref["step_iterations"] and rel <= 1e-9
    print(f"N={n} {t_sim}-step loop, plan {info['mode']} grid {info['grid']} units {info['units']} "
          f"fuse {info['fuse_steps']}: iterations {traj.step_iterations} vs oracle {ref['step_iterations']}, "
          f"states rel err {rel:.2e}, ok {ok} ({time.time() - t0:.0f} s)", flush=True)
    sess.close()
