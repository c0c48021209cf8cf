"""Step-0 parity at N sizes without fixtures: the device fast path against
the CPU oracle (oracle/admm_ref.py, test infrastructure) -- iteration count
equal, x1 within 1e-9 relative -- and the kernel plan that ran.
usage: python tools/n_oracle_sweep.py N [N ...]"""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import paper_2103_14990_b200 as pb
from oracle import admm_ref
for n in [int(a) for a in sys.argv[1:]] or [300, 2000]:
    t0 = time.time()
    system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=n, d=3, horizon=10, t_sim=1, seed=1))
    tables = pb.LayoutTables(mask)
    cs = pb.precompute_column_solvers(pb.build_dynamics_operator(system, 10), mask)
    ref = admm_ref.simulate(system, spec, tables, cs, x0, 1, workers=os.cpu_count() or 1)
    sess = pb.DlmpcSession(system, spec, mask, "b200")
    traj, _ = sess.simulate(x0, 1)
    info = sess.device.info()
    rel = float(np.max(np.abs(traj.states[1] - ref["states"][1])) / max(1.0, np.max(np.abs(ref["states"][1]))))
    ok = list(traj.step_iterations) == ref["step_iterations"] and rel <= 1e-9
    print(f"N={n} plan {info['mode']} grid {info['grid']} units {info['units']} cache_phi {info['cache_phi']}: "
          f"iterations {traj.step_iterations} vs oracle {ref['step_iterations']}, x1 rel err {rel:.2e}, ok {ok} "
          f"({time.time() - t0:.0f} s)", flush=True)
    sess.close()
