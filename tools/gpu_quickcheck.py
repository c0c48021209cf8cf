"""Quick device-vs-oracle check used during development (not a test)."""
import sys, time, numpy as np
sys.path.insert(0, '.')
from paper_2103_14990_b200 import system_model as sm, sls_core as sc
from paper_2103_14990_b200.devlayout import DeviceLayout
from paper_2103_14990_b200.device import DeviceSession, PSI, LAM, PHI
from oracle import admm_ref

def spec_for(system, T):
    n_x, n_u = system.n_states, system.n_inputs
    sw = np.zeros((n_x, T)); sw[:, 1:T-1] = 1.0
    lo = np.full((n_x, T), -np.inf); hi = np.full((n_x, T), np.inf)
    lo[0::2, 1:] = -0.2; hi[0::2, 1:] = 1.2
    return sc.ProblemSpec(T, sw, np.ones((n_u, T-1)), np.ones(n_x), lo, hi, np.full((n_u, T-1), -np.inf), np.full((n_u, T-1), np.inf))

for (n, d, T, tsim) in [(10, 2, 5, 20), (100, 3, 10, 20)]:
    B = sm.build_chain_network(n); sp_ = spec_for(B, T)
    mb = sm.build_locality_mask(B, d, T); tb = sc.LayoutTables(mb)
    op = sc.build_dynamics_operator(B, T); cc = sc.build_column_classes(op, mb)
    cs = sc.precompute_column_solvers(op, mb, cc)
    rng = np.random.default_rng(1)
    x0 = np.empty(2*n); x0[0::2] = rng.uniform(0, 1, n); x0[1::2] = rng.uniform(-0.5, 0.5, n)
    t0 = time.time(); ref = admm_ref.simulate(B, sp_, tb, cs, x0, tsim); t1 = time.time()
    for exact in (True, False):
        L = DeviceLayout(B, sp_, mb, cc, exact=exact)
        ds = DeviceSession(L)
        print(n, "exact" if exact else "fast", ds.info(), flush=True)
        # single solve parity (step 0)
        ds.set_x(x0)
        it, hist, ok = ds.solve(5000, 1e-4, 1e-4)
        w, lo, hi = sp_.row_arrays()
        orc = admm_ref.OracleSolver(tb, cs, 1.0); rd, _ = admm_ref.row_data_for(x0, tb, w, lo, hi)
        it2, hist2, ok2 = orc.solve(rd, 5000, 1e-4, 1e-4)
        cg = L.column_gather(tb)
        psi_c = np.where(cg >= 0, ds.get(PSI)[np.maximum(cg, 0)], 0.0)
        print("  solve iters", it, it2, "hist equal", np.array_equal(hist, np.array(hist2)), "max hist diff", np.max(np.abs(hist - np.array(hist2))) if it == it2 else None,
              "psi equal", np.array_equal(psi_c, orc.psi_c), "psi maxdiff", np.max(np.abs(psi_c - orc.psi_c)), flush=True)
        out = ds.simulate(x0, tsim, 5000, 1e-4, 1e-4)
        ms, _ = ds.last_timing()
        print("  sim iters", out['step_iterations'] == ref['step_iterations'], sum(out['step_iterations']),
              "states equal", np.array_equal(out['states'], ref['states']), "rel", np.max(np.abs(out['states'] - ref['states'])) / np.max(np.abs(ref['states'])),
              f"gpu {ms:.3f} ms  oracle {1e3*(t1-t0):.1f} ms", flush=True)
        for rep in range(3):
            out = ds.simulate(x0, tsim, 5000, 1e-4, 1e-4)
            print("   rep", ds.last_timing()[0], "ms", flush=True)
        ds.close()
