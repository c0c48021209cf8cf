"""Generate the golden fixtures of tests/golden/ by running the REFERENCE.

Run here (the reference exists only in the build container):

    python tests/golden/make_golden.py [--big]

The reference package is copied from /root/reference/pkg/src to a temp dir
and imported from there (PYTHONDONTWRITEBYTECODE, nothing is written into
/root/reference). Every fixture is produced by the reference's own public API
(`run_scenario`, `admm_solve`, `Executor.run_iteration`, setup builders) and
stored as a small .npz; the tests compare the oracle and the device path
against these files on machines where the reference is absent.
"""

import argparse
import os
import shutil
import sys
import tempfile

os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
sys.dont_write_bytecode = True

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def import_reference():
    tmp = tempfile.mkdtemp(prefix="refpkg_")
    shutil.copytree("/root/reference/pkg/src/locality_mpc", os.path.join(tmp, "locality_mpc"))
    sys.path.insert(0, tmp)
    import locality_mpc as lm
    return lm


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print("wrote", path, sorted(arrays))


def closed_loop(lm, n, d, t, t_sim, seed, strategy="fused", bounded=True, eps=1e-4, max_iters=5000):
    scn = lm.Scenario(n=n, horizon=t, d=d, t_sim=t_sim, seed=seed, strategy=strategy,
                      bounded=bounded, eps=eps, max_iters=max_iters)
    traj, rep = lm.run_scenario(scn)
    system = lm.build_chain_network(n)
    x0 = lm.sample_initial_state(system.partition, np.random.default_rng(seed))
    return dict(x0=x0, states=traj.states, inputs=traj.inputs,
                step_iters=np.array(traj.step_iterations), cost=np.array(rep.closed_loop_cost),
                config=np.array([n, d, t, t_sim, seed]), bounded=np.array(bounded),
                eps=np.array(eps))


def bundle(lm, n, t, d, bounded=True, eps=1e-4, max_iters=5000):
    system = lm.build_chain_network(n)
    spec = lm.make_benchmark_spec(system, t, eps=eps, bounded=bounded, max_iters=max_iters)
    mask = lm.build_locality_mask(system, d, t)
    tables = lm.LayoutTables(mask)
    op = lm.build_dynamics_operator(system, t)
    cs = lm.precompute_column_solvers(op, mask)
    metas = lm.row_index_map(system.partition, t, spec)
    return system, spec, mask, tables, op, cs, metas


def solve_trace(lm, n, t, d, seed, iters, variant="sequential"):
    """Per-iteration residuals + final triple of `iters` Executor iterations."""
    from locality_mpc.admm import AdmmWorkspace
    system, spec, mask, tables, op, cs, metas = bundle(lm, n, t, d)
    x = lm.sample_initial_state(system.partition, np.random.default_rng(seed))
    rd = lm.precompute_row_data(x, spec, tables, metas)
    triple = lm.PhiTriple(tables)
    ws = AdmmWorkspace(triple, cs, spec, row_data=rd)
    res = []
    snaps = {}
    with lm.Executor(lm.ExecStrategy(variant)) as ex:
        for k in range(iters):
            res.append(ex.run_iteration(ws))
            if k in (0, 4, iters - 1):
                for name in ("phi_r", "psi_r", "lam_r", "phi_c", "psi_c", "lam_c", "psi_prev_c"):
                    snaps[f"it{k}_{name}"] = getattr(triple, name).copy()
    return dict(x=x, residuals=np.array(res), config=np.array([n, d, t, seed, iters]), **snaps)


def setup_fixture(lm, n, t, d):
    system, spec, mask, tables, op, cs, metas = bundle(lm, n, t, d)
    out = dict(config=np.array([n, d, t]))
    out["z_indptr"], out["z_indices"], out["z_data"] = op.z.indptr, op.z.indices, op.z.data
    for name in ("rs", "cs", "row_len", "col_len", "col_slot_in_row", "c2r_flat", "r2c_flat",
                 "elem_flat_col", "owner_col"):
        out["tab_" + name] = getattr(tables, name)
    for c, pre in enumerate(cs):
        out[f"col{c}_g"] = pre.g
        out[f"col{c}_rhs"] = pre.rhs
        out[f"col{c}_P"] = pre.projector
        out[f"col{c}_rows"] = pre.constraint_rows
    w = np.array([m.weight for m in metas]); lo = np.array([m.lo for m in metas]); hi = np.array([m.hi for m in metas])
    out["row_w"], out["row_lo"], out["row_hi"] = w, lo, hi
    out["a_indptr"], out["a_indices"], out["a_data"] = system.a.indptr, system.a.indices, system.a.data
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also the N=1000 one-step fixture (~3 min)")
    ap.add_argument("--c2-seeds", action="store_true",
                    help="only the C2 closed loops for seeds 1..20 (the bench's timed seeds, ~6 min)")
    ap.add_argument("--c3", type=int, default=0,
                    help="only the chain N=<c3>, d=3, T=10 step-0 solve (N=3000: ~15 min, 3 GB)")
    args = ap.parse_args()
    lm = import_reference()
    if args.c2_seeds:
        # every seed bench.py cycles through (bench.py: seeds 1..max(8, steps))
        out = {}
        for seed in range(1, 21):
            r = closed_loop(lm, 100, 3, 10, 20, seed)
            out[f"s{seed}_x0"], out[f"s{seed}_states"] = r["x0"], r["states"]
            out[f"s{seed}_inputs"], out[f"s{seed}_iters"] = r["inputs"], r["step_iters"]
            out[f"s{seed}_cost"] = r["cost"]
            print("seed", seed, list(r["step_iters"]), flush=True)
        save("c2_loops_seeds1_20", **out)
        return
    if args.c3:
        save(f"c3_n{args.c3}_step0", **closed_loop(lm, args.c3, 3, 10, 1, 1))
        return

    # C1 step 0 known answers + full 20-step loops
    system, spec, mask, tables, op, cs, metas = bundle(lm, 10, 5, 2)
    x0 = lm.sample_initial_state(system.partition, np.random.default_rng(1))
    rd = lm.precompute_row_data(x0, spec, tables, metas)
    triple = lm.PhiTriple(tables)
    st = lm.admm_solve(rd, cs, triple, spec, lm.ExecStrategy("sequential"))
    u0 = lm.extract_control(triple, x0, metas)
    save("c1_step0", x0=x0, history=np.array(st.residual_history), iterations=np.array(st.iterations),
         u0=u0, **{k: getattr(triple, k) for k in ("phi_r", "psi_r", "lam_r", "phi_c", "psi_c",
                                                     "lam_c", "psi_prev_c")})
    save("c1_loop_seed1", **closed_loop(lm, 10, 2, 5, 20, 1, "sequential"))
    for seed in (2, 3):
        save(f"c1_loop_seed{seed}", **closed_loop(lm, 10, 2, 5, 20, seed))
    save("c2_loop_seed1", **closed_loop(lm, 100, 3, 10, 20, 1))
    save("d1_loop_n30", **closed_loop(lm, 30, 1, 5, 4, 1))
    save("d4_loop_n20", **closed_loop(lm, 20, 4, 6, 5, 2))
    save("unbounded_loop_n8", **closed_loop(lm, 8, 2, 4, 6, 5, bounded=False))
    save("trace_n6_d1_t4", **solve_trace(lm, 6, 4, 1, 1234, 30))
    save("trace_n5_d2_t4", **solve_trace(lm, 5, 4, 2, 7, 20))
    for n, t, d in ((3, 3, 1), (4, 3, 1), (6, 4, 2), (3, 3, 2)):
        save(f"setup_n{n}_t{t}_d{d}", **setup_fixture(lm, n, t, d))
    # edge behaviours
    system, spec, mask, tables, op, cs, metas = bundle(lm, 3, 3, 1)
    traj, rep = lm.dlmpc_simulate(system, spec, mask, np.zeros(6), 5, lm.ExecStrategy("fused"))
    save("zero_state_n3", states=traj.states, inputs=traj.inputs, step_iters=np.array(traj.step_iterations))
    try:
        b = bundle(lm, 3, 3, 1, max_iters=2, eps=1e-12)
        x = lm.sample_initial_state(b[0].partition, np.random.default_rng(1234))
        rd = lm.precompute_row_data(x, b[1], b[3], b[6])
        lm.admm_solve(rd, b[5], lm.PhiTriple(b[3]), b[1], lm.ExecStrategy("sequential"))
    except lm.NotConverged as err:
        save("not_converged_n3", x=x, history=np.array(err.residual_history))
    # the reference's dense KKT oracle (oracle.py:111-127) on unbounded instances
    kk = {}
    for n, t, d in ((2, 3, 1), (3, 4, 2), (4, 3, 1), (4, 4, 2)):
        system = lm.build_chain_network(n)
        spec = lm.make_benchmark_spec(system, t, eps=1e-6, bounded=False)
        mask = lm.build_locality_mask(system, d, t)
        x0 = lm.sample_initial_state(system.partition, np.random.default_rng(31 + n))
        ref = lm.simulate_with_oracle(system, spec, mask, x0, 8)
        kk[f"n{n}_t{t}_d{d}_states"] = ref.states
        kk[f"n{n}_t{t}_d{d}_inputs"] = ref.inputs
        kk[f"n{n}_t{t}_d{d}_x0"] = x0
    save("kkt_oracle", **kk)
    if args.big:
        save("c3_n1000_step0", **closed_loop(lm, 1000, 3, 10, 1, 1))


if __name__ == "__main__":
    main()
