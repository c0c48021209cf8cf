"""Device path vs the reference (golden fixtures) and vs the oracle.

Both arithmetic flavours go through the public API and the C ABI:
  b200-exact : bit-identical to the reference (np.array_equal on every array)
  b200       : identical iteration counts; iterates within FAST_RTOL
               (north_star: 1e-6 in FP64; measured ~1e-14).
"""

import os

import numpy as np
import pytest

import paper_2103_14990_b200 as pb
from conftest import chain_bundle, golden, random_graph_system
from oracle import admm_ref

pytestmark = pytest.mark.gpu

EXACT, FAST = "b200-exact", "b200"
FAST_RTOL = 1e-9
TRIPLE = ("phi_r", "psi_r", "lam_r", "phi_c", "psi_c", "lam_c", "psi_prev_c")
LOOPS = ["c1_loop_seed1", "c1_loop_seed2", "c1_loop_seed3", "c2_loop_seed1", "d1_loop_n30",
         "d4_loop_n20", "unbounded_loop_n8"]


def rel_err(a, b):
    scale = max(1.0, float(np.max(np.abs(b))))
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)))) / scale


def loop_problem(g):
    n, d, t, t_sim, seed = (int(v) for v in g["config"])
    system = pb.build_chain_network(n)
    spec = pb.make_benchmark_spec(system, t, eps=float(g["eps"]), bounded=bool(g["bounded"]))
    mask = pb.build_locality_mask(system, d, t)
    return system, spec, mask, t_sim


@pytest.mark.parametrize("variant", [EXACT, FAST])
def test_c1_step0_admm_solve(variant):
    g = golden("c1_step0")
    b = chain_bundle(10, 5, 2)
    rd = pb.precompute_row_data(g["x0"], b["spec"], b["tables"])
    triple = pb.PhiTriple(b["tables"])
    st = pb.admm_solve(rd, b["col_solvers"], triple, b["spec"], variant)
    assert st.converged and st.iterations == 37 == int(g["iterations"])
    hist = np.array(st.residual_history)
    if variant == EXACT:
        assert np.array_equal(hist, g["history"])
        for name in TRIPLE:
            assert np.array_equal(getattr(triple, name), g[name]), name
    else:
        np.testing.assert_allclose(hist, g["history"], rtol=1e-6, atol=1e-12)
        for name in TRIPLE:
            assert rel_err(getattr(triple, name), g[name]) <= FAST_RTOL, name
    assert triple.padding_leak() == 0.0
    assert triple.layout_disagreement() == 0.0


@pytest.mark.parametrize("variant", [EXACT, FAST])
@pytest.mark.parametrize("name", LOOPS)
def test_closed_loops_against_reference(name, variant):
    g = golden(name)
    system, spec, mask, t_sim = loop_problem(g)
    traj, rep = pb.dlmpc_simulate(system, spec, mask, g["x0"], t_sim, variant)
    assert list(traj.step_iterations) == list(g["step_iters"])
    if variant == EXACT:
        assert np.array_equal(traj.states, g["states"])
        assert np.array_equal(traj.inputs, g["inputs"])
        assert rep.closed_loop_cost == float(g["cost"])
    else:
        assert rel_err(traj.states, g["states"]) <= FAST_RTOL
        assert rel_err(traj.inputs, g["inputs"]) <= FAST_RTOL
    assert rep.ledger.counts_consistent()
    assert rep.ledger.solve_launches == 1


@pytest.mark.parametrize("name", ["c1_loop_seed1", "c2_loop_seed1"])
def test_patch_schedules_against_reference(name, monkeypatch):
    """The patch kernel's two Ψ schedules for chunks of <= 2 columns: the
    register-blocked GEMV pair (kPatchRb, the default at this size) and the
    DMMA tiles it replaces (DLMPC_RB_GEMV=0); both take the reference's
    iteration counts with iterates within FAST_RTOL, and agree to rounding."""
    g = golden(name)
    system, spec, mask, t_sim = loop_problem(g)
    out = {}
    for rb in ("1", "0"):
        monkeypatch.setenv("DLMPC_RB_GEMV", rb)
        sess = pb.DlmpcSession(system, spec, mask, FAST)
        traj, _ = sess.simulate(g["x0"], t_sim)
        assert sess.device.info()["mode"] == "patch"
        sess.close()
        assert list(traj.step_iterations) == list(g["step_iters"])
        assert rel_err(traj.states, g["states"]) <= FAST_RTOL
        assert rel_err(traj.inputs, g["inputs"]) <= FAST_RTOL
        out[rb] = traj.states
    assert rel_err(out["1"], out["0"]) <= 1e-12


def test_c1_band_holds():
    g = golden("c1_loop_seed1")
    system, spec, mask, t_sim = loop_problem(g)
    traj, _ = pb.dlmpc_simulate(system, spec, mask, g["x0"], t_sim, FAST)
    firsts = traj.states[:, 0::2]
    assert firsts.min() >= -0.2 - 1e-6 and firsts.max() <= 1.2 + 1e-6


@pytest.mark.parametrize("variant", [EXACT, FAST])
@pytest.mark.parametrize("name", ["trace_n6_d1_t4", "trace_n5_d2_t4"])
def test_iteration_traces(name, variant):
    """Executor.run_iteration one iteration at a time (reference
    test_strategies.py:187-208): residuals and triple snapshots."""
    g = golden(name)
    n, d, t, seed, iters = (int(v) for v in g["config"])
    b = chain_bundle(n, t, d)
    rd = pb.precompute_row_data(g["x"], b["spec"], b["tables"])
    triple = pb.PhiTriple(b["tables"])
    ws = pb.AdmmWorkspace(triple, b["col_solvers"], b["spec"], row_data=rd)
    with pb.Executor(pb.ExecStrategy(variant)) as ex:
        for k in range(iters):
            res = ex.run_iteration(ws)
            if variant == EXACT:
                assert res == tuple(g["residuals"][k]), k
            else:
                np.testing.assert_allclose(res, g["residuals"][k], rtol=1e-6, atol=1e-13)
            if f"it{k}_psi_c" in g:
                for nm in TRIPLE:
                    if variant == EXACT:
                        assert np.array_equal(getattr(triple, nm), g[f"it{k}_{nm}"]), (k, nm)
                    else:
                        assert rel_err(getattr(triple, nm), g[f"it{k}_{nm}"]) <= FAST_RTOL, (k, nm)
        assert ex.ledger.iterations == iters and ex.ledger.counts_consistent()
    ws.close()


@pytest.mark.parametrize("variant", [EXACT, FAST])
def test_zero_initial_state_stays_at_origin(variant):
    g = golden("zero_state_n3")
    b = chain_bundle(3, 3, 1)
    traj, rep = pb.dlmpc_simulate(b["system"], b["spec"], b["mask"], np.zeros(6), 5, variant)
    assert list(traj.step_iterations) == list(g["step_iters"])
    assert traj.step_iterations[-1] == 1
    assert np.max(np.abs(traj.states)) <= 1e-9


@pytest.mark.parametrize("variant", [EXACT, FAST])
def test_not_converged_carries_history(variant):
    g = golden("not_converged_n3")
    b = chain_bundle(3, 3, 1, eps=1e-12, max_iters=2)
    rd = pb.precompute_row_data(g["x"], b["spec"], b["tables"])
    with pytest.raises(pb.NotConverged) as exc:
        pb.admm_solve(rd, b["col_solvers"], pb.PhiTriple(b["tables"]), b["spec"], variant)
    hist = np.array(exc.value.residual_history)
    assert hist.shape == (2, 2)
    if variant == EXACT:
        assert np.array_equal(hist, g["history"])
    with pytest.raises(pb.NotConverged) as exc:
        pb.dlmpc_simulate(b["system"], b["spec"], b["mask"], g["x"], 3, variant)
    assert exc.value.step == 0 and len(exc.value.residual_history) == 2


def test_huge_tolerance_converges_in_one_iteration():
    b = chain_bundle(2, 3, 1, eps=1e6)
    x = pb.sample_initial_state(b["system"].partition, np.random.default_rng(1234))
    rd = pb.precompute_row_data(x, b["spec"], b["tables"])
    st = pb.admm_solve(rd, b["col_solvers"], pb.PhiTriple(b["tables"]), b["spec"])
    assert st.iterations == 1


@pytest.mark.parametrize("variant", [EXACT, FAST])
def test_row_infeasible_reports_reference_row_and_step(variant):
    b = chain_bundle(2, 3, 1)
    spec = b["spec"]
    spec.state_lo[0, 1] = 0.5
    spec.state_hi[0, 1] = 1.0
    with pytest.raises(pb.RowInfeasible) as ref_exc:
        pb.precompute_row_data(np.zeros(4), spec, b["tables"])
    with pytest.raises(pb.RowInfeasible) as exc:
        pb.dlmpc_simulate(b["system"], spec, b["mask"], np.zeros(4), 3, variant)
    assert exc.value.row == ref_exc.value.row
    assert exc.value.step == 0


@pytest.mark.parametrize("variant", [EXACT, FAST])
def test_generic_graph_against_oracle(variant):
    """Non-contiguous balls: the generic two-phase kernel and col_irow tables."""
    rng = np.random.default_rng(11)
    system = random_graph_system(9, rng)
    spec = pb.make_benchmark_spec(system, 3)
    mask = pb.build_locality_mask(system, 2, 3)
    tables = pb.LayoutTables(mask)
    cs = pb.precompute_column_solvers(pb.build_dynamics_operator(system, 3), mask)
    x0 = rng.uniform(0.0, 1.0, system.n_states)
    ref = admm_ref.simulate(system, spec, tables, cs, x0, 4)
    traj, _ = pb.dlmpc_simulate(system, spec, mask, x0, 4, variant)
    assert list(traj.step_iterations) == ref["step_iterations"]
    if variant == EXACT:
        assert np.array_equal(traj.states, ref["states"])
    else:
        assert rel_err(traj.states, ref["states"]) <= FAST_RTOL


@pytest.mark.parametrize("variant", [EXACT, FAST])
@pytest.mark.parametrize("kw", [{"two_inputs": True}, {"coupling_radius": 2}])
def test_chain_variants_against_oracle(variant, kw):
    b = chain_bundle(9, 4, 2, **kw)
    x0 = pb.sample_initial_state(b["system"].partition, np.random.default_rng(2))
    ref = admm_ref.simulate(b["system"], b["spec"], b["tables"], b["col_solvers"], x0, 5)
    traj, _ = pb.dlmpc_simulate(b["system"], b["spec"], b["mask"], x0, 5, variant)
    assert list(traj.step_iterations) == ref["step_iterations"]
    if variant == EXACT:
        assert np.array_equal(traj.states, ref["states"])
        assert np.array_equal(traj.inputs, ref["inputs"])
    else:
        assert rel_err(traj.states, ref["states"]) <= FAST_RTOL


def test_warm_start_and_cold_start_semantics():
    g = golden("c1_loop_seed1")
    system, spec, mask, _ = loop_problem(g)
    cold, _ = pb.dlmpc_simulate(system, spec, mask, g["x0"], 4, EXACT, warm_start=False)
    warm, _ = pb.dlmpc_simulate(system, spec, mask, g["x0"], 4, EXACT)
    assert warm.step_iterations == list(g["step_iters"][:4])
    assert cold.step_iterations[0] == warm.step_iterations[0]
    assert sum(cold.step_iterations) > sum(warm.step_iterations)
    # a second call starts cold again (fresh PhiTriple in the reference)
    again, _ = pb.dlmpc_simulate(system, spec, mask, g["x0"], 4, EXACT)
    assert np.array_equal(again.states, warm.states)


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(__file__), "golden",
                                                    "c3_n1000_step0.npz")), reason="fixture not generated")
@pytest.mark.parametrize("variant", [EXACT, FAST])
def test_n1000_step0_against_reference(variant):
    g = golden("c3_n1000_step0")
    system, spec, mask, t_sim = loop_problem(g)
    traj, _ = pb.dlmpc_simulate(system, spec, mask, g["x0"], t_sim, variant)
    assert list(traj.step_iterations) == list(g["step_iters"]) == [78]
    if variant == EXACT:
        assert np.array_equal(traj.states, g["states"])
    else:
        assert rel_err(traj.states, g["states"]) <= FAST_RTOL


def test_patch_and_twophase_kernels_agree():
    """The contiguous patch kernel and the generic two-phase kernel agree:
    identical iteration counts, iterates equal to rounding (the patch kernel
    multiplies by per-step reciprocals and takes the GEMV path for small
    chunks)."""
    system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=300, d=3, horizon=10, seed=4))
    a = pb.DlmpcSession(system, spec, mask, FAST)
    os.environ["DLMPC_FORCE_TWOPHASE"] = "1"
    try:
        b = pb.DlmpcSession(system, spec, mask, FAST)
    finally:
        os.environ.pop("DLMPC_FORCE_TWOPHASE")
    ta, _ = a.simulate(x0, 3)
    tb, _ = b.simulate(x0, 3)
    assert ta.step_iterations == tb.step_iterations
    assert rel_err(ta.states, tb.states) <= 1e-12
    a.close(); b.close()


@pytest.mark.parametrize("n,t_sim", [(100, 4), (2500, 2)])
def test_stream_and_patch_kernels_agree(n, t_sim):
    """The stream kernel (Φ dots accumulated by the Ψ epilogues, ψ/λ staged
    by cp.async, register epilogue) and the patch kernel agree: identical
    iteration counts, iterates equal to rounding; and the stream kernel is
    run to run deterministic (its cross-unit Φ partials are summed in a
    fixed unit order)."""
    system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=n, d=3, horizon=10, seed=5))
    os.environ["DLMPC_FORCE_STREAM"] = "1"
    try:
        a = pb.DlmpcSession(system, spec, mask, FAST)
    finally:
        os.environ.pop("DLMPC_FORCE_STREAM")
    os.environ["DLMPC_NO_STREAM"] = "1"
    try:
        b = pb.DlmpcSession(system, spec, mask, FAST)
    finally:
        os.environ.pop("DLMPC_NO_STREAM")
    os.environ.update(DLMPC_FORCE_STREAM="1", DLMPC_WARP_SPEC="0")
    try:
        c = pb.DlmpcSession(system, spec, mask, FAST)   # lockstep chunk loop (no warp split)
    finally:
        os.environ.pop("DLMPC_FORCE_STREAM"); os.environ.pop("DLMPC_WARP_SPEC")
    assert a.device.info()["mode"] == "stream" and b.device.info()["mode"] == "patch"
    ta, _ = a.simulate(x0, t_sim)
    ta2, _ = a.simulate(x0, t_sim)
    tb, _ = b.simulate(x0, t_sim)
    tc, _ = c.simulate(x0, t_sim)
    assert ta.step_iterations == tb.step_iterations
    assert rel_err(ta.states, tb.states) <= 1e-12
    assert np.array_equal(ta.states, ta2.states) and np.array_equal(ta.inputs, ta2.inputs)
    # the warp split changes who computes, not what: bit for bit
    assert np.array_equal(ta.states, tc.states) and np.array_equal(ta.inputs, tc.inputs)
    a.close(); b.close(); c.close()


@pytest.mark.slow
def test_large_network_properties():
    """N = 20,000 (beyond the oracle): convergence, determinism, feasibility
    of ψ (g ψ = rhs per column, checked on sampled columns), and exact vs fast
    agreement of iteration counts."""
    from paper_2103_14990_b200.device import PSI
    system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=20000, d=3, horizon=10, seed=1))
    sess = pb.DlmpcSession(system, spec, mask, FAST)
    t1, _ = sess.simulate(x0, 2)
    t2, _ = sess.simulate(x0, 2)
    assert t1.step_iterations == t2.step_iterations
    assert np.array_equal(t1.states, t2.states)
    L = sess.layout
    psi = sess.device.get(PSI)
    cc = sess.classes
    rng = np.random.default_rng(0)
    for c in rng.choice(L.n_cols, 64, replace=False):
        cl = cc.classes[cc.col_class[c]]
        j = L.col_owner[c]
        s = int(L.col_len[c])
        col_ref = psi[c * L.s_pad + L.ref_pos[j, :s]]
        assert np.max(np.abs(cl.g @ col_ref - cc.rhs[c])) <= 1e-10
    ex = pb.DlmpcSession(system, spec, mask, EXACT)
    te, _ = ex.simulate(x0, 1)
    assert te.step_iterations[0] == t1.step_iterations[0]
    assert rel_err(te.states, t1.states[:2]) <= FAST_RTOL
    sess.close(); ex.close()


C4_GRID = [(20, 1, 5), (16, 1, 10), (20, 2, 20), (14, 3, 30), (20, 4, 10), (20, 5, 5), (20, 6, 5)]


@pytest.mark.parametrize("variant", [EXACT, FAST])
@pytest.mark.parametrize("n,d,t", C4_GRID)
def test_locality_horizon_sweep_against_oracle(n, d, t, variant):
    """SURVEY config C4 (d = 1..6, T = 5..30; longest-vector padding): iteration
    counts and trajectories vs the oracle on a 2-step closed loop. T=30 and
    d=3 makes the Ψ operator (623 x 175) too large for shared memory, which
    exercises the global-operator path and wide rows."""
    system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=n, d=d, horizon=t, seed=3))
    tables = pb.LayoutTables(mask)
    cs = pb.precompute_column_solvers(pb.build_dynamics_operator(system, t), mask)
    ref = admm_ref.simulate(system, spec, tables, cs, x0, 2)
    traj, _ = pb.dlmpc_simulate(system, spec, mask, x0, 2, variant)
    assert list(traj.step_iterations) == ref["step_iterations"]
    if variant == EXACT:
        assert np.array_equal(traj.states, ref["states"])
        assert np.array_equal(traj.inputs, ref["inputs"])
    else:
        assert rel_err(traj.states, ref["states"]) <= FAST_RTOL


@pytest.mark.parametrize("variant", [EXACT, FAST])
def test_closed_loop_cost_matches_kkt_oracle(variant):
    """The reference's acceptance criterion (test_acceptance.py:112-132): on
    12 unbounded chains the ADMM closed-loop cost is within 1e-4 (relative)
    of the dense KKT solve -- an independent algorithm (oracle/kkt.py)."""
    from oracle import kkt
    worst = 0.0
    for n in (2, 3, 4):
        for t in (3, 4):
            for d in (1, 2):
                system = pb.build_chain_network(n)
                spec = pb.make_benchmark_spec(system, t, eps=1e-6, bounded=False)
                mask = pb.build_locality_mask(system, d, t)
                x0 = pb.sample_initial_state(system.partition, np.random.default_rng(31 + n))
                traj, rep = pb.dlmpc_simulate(system, spec, mask, x0, 8, variant)
                states, inputs = kkt.kkt_closed_loop(system, spec, mask, x0, 8)
                ref_cost = float(np.sum(states ** 2) + np.sum(inputs ** 2))
                rel = abs(rep.closed_loop_cost - ref_cost) / max(1.0, ref_cost)
                worst = max(worst, rel)
                assert rel <= 1e-4, (n, t, d, rel)


class TestVerifyFixedPoint:
    """On-device audit (reference verify_fixed_point, admm.py:417-434, and
    its tests test_admm.py:312-363)."""

    def test_exact_fixed_point_by_construction(self):
        import scipy.sparse as sp
        part = pb.SubsystemPartition(((0, 1),), ((0, 0),))
        graph = pb.SubsystemGraph.from_edges(1, [])
        system = pb.LtiSystem(sp.csr_matrix((1, 1)), sp.csr_matrix((1, 0)), part, graph)
        mask = pb.build_locality_mask(system, 0, 2)
        tables = pb.LayoutTables(mask)
        operator = pb.build_dynamics_operator(system, 2)
        spec = pb.make_benchmark_spec(system, 2, bounded=False)
        rd = pb.precompute_row_data(np.zeros(1), spec, tables)
        triple = pb.PhiTriple(tables)
        pinned = np.array([1.0, 0.0])
        triple.phi_r[:, 0] = pinned
        triple.psi_r[:, 0] = pinned
        triple.exchange_phi_row_to_col()
        triple.psi_c[:] = triple.phi_c
        rep = pb.verify_fixed_point(triple, rd, operator, spec)
        assert (rep.dynamics_residual, rep.resolve_residual, rep.consensus_gap) == (0.0, 0.0, 0.0)

    @pytest.mark.parametrize("variant", [EXACT, FAST])
    def test_converged_solve_passes_and_perturbation_fails(self, variant):
        b = chain_bundle(4, 4, 2)
        x0 = pb.sample_initial_state(b["system"].partition, np.random.default_rng(1234))
        rd = pb.precompute_row_data(x0, b["spec"], b["tables"])
        triple = pb.PhiTriple(b["tables"])
        pb.admm_solve(rd, b["col_solvers"], triple, b["spec"], variant)
        rep = pb.verify_fixed_point(triple, rd, b["operator"], b["spec"])
        assert rep.passed
        assert max(rep.dynamics_residual, rep.resolve_residual, rep.consensus_gap) <= 1e-3
        assert rep.dynamics_residual <= 1e-12
        triple.phi_r[0, 0] += 0.1
        rep = pb.verify_fixed_point(triple, rd, b["operator"], b["spec"])
        assert rep.resolve_residual >= 0.09
        assert not rep.passed

    def test_audit_matches_host_recomputation(self):
        """The device audit equals a host recomputation of the reference's
        three residuals on the same (exact-mode) triple."""
        b = chain_bundle(6, 4, 2)
        x0 = pb.sample_initial_state(b["system"].partition, np.random.default_rng(5))
        rd = pb.precompute_row_data(x0, b["spec"], b["tables"])
        triple = pb.PhiTriple(b["tables"])
        pb.admm_solve(rd, b["col_solvers"], triple, b["spec"], EXACT)
        rep = pb.verify_fixed_point(triple, rd, b["operator"], b["spec"])
        tb = b["tables"]
        dyn = float(np.max(np.abs(b["operator"].residual(triple.psi_dense()))))
        orc = admm_ref.OracleSolver(tb, b["col_solvers"], 1.0)
        w, lo, hi = b["spec"].row_arrays()
        orc.row_data, _ = admm_ref.row_data_for(x0, tb, w, lo, hi)
        orc.psi_r[:], orc.lam_r[:] = triple.psi_r, triple.lam_r
        orc._phi(0, tb.n_rows)
        res = float(np.max(np.abs((orc.phi_r - triple.phi_r)[tb.row_valid])))
        gap = float(np.max(np.abs((triple.phi_r - triple.psi_r)[tb.row_valid])))
        assert rep.resolve_residual == res and rep.consensus_gap == gap
        np.testing.assert_allclose(rep.dynamics_residual, dyn, rtol=1e-6, atol=1e-15)

    @pytest.mark.parametrize("variant", [EXACT, FAST])
    def test_closed_loop_audit(self, variant):
        """dlmpc_simulate(audit=True): worst residuals over the loop within
        10 x eps (the reference's acceptance audit, test_acceptance.py:98-109),
        and the audited loop reproduces the reference trajectory."""
        g = golden("c1_loop_seed1")
        system, spec, mask, t_sim = loop_problem(g)
        traj, rep = pb.dlmpc_simulate(system, spec, mask, g["x0"], t_sim, variant, audit=True)
        assert list(traj.step_iterations) == list(g["step_iters"])
        for key in ("dynamics_residual", "resolve_residual", "consensus_gap"):
            assert rep.audit_worst[key] <= 1e-3, key
        if variant == EXACT:
            assert np.array_equal(traj.states, g["states"])


def test_stream_host_driven_iterations_equal_one_solve():
    """Host-driven dlmpc_iterate(1) calls continue the stream kernel's Φ-dot
    partials across launches (the partitioned driver's loop): bit for bit the
    same iterates and residual history as one dlmpc_solve."""
    from paper_2103_14990_b200.device import PSI, LAM
    system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=2500, d=3, horizon=10, seed=3))
    os.environ["DLMPC_FORCE_STREAM"] = "1"
    try:
        s = pb.DlmpcSession(system, spec, mask, FAST)
    finally:
        os.environ.pop("DLMPC_FORCE_STREAM")
    dev = s.device
    assert dev.info()["mode"] == "stream"
    dev.zero(); dev.set_x(x0)
    n, hist, ok = dev.solve(spec.max_iters, spec.eps_pri, spec.eps_dual)
    assert ok
    psi_a, lam_a = dev.get(PSI), dev.get(LAM)
    dev.zero(); dev.set_x(x0)
    hist_b = np.concatenate([dev.iterate(1) for _ in range(n)])
    assert np.array_equal(hist, hist_b)
    assert np.array_equal(dev.get(PSI), psi_a) and np.array_equal(dev.get(LAM), lam_a)
    s.close()


@pytest.mark.parametrize("variant", [EXACT, FAST])
def test_grid_network_against_oracle(variant):
    """A 5x6 grid (generic graph path: diamond balls, two-phase kernel)."""
    from conftest import grid_network
    system = grid_network(5, 6)
    spec = pb.make_benchmark_spec(system, 4)
    mask = pb.build_locality_mask(system, 2, 4)
    tables = pb.LayoutTables(mask)
    cs = pb.precompute_column_solvers(pb.build_dynamics_operator(system, 4), mask)
    x0 = pb.sample_initial_state(system.partition, np.random.default_rng(8))
    ref = admm_ref.simulate(system, spec, tables, cs, x0, 3)
    traj, _ = pb.dlmpc_simulate(system, spec, mask, x0, 3, variant)
    assert list(traj.step_iterations) == ref["step_iterations"]
    if variant == EXACT:
        assert np.array_equal(traj.states, ref["states"])
        assert np.array_equal(traj.inputs, ref["inputs"])
    else:
        assert rel_err(traj.states, ref["states"]) <= FAST_RTOL
