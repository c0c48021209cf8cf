"""The reference's five schedule names and scalar stage functions, on the GPU.

`naive`, `padded`, `fused` and `patch-local` run as per-iteration device
schedules over the reference's own dual padded layout
(csrc/dlmpc_schedules.cuh); `sequential` is the single-launch exact kernel.
All of them use the reference's arithmetic, so every iterate, history and
trajectory must equal the reference's fixtures BIT FOR BIT (the reference's
own cross-strategy determinism property, test_acceptance.py:55-65), and the
ledger must count the reference's per-iteration constants from real device
events (strategies.py:49-55, 120-123).
"""

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2103_14990_b200 as pb
from conftest import chain_bundle, golden
from paper_2103_14990_b200.admm import AdmmWorkspace

pytestmark = pytest.mark.gpu

REF = ("sequential", "naive", "padded", "fused", "patch-local")
STAGED = ("naive", "padded", "fused", "patch-local")
TRIPLE = ("phi_r", "psi_r", "lam_r", "phi_c", "psi_c", "lam_c", "psi_prev_c")
COUNTS = {"sequential": (0, 0, 0), "naive": (4, 4, 0), "padded": (4, 4, 0), "fused": (1, 2, 1),
          "patch-local": (0, 1, 1)}


@pytest.mark.parametrize("variant", REF)
def test_c1_step0_solve_bitwise(variant):
    g = golden("c1_step0")
    b = chain_bundle(10, 5, 2)
    rd = pb.precompute_row_data(g["x0"], b["spec"], b["tables"])
    triple = pb.PhiTriple(b["tables"])
    ex = pb.Executor(pb.ExecStrategy(variant))
    st = pb.admm_solve(rd, b["col_solvers"], triple, b["spec"], executor=ex)
    assert st.iterations == int(g["iterations"]) == 37
    assert np.array_equal(np.array(st.residual_history), g["history"])
    for name in TRIPLE:
        assert np.array_equal(getattr(triple, name), g[name]), name
    assert triple.padding_leak() == 0.0 and triple.layout_disagreement() == 0.0
    led = ex.ledger
    assert (led.host_syncs_per_iter, led.kernel_launches_per_iter, led.flag_reads_per_iter) == COUNTS[variant]
    assert led.counts_consistent()
    if variant in STAGED:
        assert led.iterations == 37
        assert led.kernel_launch_events == 37 * COUNTS[variant][1]
    if variant == "patch-local":
        assert led.duplicated_row_computations == 37 * pb.patch_duplication(pb.build_patches(b["tables"]))


@pytest.mark.parametrize("variant", STAGED)
@pytest.mark.parametrize("name", ["trace_n6_d1_t4", "trace_n5_d2_t4"])
def test_executor_traces_bitwise(name, variant):
    """Executor.run_iteration one iteration at a time (the triple crosses the
    boundary every call): residuals and snapshots of the reference's traces."""
    g = golden(name)
    n, d, t, seed, iters = (int(v) for v in g["config"])
    b = chain_bundle(n, t, d)
    rd = pb.precompute_row_data(g["x"], b["spec"], b["tables"])
    triple = pb.PhiTriple(b["tables"])
    patches = pb.build_patches(b["tables"]) if variant == "patch-local" else None
    ws = AdmmWorkspace(triple, b["col_solvers"], b["spec"], patches=patches, row_data=rd)
    with pb.Executor(pb.ExecStrategy(variant)) as ex:
        for k in range(iters):
            res = ex.run_iteration(ws)
            assert res == tuple(g["residuals"][k]), k
            assert triple.padding_leak() == 0.0
            assert triple.layout_disagreement() == 0.0
            if k in (0, 4, iters - 1):
                for nm in TRIPLE:
                    assert np.array_equal(getattr(triple, nm), g[f"it{k}_{nm}"]), (k, nm)
        assert ex.ledger.counts_consistent()
    ws.close()


@pytest.mark.parametrize("variant", REF)
@pytest.mark.parametrize("name", ["c1_loop_seed1", "c1_loop_seed2", "d1_loop_n30", "unbounded_loop_n8"])
def test_closed_loops_bitwise(name, variant):
    g = golden(name)
    n, d, t, t_sim, seed = (int(v) for v in g["config"])
    system = pb.build_chain_network(n)
    spec = pb.make_benchmark_spec(system, t, eps=float(g["eps"]), bounded=bool(g["bounded"]))
    mask = pb.build_locality_mask(system, d, t)
    traj, rep = pb.dlmpc_simulate(system, spec, mask, g["x0"], t_sim, pb.ExecStrategy(variant))
    assert list(traj.step_iterations) == list(g["step_iters"])
    assert np.array_equal(traj.states, g["states"]) and np.array_equal(traj.inputs, g["inputs"])
    assert rep.closed_loop_cost == float(g["cost"])
    assert rep.ledger.counts_consistent()
    assert rep.ledger.host_syncs_per_iter == COUNTS[variant][0]
    assert rep.iters_total == int(np.sum(g["step_iters"]))


@pytest.mark.parametrize("variant", STAGED)
def test_staged_closed_loop_audit_and_failures(variant):
    """audit=True and the failure paths (NotConverged carries the step,
    RowInfeasible the reference row) through a device schedule."""
    b = chain_bundle(4, 4, 2)
    x0 = pb.sample_initial_state(b["system"].partition, np.random.default_rng(3))
    traj, rep = pb.dlmpc_simulate(b["system"], b["spec"], b["mask"], x0, 3, pb.ExecStrategy(variant), audit=True)
    for key in ("dynamics_residual", "resolve_residual", "consensus_gap"):
        assert rep.audit_worst[key] <= 1e-3
    tight = pb.make_benchmark_spec(b["system"], 4, eps=1e-12, max_iters=2)
    with pytest.raises(pb.NotConverged) as exc:
        pb.dlmpc_simulate(b["system"], tight, b["mask"], x0, 2, pb.ExecStrategy(variant))
    assert exc.value.step == 0 and len(exc.value.residual_history) == 2


def test_workspace_stage_methods_compose_to_an_iteration():
    """The reference's AdmmWorkspace stage kernels, called one by one in the
    `sequential` order (strategies.py:262-281) on row / column slices, give
    the reference's iteration bit for bit; _phi_compute writes nothing."""
    g = golden("trace_n5_d2_t4")
    n, d, t, seed, iters = (int(v) for v in g["config"])
    b = chain_bundle(n, t, d)
    rd = pb.precompute_row_data(g["x"], b["spec"], b["tables"])
    triple = pb.PhiTriple(b["tables"])
    ws = AdmmWorkspace(triple, b["col_solvers"], b["spec"], row_data=rd)
    for k in range(5):
        before = triple.phi_r.copy()
        fresh = ws._phi_compute(slice(0, ws.n_rows))
        assert np.array_equal(triple.phi_r, before)
        for r in range(ws.n_rows):
            ws.phi_rows(slice(r, r + 1))
        assert np.array_equal(triple.phi_r, fresh)
        ws.exchange_phi_to_col()
        for c in range(ws.n_cols):
            ws.psi_cols(slice(c, c + 1))
        ws.lambda_cols(np.arange(ws.n_cols))
        ws.conv_cols(slice(0, ws.n_cols))
        ws.exchange_psi_lam_to_row()
        assert ws.reduce_residuals() == tuple(g["residuals"][k])
    for nm in TRIPLE:
        assert np.array_equal(getattr(triple, nm), g[f"it4_{nm}"]), nm
    ws.close()


class TestScalarStageFunctions:
    """The reference's scalar functions (admm.py:28-74, 350-369) as device
    operators, against the reference's own known answers
    (pkg/tests/test_admm.py) and against numpy restatements."""

    def make_row(self, a, weight=1.0, lo=-np.inf, hi=np.inf):
        a = np.asarray(a, float)
        return pb.RowPrecomp(0, np.arange(a.size), a, float(a @ a), weight, lo, hi)

    def test_phi_row_solve_known_answers(self):
        v = np.array([0.3, 0.7])
        assert np.array_equal(pb.phi_row_solve(self.make_row([2.0, -1.0], weight=0.0), v), v)
        assert np.array_equal(pb.phi_row_solve(self.make_row([0.0, 0.0], lo=-1.0, hi=1.0), np.array([0.4, -0.2])),
                              [0.4, -0.2])
        np.testing.assert_allclose(pb.phi_row_solve(self.make_row([1.0, 0.0]), np.array([1.0, 1.0])),
                                   [1.0 / 3.0, 1.0], atol=1e-12)
        np.testing.assert_allclose(pb.phi_row_solve(self.make_row([1.0, 0.0], lo=0.5, hi=2.0), np.array([1.0, 1.0])),
                                   [0.5, 1.0], atol=1e-12)
        with pytest.raises(pb.RowInfeasible):
            pb.phi_row_solve(self.make_row([0.0], lo=0.5, hi=1.0), np.array([0.0]))

    def test_phi_row_solve_matches_closed_form_bitwise(self, rng):
        for _ in range(50):
            k = int(rng.integers(1, 6))
            a, v = rng.standard_normal(k), rng.standard_normal(k)
            w, rho = float(rng.uniform(0, 3)), float(rng.uniform(0.2, 4))
            lo, hi = sorted(rng.uniform(-2, 2, 2))
            row = self.make_row(a, weight=w, lo=lo, hi=hi)
            c = float(pb.ascending_dot(v, a))
            y = min(max(rho * c / (rho + 2.0 * w * row.a_dot_a), lo), hi)
            assert np.array_equal(pb.phi_row_solve(row, v, rho=rho), v + ((y - c) / row.a_dot_a) * a)

    def test_psi_column_solve_matches_pairwise_and_pinv(self, rng):
        for _ in range(20):
            m, n = int(rng.integers(1, 4)), int(rng.integers(4, 40))
            g = rng.standard_normal((m, n))
            rhs, k = rng.standard_normal(m), rng.standard_normal(n)
            proj = g.T @ np.linalg.inv(g @ g.T)
            pre = pb.ColumnPrecomp(0, np.arange(n), np.arange(m), g, rhs, proj)
            got = pb.psi_column_solve(pre, k)
            resid = rhs - (g * k).sum(axis=1)
            assert np.array_equal(got, k + (proj * resid).sum(axis=1))
            np.testing.assert_allclose(got, k - np.linalg.pinv(g) @ (g @ k - rhs), atol=1e-10)

    def test_lambda_and_residuals(self):
        assert np.array_equal(pb.lambda_update(np.array([0.5]), np.array([1.0]), np.array([0.25])), [1.25])
        with pytest.raises(ValueError):
            pb.lambda_update(np.zeros(2), np.zeros(3), np.zeros(2))
        system = pb.build_chain_network(1)
        mask = pb.build_locality_mask(system, 0, 2)
        triple = pb.PhiTriple(pb.LayoutTables(mask))
        triple.phi_c[0, 0], triple.psi_c[0, 0] = 1.0, 0.75
        prev = triple.psi_prev_c[0].copy()
        prev[0] = 0.5
        assert pb.column_residuals(triple, 0, prev, rho=2.0) == (0.25, 0.5)

    def test_extract_control_and_step_dynamics(self):
        g = golden("c1_step0")
        b = chain_bundle(10, 5, 2)
        triple = pb.PhiTriple(b["tables"])
        triple.phi_r[:] = g["phi_r"]
        metas = pb.row_index_map(b["system"].partition, 5, b["spec"])
        u = pb.extract_control(triple, g["x0"], metas)
        assert np.array_equal(u, g["u0"])
        x1 = pb.step_dynamics(b["system"], g["x0"], u)
        assert np.array_equal(x1, b["system"].a @ g["x0"] + b["system"].b @ u)
        with pytest.raises(ValueError):
            pb.step_dynamics(b["system"], np.zeros(3), u)
        # an isolated node and zero dynamics (reference test_admm.py:234-247)
        s1 = pb.build_chain_network(1)
        np.testing.assert_allclose(pb.step_dynamics(s1, np.array([1.0, 0.0]), np.zeros(1)), [1.0, -0.3])
        z = pb.LtiSystem(sp.csr_matrix((2, 2)), sp.csr_matrix((2, 1)), s1.partition, s1.graph)
        assert np.array_equal(pb.step_dynamics(z, np.array([1.0, 2.0]), np.zeros(1)), [0.0, 0.0])
