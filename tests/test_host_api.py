"""Host-side API behaviour (no GPU): plant/graph/mask builders against brute
force and the reference's unit-test goldens, spec validation, strategy
plugin, ledger, report, error types."""

import math

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.csgraph as csgraph

import paper_2103_14990_b200 as pb
from paper_2103_14990_b200.system_model import phi_row_owners


def chain_graph(n):
    return pb.SubsystemGraph.from_edges(n, [(i, i + 1) for i in range(n - 1)])


def all_pairs(graph):
    n = graph.node_count
    m = sp.lil_matrix((n, n))
    for i, nb in enumerate(graph.adjacency):
        for j in nb:
            m[i, j] = 1
    return csgraph.shortest_path(m.tocsr(), unweighted=True)


class TestGraph:
    def test_distances_match_brute_force(self, rng):
        for _ in range(8):
            n = int(rng.integers(2, 12))
            edges = [(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < 0.3]
            g = pb.SubsystemGraph.from_edges(n, edges)
            ref = all_pairs(g)
            for i in range(n):
                for j in range(n):
                    got = pb.graph_distance(g, i, j)
                    assert (math.isinf(ref[i, j]) and got == pb.UNREACHABLE) or got == ref[i, j]

    def test_balls_csr_matches_bfs(self, rng):
        g = pb.SubsystemGraph.from_edges(10, [(0, 3), (3, 7), (7, 9), (1, 2), (2, 5)])
        for r in range(4):
            ptr, idx = g.balls(r)
            for i in range(10):
                assert np.array_equal(idx[ptr[i]:ptr[i + 1]], g.ball(i, r))

    def test_validation(self):
        with pytest.raises(ValueError):
            pb.SubsystemGraph(2, (np.array([1], np.int32), np.array([], np.int32)))
        with pytest.raises(ValueError):
            pb.SubsystemPartition(((0, 2), (3, 4)), ((0, 1), (1, 2)))
        with pytest.raises(ValueError):
            pb.SubsystemPartition(((0, 0),), ((0, 0),))
        with pytest.raises(ValueError):
            pb.graph_distance(chain_graph(3), 0, 3)
        part = pb.SubsystemPartition.uniform(2, 1, 1)
        with pytest.raises(ValueError):
            pb.LtiSystem(sp.csr_matrix(np.array([[1.0, 0.5], [0.0, 1.0]])), sp.csr_matrix(np.eye(2)),
                         part, pb.SubsystemGraph.from_edges(2, []))


class TestChainAndMask:
    def test_chain_blocks(self):
        a = pb.build_chain_network(3).a.toarray()
        np.testing.assert_array_equal(a[2:4, 2:4], [[1.0, 0.1], [-0.3, 0.7]])
        np.testing.assert_array_equal(a[2:4, 0:2], [[0.0, 0.0], [0.1, 0.1]])
        np.testing.assert_array_equal(a[0:2, 4:6], np.zeros((2, 2)))
        with pytest.raises(ValueError):
            pb.build_chain_network(0)

    def test_mask_against_brute_force(self):
        system = pb.build_chain_network(5)
        for d in range(4):
            mask = pb.build_locality_mask(system, d, 3)
            dist = all_pairs(system.graph)
            owners_r = phi_row_owners(system.partition, 3)
            owners_c = system.partition.state_owner()
            want = {(r, c) for r in range(mask.n_rows) for c in range(mask.n_cols)
                    if dist[owners_r[r], owners_c[c]] <= d}
            got = {(r, int(c)) for r, s in enumerate(mask.row_supports) for c in s}
            assert got == want
            got_c = {(int(r), c) for c, s in enumerate(mask.col_supports) for r in s}
            assert got_c == want
            assert mask.n_entries == len(want)

    def test_lemma1(self):
        assert pb.lemma1_bounds(2, 2, 2, 5) == (14, 126)
        assert pb.lemma1_bounds(1, 2, 0, 2) == (1, 3)
        for n in (3, 10):
            system = pb.build_chain_network(n)
            for d in range(4):
                mask = pb.build_locality_mask(system, d, 5)
                rb, cb = pb.lemma1_bounds(2, 2, d, 5)
                assert mask.d_row <= rb and mask.d_col <= cb

    def test_closed_forms_survey(self):
        """D_row = 2(2d+1), D_col = (2d+1)(3T-1), nnz formula."""
        for n, d, t in ((100, 3, 10), (40, 2, 5), (30, 1, 7)):
            mask = pb.build_locality_mask(pb.build_chain_network(n), d, t)
            assert mask.d_row == 2 * (2 * d + 1)
            assert mask.d_col == (2 * d + 1) * (3 * t - 1)
            assert mask.n_entries == 2 * (3 * t - 1) * ((2 * d + 1) * n - d * (d + 1))

    def test_compact_mask_scales(self):
        mask = pb.build_locality_mask(pb.build_chain_network(200000), 3, 10)
        assert mask.n_rows == 200000 * 29 and mask.d_col == 203
        assert mask._row_supports is None   # nothing per-row materialised

    def test_rejects_bad_arguments(self):
        system = pb.build_chain_network(2)
        with pytest.raises(ValueError):
            pb.build_locality_mask(system, -1, 3)
        with pytest.raises(ValueError):
            pb.build_locality_mask(system, 1, 1)


class TestSpecAndRows:
    def test_spec_validation(self):
        base = dict(horizon=3, state_weights=np.ones((2, 3)), input_weights=np.ones((1, 2)),
                    terminal_weights=np.ones(2), state_lo=np.full((2, 3), -np.inf),
                    state_hi=np.full((2, 3), np.inf), input_lo=np.full((1, 2), -np.inf),
                    input_hi=np.full((1, 2), np.inf))
        pb.ProblemSpec(**base)
        with pytest.raises(ValueError):
            pb.ProblemSpec(**{**base, "state_lo": np.full((2, 3), 2.0), "state_hi": np.full((2, 3), 1.0)})
        with pytest.raises(ValueError):
            pb.ProblemSpec(**base, rho=0.0)
        with pytest.raises(ValueError):
            pb.ProblemSpec(**{**base, "input_weights": -np.ones((1, 2))})

    def test_row_index_map_order(self):
        part = pb.SubsystemPartition.uniform(1, 2, 1)
        rows = pb.row_index_map(part, 3)
        assert [m.kind for m in rows] == ["state"] * 6 + ["input"] * 2
        assert [m.time for m in rows] == [0, 0, 1, 1, 2, 2, 0, 1]
        assert rows[0] == pb.RowMeta("state", 0, 0, 0)

    def test_row_arrays_match_row_metas(self):
        system = pb.build_chain_network(3)
        spec = pb.make_benchmark_spec(system, 4)
        metas = pb.row_index_map(system.partition, 4, spec)
        w, lo, hi = spec.row_arrays()
        for r, m in enumerate(metas):
            assert (m.weight, m.lo, m.hi) == (spec.row_weight(m.kind, m.signal, m.time),
                                              *spec.row_bounds(m.kind, m.signal, m.time))
            assert (w[r], lo[r], hi[r]) == (m.weight, m.lo, m.hi)

    def test_row_data_support_restriction(self):
        part = pb.SubsystemPartition(((0, 1), (1, 2), (2, 3)), ((0, 0), (0, 0), (0, 0)))
        graph = pb.SubsystemGraph.from_edges(3, [(0, 2)])
        system = pb.LtiSystem(sp.csr_matrix(np.eye(3) * 0.5), sp.csr_matrix((3, 0)), part, graph)
        mask = pb.build_locality_mask(system, 1, 2)
        np.testing.assert_array_equal(mask.row_supports[0], [0, 2])
        tables = pb.LayoutTables(mask)
        spec = pb.make_benchmark_spec(system, 2, bounded=False)
        rd = pb.precompute_row_data(np.array([3.0, 9.0, 4.0]), spec, tables)
        row = rd.row(0)
        np.testing.assert_array_equal(row.a, [3.0, 4.0])
        assert row.a_dot_a == 25.0

    def test_row_infeasible(self):
        system = pb.build_chain_network(2)
        spec = pb.make_benchmark_spec(system, 3)
        spec.state_lo[0, 1] = 0.5
        spec.state_hi[0, 1] = 1.0
        tables = pb.LayoutTables(pb.build_locality_mask(system, 1, 3))
        with pytest.raises(pb.RowInfeasible) as exc:
            pb.precompute_row_data(np.zeros(4), spec, tables)
        assert exc.value.row == 4   # state 0 at time 1: row 1*n_x + 0

    def test_ascending_dot(self, rng):
        x, y = rng.standard_normal((7, 5)), rng.standard_normal((7, 5))
        np.testing.assert_allclose(pb.ascending_dot(x, y), (x * y).sum(axis=1), rtol=1e-15)

    def test_layout_round_trip_no_leak(self, rng):
        tables = pb.LayoutTables(pb.build_locality_mask(pb.build_chain_network(4), 1, 3))
        t = pb.PhiTriple(tables)
        t.phi_r[:] = np.where(tables.row_valid, rng.standard_normal(tables.rs.shape), 0.0)
        t.exchange_phi_row_to_col()
        np.testing.assert_array_equal(t._dense_from_row(t.phi_r), t._dense_from_col(t.phi_c))
        t.psi_c[:] = t.phi_c
        t.lam_c[:] = 0.25 * t.phi_c
        t.exchange_psi_lam_col_to_row()
        np.testing.assert_array_equal(t.psi_r, t.phi_r)
        assert t.padding_leak() == 0.0
        assert np.all(tables.owner_col == tables.rs[:, 0])


class TestStrategyPlugin:
    def test_variants(self):
        # the production variants plus the reference's five names (strategies.py:46)
        assert pb.STRATEGY_NAMES == ("sequential", "naive", "padded", "fused", "patch-local")
        assert pb.VARIANTS == ("b200", "b200-exact") + pb.STRATEGY_NAMES
        assert pb.ExecStrategy().variant == "b200"
        assert pb.ExecStrategy("b200-exact").exact and not pb.ExecStrategy("b200").exact
        for v in ("sequential", "naive", "padded", "fused", "patch-local"):
            s = pb.ExecStrategy(v, worker_count=4)
            assert s.exact                     # reference arithmetic: bit-identical iterates
            assert s.staged == (v != "sequential")
        with pytest.raises(ValueError):
            pb.ExecStrategy("gpu")
        with pytest.raises(ValueError):
            pb.ExecStrategy("b200", 0)

    def test_reference_ledger_constants(self):
        """strategies.py:49-55: (host syncs, kernel launches, flag reads)."""
        want = {"sequential": (0, 0, 0), "naive": (4, 4, 0), "padded": (4, 4, 0), "fused": (1, 2, 1),
                "patch-local": (0, 1, 1)}
        for v, c in want.items():
            led = pb.SyncLedger.for_variant(v)
            assert (led.host_syncs_per_iter, led.kernel_launches_per_iter, led.flag_reads_per_iter) == c

    def test_patches(self):
        """build_patches / patch_duplication (strategies.py:147-157): one patch
        per column holding its support rows; duplication = nnz - n_rows."""
        mask = pb.build_locality_mask(pb.build_chain_network(6), 2, 4)
        tables = pb.LayoutTables(mask)
        patches = pb.build_patches(tables)
        assert len(patches) == tables.n_cols
        for p in patches:
            assert np.array_equal(p.member_rows, tables.cs[p.column, :tables.col_len[p.column]])
        assert pb.patch_duplication(patches) == int(tables.col_len.sum()) - tables.n_rows
        sizes = pb.prepare_work_items(pb.ExecStrategy("padded"), tables, pb.SyncLedger.for_variant("padded"))
        assert sizes == (tables.d_row, tables.d_col)

    def test_ledger(self):
        led = pb.SyncLedger.for_variant("b200")
        assert (led.host_syncs_per_iter, led.kernel_launches_per_iter, led.flag_reads_per_iter) == (0, 0, 0)
        led.record_launch(37, 1.5)
        assert led.counts_consistent() and led.iterations == 37 and led.solve_launches == 1
        assert led.as_dict()["device_time_ms"] == 1.5

    def test_reduce_convergence(self, rng):
        pri, dual = rng.uniform(0, 1, 10), rng.uniform(0, 1, 10)
        perm = rng.permutation(10)
        assert pb.reduce_convergence(pri, dual, 1e-4, 1e-4) == \
            pb.reduce_convergence(pri[perm], dual[perm], 1e-4, 1e-4)
        assert pb.reduce_convergence(np.zeros(3), np.zeros(3), 1e-4, 1e-4)[2]

    def test_report_metric(self):
        rep = pb.RunReport({}, {"setup": 1.0, "precompute_global": 2.0, "precompute_per_step": 0.0,
                                "optimize": 40.0, "dynamics": 0.0}, [3, 5], pb.SyncLedger.for_variant("b200"),
                           1.0, True, 50.0)
        assert rep.mean_per_mpc_step_ms() == 20.0 and rep.iters_total == 8
        assert set(rep.as_dict()) >= {"mean_per_mpc_step_ms", "per_step_iters", "ledger"}


class TestErrors:
    def test_attributes(self):
        e = pb.NotConverged([(1.0, 2.0)], step=3)
        assert e.step == 3 and e.residual_history == [(1.0, 2.0)]
        assert pb.RowInfeasible(5).row == 5
        li = pb.LocalityInfeasible(2, 0.5)
        assert (li.column, li.residual) == (2, 0.5)
        assert pb.ConfigError("x", 4).line_no == 4
        for cls in (pb.NotConverged, pb.RowInfeasible, pb.LocalityInfeasible, pb.DeviceError):
            assert issubclass(cls, pb.LocalityMpcError)

    def test_simulate_argument_errors(self):
        system = pb.build_chain_network(2)
        spec = pb.make_benchmark_spec(system, 3)
        mask = pb.build_locality_mask(system, 1, 3)
        with pytest.raises(ValueError):
            pb.dlmpc_simulate(system, spec, mask, np.zeros(3), 2)
        with pytest.raises(ValueError):
            pb.dlmpc_simulate(system, spec, mask, np.zeros(4), 0)
