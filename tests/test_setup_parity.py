"""Host-side setup vs the reference's own objects (golden fixtures made by
tests/golden/make_golden.py from the reference): dynamics operator, layout
tables, column operators, row costs, plant CSR -- all bit for bit."""

import numpy as np
import pytest

import paper_2103_14990_b200 as pb
from conftest import chain_bundle, golden

SETUPS = ["setup_n3_t3_d1", "setup_n4_t3_d1", "setup_n6_t4_d2", "setup_n3_t3_d2"]


@pytest.mark.parametrize("name", SETUPS)
def test_dynamics_operator_bitwise(name):
    g = golden(name)
    n, d, t = (int(v) for v in g["config"])
    b = chain_bundle(n, t, d)
    z = b["operator"].z
    assert np.array_equal(z.indptr, g["z_indptr"])
    assert np.array_equal(z.indices, g["z_indices"])
    assert np.array_equal(z.data, g["z_data"])


@pytest.mark.parametrize("name", SETUPS)
def test_layout_tables_bitwise(name):
    g = golden(name)
    n, d, t = (int(v) for v in g["config"])
    tab = chain_bundle(n, t, d)["tables"]
    for key in ("rs", "cs", "row_len", "col_len", "col_slot_in_row", "c2r_flat", "r2c_flat",
                "elem_flat_col", "owner_col"):
        assert np.array_equal(getattr(tab, key), g["tab_" + key]), key


@pytest.mark.parametrize("name", SETUPS)
def test_column_operators_bitwise(name):
    """Class-deduplicated setup reproduces every per-column projector of the
    reference (sls_core.py:253-289) exactly."""
    g = golden(name)
    n, d, t = (int(v) for v in g["config"])
    cs = chain_bundle(n, t, d)["col_solvers"]
    for c, pre in enumerate(cs):
        assert np.array_equal(pre.g, g[f"col{c}_g"])
        assert np.array_equal(pre.rhs, g[f"col{c}_rhs"])
        assert np.array_equal(pre.projector, g[f"col{c}_P"])
        assert np.array_equal(pre.constraint_rows, g[f"col{c}_rows"])


@pytest.mark.parametrize("name", SETUPS)
def test_row_costs_and_plant(name):
    g = golden(name)
    n, d, t = (int(v) for v in g["config"])
    b = chain_bundle(n, t, d)
    w, lo, hi = b["spec"].row_arrays()
    assert np.array_equal(w, g["row_w"]) and np.array_equal(lo, g["row_lo"]) \
        and np.array_equal(hi, g["row_hi"])
    metas = pb.row_index_map(b["system"].partition, t, b["spec"])
    assert [m.weight for m in metas] == list(g["row_w"])
    a = b["system"].a
    assert np.array_equal(a.indptr, g["a_indptr"]) and np.array_equal(a.indices, g["a_indices"]) \
        and np.array_equal(a.data, g["a_data"])


@pytest.mark.parametrize("name", ["c1_loop_seed1", "c1_loop_seed2", "c2_loop_seed1", "d1_loop_n30"])
def test_initial_state_sampler_bitwise(name):
    g = golden(name)
    n, d, t, t_sim, seed = (int(v) for v in g["config"])
    system = pb.build_chain_network(n)
    x0 = pb.sample_initial_state(system.partition, np.random.default_rng(seed))
    assert np.array_equal(x0, g["x0"])


def test_class_dedup_counts():
    """SURVEY §0 finding 2: 2(d+1)+1 classes on the chain whatever N is."""
    for n in (20, 40, 80):
        b = chain_bundle(n, 10, 3)
        assert len(b["classes"].classes) == 9
    b = chain_bundle(30, 5, 1)
    assert len(b["classes"].classes) == 5


def test_locality_infeasible_d0():
    system = pb.build_chain_network(2)
    mask = pb.build_locality_mask(system, 0, 3)
    op = pb.build_dynamics_operator(system, 3)
    with pytest.raises(pb.LocalityInfeasible) as exc:
        pb.precompute_column_solvers(op, mask)
    assert exc.value.column >= 0


def test_projector_feasible_and_matches_pinv(rng):
    import scipy.linalg as sla
    b = chain_bundle(4, 3, 1)
    for pre in b["col_solvers"]:
        k = rng.standard_normal(pre.support.size)
        psi = k + pre.projector @ (pre.rhs - pre.g @ k)
        assert np.max(np.abs(pre.g @ psi - pre.rhs)) <= 1e-10
        ref = k - sla.pinv(pre.g) @ (pre.g @ k - pre.rhs)
        np.testing.assert_allclose(psi, ref, atol=1e-10)


def test_null_space_form_equals_projector(rng):
    """The fast path's Ψ = q + N Nᵀ k equals k + P(rhs - g k) (admm.py:186)."""
    b = chain_bundle(12, 6, 2)
    cc = b["classes"]
    for c, pre in enumerate(b["col_solvers"]):
        cl = cc.classes[cc.col_class[c]]
        k = rng.standard_normal(pre.support.size)
        ref = k + pre.projector @ (pre.rhs - pre.g @ k)
        fast = cc.particular(c) + cl.null @ (cl.null.T @ k)
        np.testing.assert_allclose(fast, ref, rtol=0, atol=1e-12)


@pytest.mark.parametrize("case", ["chain30", "chain_r2", "chain_two_inputs", "random_graph", "grid"])
def test_structural_builder_equals_reference_builder(case):
    """build_column_classes_structural (fingerprints + window extraction, used
    by the device session at scale) yields the same operators, bit for bit,
    as the reference-faithful per-support-set builder."""
    from conftest import random_graph_system
    from paper_2103_14990_b200 import sls_core as sc
    if case == "chain30":
        system, t, d = pb.build_chain_network(30), 10, 3
    elif case == "chain_r2":
        system, t, d = pb.build_chain_network(12, 2), 4, 2
    elif case == "chain_two_inputs":
        system, t, d = pb.build_chain_network(10, 1, True), 5, 2
    elif case == "grid":
        from conftest import grid_network
        system, t, d = grid_network(6, 7), 4, 2
    else:
        system, t, d = random_graph_system(9, np.random.default_rng(11)), 3, 2
    mask = pb.build_locality_mask(system, d, t)
    a = sc.build_column_classes(pb.build_dynamics_operator(system, t), mask)
    b = sc.build_column_classes_structural(system, t, mask)
    assert len(a.classes) == len(b.classes)
    for c in range(mask.n_cols):
        ca, cb = a.classes[a.col_class[c]], b.classes[b.col_class[c]]
        assert np.array_equal(ca.g, cb.g) and np.array_equal(ca.projector, cb.projector)
        assert np.array_equal(ca.null, cb.null)
        assert np.array_equal(a.reduced_rhs(c), b.reduced_rhs(c))


def test_structural_builder_scales():
    import time
    from paper_2103_14990_b200 import sls_core as sc
    system = pb.build_chain_network(100000)
    mask = pb.build_locality_mask(system, 3, 10)
    t0 = time.perf_counter()
    cc = sc.build_column_classes_structural(system, 10, mask)
    assert time.perf_counter() - t0 < 60
    assert len(cc.classes) == 9 and cc.col_class.size == 200000
