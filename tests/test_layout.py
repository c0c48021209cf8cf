"""Device layout maps, checked on CPU with a numpy emulation of the kernel's
data flow (tests/layout_emulator.py): in exact mode the emulator walks the
internal block layout exactly as csrc/dlmpc.cu does and must reproduce the
oracle's iterates bit for bit; this pins every index table (ball offsets,
row-support descriptors, reference<->internal permutations, generic
non-contiguous supports) before any GPU runs."""

import numpy as np
import pytest

import paper_2103_14990_b200 as pb
from paper_2103_14990_b200.devlayout import DeviceLayout, _ld_frag
from conftest import chain_bundle, random_graph_system
from layout_emulator import LayoutEmulator
from oracle import admm_ref


def _bundle_from_system(system, t, d, bounded=True):
    spec = pb.make_benchmark_spec(system, t, bounded=bounded)
    mask = pb.build_locality_mask(system, d, t)
    tables = pb.LayoutTables(mask)
    op = pb.build_dynamics_operator(system, t)
    classes = pb.build_column_classes(op, mask)
    return {"system": system, "spec": spec, "mask": mask, "tables": tables,
            "classes": classes, "col_solvers": pb.precompute_column_solvers(op, mask, classes)}


def _compare(b, x0, exact, iters=8):
    L = DeviceLayout(b["system"], b["spec"], b["mask"], b["classes"], exact=exact)
    tb = b["tables"]
    orc = admm_ref.OracleSolver(tb, b["col_solvers"], b["spec"].rho)
    w, lo, hi = b["spec"].row_arrays()
    orc.row_data, _ = admm_ref.row_data_for(x0, tb, w, lo, hi)
    em = LayoutEmulator(L)
    em.set_x(x0)
    cg, rg = L.column_gather(tb), L.row_gather(tb)
    cgs, rgs = np.where(cg >= 0, cg, 0), np.where(rg >= 0, rg, 0)
    for it in range(iters):
        r_ref = orc.iterate()
        r_em = em.iterate()
        psi_c = np.where(cg >= 0, em.psi[cgs], 0.0)
        lam_r = np.where(rg >= 0, em.lam[rgs], 0.0)
        phi_r = np.where(rg >= 0, em.phi[rgs], 0.0)
        prev_c = np.where(cg >= 0, em.psi_prev[cgs], 0.0)
        if exact:
            assert r_em == r_ref, it
            assert np.array_equal(psi_c, orc.psi_c), it
            assert np.array_equal(lam_r, orc.lam_r), it
            assert np.array_equal(phi_r, orc.phi_r), it
            assert np.array_equal(prev_c, orc.psi_prev_c), it
        else:
            assert np.allclose(r_em, r_ref, rtol=1e-9, atol=1e-13)
            assert np.max(np.abs(psi_c - orc.psi_c)) <= 1e-11
    return L


@pytest.mark.parametrize("exact", [True, False])
@pytest.mark.parametrize("n,t,d", [(10, 5, 2), (6, 4, 1), (3, 3, 2), (12, 3, 3)])
def test_chain_layout_emulation(n, t, d, exact):
    b = chain_bundle(n, t, d)
    x0 = pb.sample_initial_state(b["system"].partition, np.random.default_rng(n + d))
    L = _compare(b, x0, exact)
    assert L.contiguous


@pytest.mark.parametrize("exact", [True, False])
def test_generic_graph_layout_emulation(exact):
    rng = np.random.default_rng(5)
    system = random_graph_system(7, rng)
    b = _bundle_from_system(system, 3, 2)
    x0 = rng.uniform(-0.5, 1.0, system.n_states)
    L = _compare(b, x0, exact, iters=6)
    assert not L.contiguous


@pytest.mark.parametrize("exact", [True, False])
def test_two_inputs_and_radius2(exact):
    b = chain_bundle(8, 4, 2, two_inputs=True)
    x0 = pb.sample_initial_state(b["system"].partition, np.random.default_rng(3))
    _compare(b, x0, exact, iters=5)
    b = chain_bundle(9, 4, 2, coupling_radius=2)
    x0 = pb.sample_initial_state(b["system"].partition, np.random.default_rng(4))
    _compare(b, x0, exact, iters=5)


def test_padding_and_strides():
    b = chain_bundle(20, 10, 3)
    L = DeviceLayout(b["system"], b["spec"], b["mask"], b["classes"])
    assert L.s_pad % 4 == 0 and L.s_pad >= b["mask"].d_col
    assert all(ld % 16 in (4, 12) for ld in L.class_ldn)
    assert _ld_frag(48) == 52 and _ld_frag(8) == 12 and _ld_frag(56) == 60
    # longest-vector padding: interior class is 203 wide (SURVEY key shapes)
    interior = int(np.bincount(L.col_class).argmax())
    assert int(L.class_s[interior]) == 203 and int(L.class_n0[interior]) == 47
    assert int(L.class_m[interior]) == 156
    # the null-space blocks are zero outside [s, n0]
    for k in range(L.n_classes):
        blk = L.null_pool[L.class_null_off[k]:L.class_null_off[k + 1]].reshape(-1, L.class_ldn[k])
        assert np.all(blk[L.class_s[k]:] == 0) and np.all(blk[:, L.class_n0[k]:] == 0)
    # tiles cover every column exactly once, grouped by class
    seen = np.sort(np.concatenate([L.tile_colv[f:f + c] for f, c in zip(L.tile_first, L.tile_count)]))
    assert np.array_equal(seen, np.arange(L.n_cols))
    for k, f, c in zip(L.tile_class, L.tile_first, L.tile_count):
        assert np.all(L.col_class[L.tile_colv[f:f + c]] == k)


def test_row_support_descriptor_is_ascending():
    b = chain_bundle(9, 4, 2)
    L = DeviceLayout(b["system"], b["spec"], b["mask"], b["classes"])
    tb = b["tables"]
    for i in range(L.n_sub):
        cols = L.supp_col[i, :L.supp_len[i]]
        assert np.all(np.diff(cols) > 0)
        r_ref = L.int_to_ref[L.row_start[i]]
        assert np.array_equal(cols, tb.rs[r_ref, :tb.row_len[r_ref]])


def test_first_bad_row_matches_reference_scan():
    b = chain_bundle(4, 3, 1)
    spec = b["spec"]
    spec.state_lo[0, 1] = 0.5
    spec.state_hi[0, 1] = 1.0
    L = DeviceLayout(b["system"], spec, b["mask"], b["classes"])
    with pytest.raises(pb.RowInfeasible) as exc:
        pb.precompute_row_data(np.zeros(8), spec, b["tables"])
    assert int(L.sub_first_bad[L.sub_first_bad >= 0].min()) == exc.value.row
