"""Fused MPC-step transitions (patch mode with the per-CTA Φ cache,
`fused_transition` in dlmpc_device.cuh): each CTA computes the control, the
plant step and the next step's Φ cache for its own window, with no grid
barrier between steps. Checked bit for bit against the grid-barrier
transition (DLMPC_FUSE_STEPS=0 at session creation), against the oracle, and
on the RowInfeasible path that the fused loop defers to the next step's
first iteration barrier."""
import os

import numpy as np
import pytest

import paper_2103_14990_b200 as pb
from conftest import chain_bundle
from oracle import admm_ref

pytestmark = pytest.mark.gpu

FAST = "b200"


def _session(system, spec, mask, fuse, variant=FAST):
    old = os.environ.pop("DLMPC_FUSE_STEPS", None)
    try:
        # on by default only for the register-blocked GEMV plans (C2); forced
        # here so every plan family is checked
        os.environ["DLMPC_FUSE_STEPS"] = "1" if fuse else "0"
        return pb.DlmpcSession(system, spec, mask, variant)
    finally:
        os.environ.pop("DLMPC_FUSE_STEPS", None)
        if old is not None:
            os.environ["DLMPC_FUSE_STEPS"] = old


@pytest.mark.parametrize("n,d,t,eps,max_iters,t_sim", [
    (100, 3, 10, 1e-4, 5000, 20),    # C2, the bench workload
    (100, 3, 10, 1e-4, 5000, 150),   # a long loop: the residual regions and RowInfeasible slots wrap many times
    (12, 2, 4, 1e-4, 5000, 9),       # fewer units than CTAs (idle CTAs on the split barrier)
    (40, 1, 3, 1e6, 1, 7),           # one iteration per step: the max_iters stop test path
    (300, 2, 5, 1e-4, 5000, 6),      # two subsystems per unit
])
def test_fused_transition_bitwise_equal_to_grid_barrier(n, d, t, eps, max_iters, t_sim):
    system = pb.build_chain_network(n)
    spec = pb.make_benchmark_spec(system, t, eps=eps, max_iters=max_iters)
    mask = pb.build_locality_mask(system, d, t)
    a = _session(system, spec, mask, False)
    b = _session(system, spec, mask, True)
    try:
        assert a.device.info()["fuse_steps"] == 0
        assert b.device.info()["fuse_steps"] == 1, b.device.info()
        for seed in (1, 2, 3):
            x0 = pb.sample_initial_state(system.partition, np.random.default_rng(seed))
            ta, _ = a.simulate(x0, t_sim)
            tb, _ = b.simulate(x0, t_sim)
            assert list(ta.step_iterations) == list(tb.step_iterations)
            assert np.array_equal(ta.states, tb.states)
            assert np.array_equal(ta.inputs, tb.inputs)
            # a second launch on the same session (the barrier counter and the
            # residual regions continue) gives the same trajectory
            tb2, _ = b.simulate(x0, t_sim)
            assert np.array_equal(tb2.states, tb.states)
    finally:
        a.close(); b.close()


def test_fused_transition_against_oracle():
    b = chain_bundle(24, 5, 2)
    x0 = pb.sample_initial_state(b["system"].partition, np.random.default_rng(5))
    ref = admm_ref.simulate(b["system"], b["spec"], b["tables"], b["col_solvers"], x0, 8)
    sess = _session(b["system"], b["spec"], b["mask"], True)
    try:
        assert sess.device.info()["fuse_steps"] == 1
        traj, _ = sess.simulate(x0, 8)
    finally:
        sess.close()
    assert list(traj.step_iterations) == ref["step_iterations"]
    scale = np.max(np.abs(ref["states"]))
    assert np.max(np.abs(traj.states - ref["states"])) <= 1e-12 * scale


def _dead_plant(n, d):
    """Chain plant whose A and B rows vanish on subsystem 0's d-hop support:
    x+ is zero there whatever the control, so the row data of step 1 is
    infeasible for a bound that excludes 0 (sls_core.py:346-348)."""
    base = pb.build_chain_network(n)
    a = base.a.tolil()
    bm = base.b.tolil()
    for r in range(2 * (d + 1)):
        a[r, :] = 0.0
        bm[r, :] = 0.0
    return pb.LtiSystem(a.tocsr(), bm.tocsr(), base.partition, base.graph)


@pytest.mark.parametrize("variant", ["b200-exact", FAST])
def test_row_infeasible_at_a_later_step(variant):
    n, t, d = 8, 3, 1
    system = _dead_plant(n, d)
    spec = pb.make_benchmark_spec(system, t)
    spec.state_lo[1, 0] = 0.5    # state 1 at t = 0: Φx(0) = I makes it x0[1]
    spec.state_hi[1, 0] = 1.0
    mask = pb.build_locality_mask(system, d, t)
    tables = pb.LayoutTables(mask)
    op = pb.build_dynamics_operator(system, t)
    cs = pb.precompute_column_solvers(op, mask, pb.build_column_classes(op, mask))
    x0 = pb.sample_initial_state(system.partition, np.random.default_rng(3))
    x0[1] = 0.7
    ref = admm_ref.simulate(system, spec, tables, cs, x0, 4)
    assert ref["status"] == "row_infeasible" and ref["at"][0] == 1, (ref["status"], ref["at"])
    if variant == FAST:
        sess = _session(system, spec, mask, True, variant)
        try:
            assert sess.device.info()["fuse_steps"] == 1
        finally:
            sess.close()
    with pytest.raises(pb.RowInfeasible) as exc:
        pb.dlmpc_simulate(system, spec, mask, x0, 4, variant)
    assert exc.value.step == 1
    assert exc.value.row == ref["at"][1]


@pytest.mark.parametrize("n,d,t,expect", [
    (100, 3, 10, {"grid": 100, "cache_phi": 1, "fuse_steps": 1, "rb_gemv": 1, "pairs": 0}),   # C2
    (1000, 3, 10, {"grid": 148, "cache_phi": 1, "fuse_steps": 0, "rb_gemv": 0}),
    (1000, 6, 30, {"cache_phi": 2, "pairs": 1}),                                               # partial Φ cache
])
def test_plan_choices_of_the_timed_configs(n, d, t, expect):
    """The kernel plans the bench and the C4 sweep time: C2
    launches only the CTAs that own a unit and fuses its step transitions;
    the largest C4 cell takes the partial Φ cache and K-split pairs."""
    system = pb.build_chain_network(n)
    spec = pb.make_benchmark_spec(system, t)
    mask = pb.build_locality_mask(system, d, t)
    sess = pb.DlmpcSession(system, spec, mask, FAST)
    try:
        info = sess.device.info()
    finally:
        sess.close()
    for k, v in expect.items():
        assert info[k] == v, (k, info)


@pytest.mark.parametrize("n,d,t", [(300, 2, 5), (1000, 3, 10), (1000, 4, 20)])
def test_partial_phi_cache_matches_full_cache(n, d, t):
    """The partial Φ cache (kVarPcache kernels, with the L1-prefetched chunk;
    taken by the largest C4 cells) forced on small plans: the same iteration
    counts as the full-cache plan and the oracle, states within the fast
    path's tolerance."""
    system = pb.build_chain_network(n)
    spec = pb.make_benchmark_spec(system, t)
    mask = pb.build_locality_mask(system, d, t)
    old = os.environ.get("DLMPC_PARTIAL_PHI")
    os.environ["DLMPC_PARTIAL_PHI"] = "2"
    try:
        os.environ["DLMPC_FUSE_STEPS"] = "0"
        part = pb.DlmpcSession(system, spec, mask, FAST)
    finally:
        os.environ.pop("DLMPC_FUSE_STEPS", None)
        if old is None:
            os.environ.pop("DLMPC_PARTIAL_PHI", None)
        else:
            os.environ["DLMPC_PARTIAL_PHI"] = old
    full = _session(system, spec, mask, False)
    try:
        info = part.device.info()
        if info["rb_gemv"]:
            pytest.skip("GEMV-pair plan (the partial cache is for the DMMA plans)")
        assert info["cache_phi"] == 2, info
        assert full.device.info()["cache_phi"] == 1
        for seed in (1, 2):
            x0 = pb.sample_initial_state(system.partition, np.random.default_rng(seed))
            ta, _ = full.simulate(x0, 4)
            tb, _ = part.simulate(x0, 4)
            assert list(ta.step_iterations) == list(tb.step_iterations)
            scale = np.max(np.abs(ta.states))
            assert np.max(np.abs(ta.states - tb.states)) <= 1e-12 * scale
    finally:
        part.close(); full.close()
