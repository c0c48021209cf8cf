"""Pin the oracle (oracle/admm_ref.py) against the reference's own outputs.

The fixtures were produced by running the reference (tests/golden/
make_golden.py); the oracle must reproduce them bit for bit, plus the known
answers of SURVEY.md Appendix B. Only then is it trusted as the checker of
the device path.
"""

import numpy as np
import pytest

import paper_2103_14990_b200 as pb
from conftest import chain_bundle, golden
from oracle import admm_ref

TRIPLE = ("phi_r", "psi_r", "lam_r", "phi_c", "psi_c", "lam_c", "psi_prev_c")


def test_c1_step0_known_answers():
    g = golden("c1_step0")
    b = chain_bundle(10, 5, 2)
    s = admm_ref.OracleSolver(b["tables"], b["col_solvers"], b["spec"].rho)
    w, lo, hi = b["spec"].row_arrays()
    rd, bad = admm_ref.row_data_for(g["x0"], b["tables"], w, lo, hi)
    assert bad == -1
    n, hist, ok = s.solve(rd, 5000, 1e-4, 1e-4)
    assert ok and n == 37 == int(g["iterations"])
    assert np.array_equal(np.array(hist), g["history"])
    # SURVEY Appendix B values
    assert hist[0] == (1.0, 1.0)
    assert hist[1] == (1.0, 0.014088949999966294)
    assert hist[36] == (9.499395713641334e-05, 1.2627433913503516e-06)
    for name in TRIPLE:
        assert np.array_equal(getattr(s, name), g[name]), name
    u = admm_ref.extract_control(s.phi_r, b["tables"], g["x0"], [20 * 5 + k for k in range(10)])
    assert np.array_equal(u, g["u0"])
    assert u[0] == -0.36628715756880204
    assert float(np.abs(s.phi_r).sum()) == pytest.approx(107.63505042622579, rel=1e-14)


@pytest.mark.parametrize("name", ["c1_loop_seed1", "c1_loop_seed2", "c1_loop_seed3",
                                  "d1_loop_n30", "d4_loop_n20", "unbounded_loop_n8"])
def test_closed_loops_bitwise(name):
    g = golden(name)
    n, d, t, t_sim, seed = (int(v) for v in g["config"])
    b = chain_bundle(n, t, d, bounded=bool(g["bounded"]), eps=float(g["eps"]))
    res = admm_ref.simulate(b["system"], b["spec"], b["tables"], b["col_solvers"], g["x0"], t_sim)
    assert res["status"] == "ok"
    assert res["step_iterations"] == list(g["step_iters"])
    assert np.array_equal(res["states"], g["states"])
    assert np.array_equal(res["inputs"], g["inputs"])


def test_c1_iteration_list_appendix_b():
    g = golden("c1_loop_seed1")
    assert list(g["step_iters"]) == [37, 25, 20, 18, 14, 12, 10, 8, 7, 6, 6, 5, 4, 4, 4, 3, 3, 3, 3, 3]
    assert float(g["cost"]) == pytest.approx(12.27316024, abs=1e-8)


def test_c2_iteration_list_appendix_b():
    g = golden("c2_loop_seed1")
    assert list(g["step_iters"]) == [72, 53, 45, 38, 30, 23, 18, 14, 11, 9, 7, 6, 5, 4, 4, 3, 3, 3, 3, 2]
    assert float(g["cost"]) == pytest.approx(163.4041939, abs=1e-7)


@pytest.mark.slow
def test_c2_closed_loop_bitwise():
    g = golden("c2_loop_seed1")
    b = chain_bundle(100, 10, 3)
    res = admm_ref.simulate(b["system"], b["spec"], b["tables"], b["col_solvers"], g["x0"], 20,
                            workers=4)
    assert res["step_iterations"] == list(g["step_iters"])
    assert np.array_equal(res["states"], g["states"])


@pytest.mark.parametrize("name", ["trace_n6_d1_t4", "trace_n5_d2_t4"])
def test_iteration_traces_bitwise(name):
    """Iteration by iteration (the reference's schedule-equivalence harness,
    test_strategies.py:187-208)."""
    g = golden(name)
    n, d, t, seed, iters = (int(v) for v in g["config"])
    b = chain_bundle(n, t, d)
    s = admm_ref.OracleSolver(b["tables"], b["col_solvers"], b["spec"].rho)
    w, lo, hi = b["spec"].row_arrays()
    s.row_data, _ = admm_ref.row_data_for(g["x"], b["tables"], w, lo, hi)
    for k in range(iters):
        assert s.iterate() == tuple(g["residuals"][k]), k
        if f"it{k}_psi_c" in g:
            for name_ in TRIPLE:
                assert np.array_equal(getattr(s, name_), g[f"it{k}_{name_}"]), (k, name_)


def test_worker_count_independence():
    b = chain_bundle(10, 5, 2)
    g = golden("c1_loop_seed1")
    r1 = admm_ref.simulate(b["system"], b["spec"], b["tables"], b["col_solvers"], g["x0"], 3, workers=1)
    r4 = admm_ref.simulate(b["system"], b["spec"], b["tables"], b["col_solvers"], g["x0"], 3, workers=4)
    assert np.array_equal(r1["states"], r4["states"])


def test_not_converged_history():
    g = golden("not_converged_n3")
    b = chain_bundle(3, 3, 1, eps=1e-12, max_iters=2)
    s = admm_ref.OracleSolver(b["tables"], b["col_solvers"], 1.0)
    w, lo, hi = b["spec"].row_arrays()
    rd, _ = admm_ref.row_data_for(g["x"], b["tables"], w, lo, hi)
    n, hist, ok = s.solve(rd, 2, 1e-12, 1e-12)
    assert not ok and n == 2
    assert np.array_equal(np.array(hist), g["history"])


def test_zero_state_loop():
    g = golden("zero_state_n3")
    b = chain_bundle(3, 3, 1)
    res = admm_ref.simulate(b["system"], b["spec"], b["tables"], b["col_solvers"], np.zeros(6), 5)
    assert res["step_iterations"] == list(g["step_iters"])
    assert np.array_equal(res["states"], g["states"])
    assert res["step_iterations"][-1] == 1


KKT_CASES = [(2, 3, 1), (3, 4, 2), (4, 3, 1), (4, 4, 2)]


@pytest.mark.parametrize("n,t,d", KKT_CASES)
def test_kkt_oracle_restatement_matches_reference(n, t, d):
    """oracle/kkt.py reproduces the reference's dense KKT closed loop."""
    from oracle import kkt
    g = golden("kkt_oracle")
    system = pb.build_chain_network(n)
    spec = pb.make_benchmark_spec(system, t, eps=1e-6, bounded=False)
    mask = pb.build_locality_mask(system, d, t)
    states, inputs = kkt.kkt_closed_loop(system, spec, mask, g[f"n{n}_t{t}_d{d}_x0"], 8)
    np.testing.assert_allclose(states, g[f"n{n}_t{t}_d{d}_states"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(inputs, g[f"n{n}_t{t}_d{d}_inputs"], rtol=1e-9, atol=1e-12)


def test_oracle_phi_rows_match_independent_minimiser():
    """The oracle's closed-form Φ row solve against scipy's bounded scalar
    minimiser (the reference's own independent check, test_admm.py:53-87):
    for y = φ·a the row objective is w·y² + (ρ/2)(y - c)²/‖a‖² on [lo, hi],
    and φ = v + (y - c)/‖a‖² · a."""
    from scipy.optimize import minimize_scalar
    g = golden("c1_step0")
    b = chain_bundle(10, 5, 2)
    s = admm_ref.OracleSolver(b["tables"], b["col_solvers"], b["spec"].rho)
    w, lo, hi = b["spec"].row_arrays()
    s.row_data, _ = admm_ref.row_data_for(g["x0"], b["tables"], w, lo, hi)
    for _ in range(3):
        s.iterate()
    v = s.psi_r - s.lam_r
    n = v.shape[0]
    s._phi(0, n)
    rd, rho = s.row_data, b["spec"].rho
    checked = 0
    for r in range(n):
        a, ada = rd.a_pad[r], rd.a_dot_a[r]
        if ada == 0.0:
            assert np.array_equal(s.phi_r[r], v[r])
            continue
        c = float(v[r] @ a)
        wr, l_, h_ = rd.weight[r], rd.lo[r], rd.hi[r]
        f = lambda y: wr * y * y + 0.5 * rho * (y - c) ** 2 / ada
        span = 10.0 * (abs(c) + 1.0)
        res = minimize_scalar(f, bounds=(max(l_, c - span), min(h_, c + span)), method="bounded",
                              options={"xatol": 1e-13})
        phi = v[r] + (res.x - c) / ada * a
        np.testing.assert_allclose(s.phi_r[r], phi, rtol=1e-6, atol=1e-7)   # Brent's accuracy
        checked += 1
    assert checked > 50


def test_sequential_schedule_restatement_bitwise():
    """The oracle's `sequential` schedule (one row / column per stage call,
    the reference's strategies.py:262-281, timed by bench.py as the 1-core
    "CPU ADMM" baseline) reproduces the reference's C1 closed loop bit for
    bit."""
    g = golden("c1_loop_seed1")
    b = chain_bundle(10, 5, 2)
    res = admm_ref.simulate(b["system"], b["spec"], b["tables"], b["col_solvers"], g["x0"], 20,
                            sequential=True)
    assert res["step_iterations"] == list(g["step_iters"])
    assert np.array_equal(res["states"], g["states"])
    assert np.array_equal(res["inputs"], g["inputs"])


@pytest.mark.parametrize("name", ["c3_n1000_step0", "c3_n3000_step0"])
def test_large_step0_bitwise_pins_the_class_shared_oracle(name):
    """The oracle with class-shared (broadcast) operators -- the form that
    generated the N=10^4 and C4 fixtures the reference cannot reach here
    (make_oracle_golden.py) -- reproduces the reference's own N=1000 and
    N=3000 step-0 solves bit for bit."""
    import os
    g = golden(name)
    n, d, t, t_sim, seed = (int(v) for v in g["config"])
    b = chain_bundle(n, t, d)
    res = admm_ref.simulate(b["system"], b["spec"], b["tables"], b["col_solvers"], g["x0"], t_sim,
                            workers=os.cpu_count() or 1)
    assert res["step_iterations"] == [int(v) for v in g["step_iters"]]
    assert np.array_equal(res["states"], g["states"])
    assert np.array_equal(res["inputs"], g["inputs"])
