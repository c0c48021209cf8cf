"""Drop-in solver API of the DLMPC hot path, executed on the B200.

Same entry points as `/root/reference/pkg/src/locality_mpc/admm.py`:
`AdmmWorkspace` (97-282), `AdmmState` (305-312), `admm_solve` (315-347),
`Trajectory` (372-378), `closed_loop_cost` (381-383) and `dlmpc_simulate`
(437-540). Every ADMM iteration, the per-step row data, the control
extraction and the plant step run inside the persistent CUDA kernel of
`csrc/dlmpc.cu` (through `device.DeviceSession`); this module only moves
arrays across the boundary and maps status codes to the reference's
exceptions. If the CUDA library or the GPU is missing, `DeviceError` is
raised: there is no CPU fallback.

Layouts: the device keeps ψ, λ in a single block column layout
(`devlayout.py`). `admm_solve` uploads the caller's `PhiTriple` (its column
layout is taken as authoritative: after any reference stage the two layouts
agree, sls_core.py:415-422), solves, and writes all seven triple arrays back
in the reference's padded layouts, so callers see exactly the reference's
in-place warm-start semantics (admm.py:320-322).
"""

from __future__ import annotations

import hashlib
import time
import weakref
from dataclasses import dataclass

import numpy as np

from .devlayout import DeviceLayout
from .device import DeviceSession, PSI, LAM, PSI_PREV, PHI
from .errors import NotConverged, RowInfeasible
from .sls_core import (ColumnClasses, LayoutTables, PhiTriple, ProblemSpec, RowData,
                       build_column_classes_structural)
from .strategies import ExecStrategy, Executor
from .system_model import LocalityMask, LtiSystem


@dataclass
class AdmmState:
    """Outcome of one consensus solve (reference admm.py:305-312)."""

    triple: PhiTriple
    iterations: int
    residual_history: list
    converged: bool


@dataclass
class Trajectory:
    """Closed-loop record (reference admm.py:372-378)."""

    states: np.ndarray        # (t_sim + 1, n_states)
    inputs: np.ndarray        # (t_sim, n_inputs)
    step_iterations: list


def closed_loop_cost(traj: Trajectory) -> float:
    """Sum of squared states and inputs (reference admm.py:381-383)."""
    return float(np.sum(traj.states ** 2) + np.sum(traj.inputs ** 2))


def _classes_of(col_solvers) -> ColumnClasses:
    if isinstance(col_solvers, ColumnClasses):
        return col_solvers
    cc = getattr(col_solvers, "classes", None)
    return cc if cc is not None else ColumnClasses.from_precomps(col_solvers)


@dataclass
class FixedPointReport:
    """Residuals of an independent audit of a solve (reference admm.py:386-414)."""

    dynamics_residual: float
    resolve_residual: float
    consensus_gap: float
    threshold: float

    @property
    def passed(self) -> bool:
        return (self.dynamics_residual <= self.threshold and self.resolve_residual <= self.threshold
                and self.consensus_gap <= self.threshold)

    def as_dict(self):
        return {"dynamics_residual": self.dynamics_residual, "resolve_residual": self.resolve_residual,
                "consensus_gap": self.consensus_gap, "threshold": self.threshold, "passed": self.passed}


def _x_of(row_data: RowData, tables: LayoutTables) -> np.ndarray:
    x = getattr(row_data, "x_tau", None)
    if x is not None:
        return np.asarray(x, dtype=np.float64)
    # every column appears in its own subsystem's rows: a_pad determines x
    x = np.zeros(tables.n_cols)
    x[tables.rs[tables.row_valid]] = row_data.a_pad[tables.row_valid]
    return x


class AdmmWorkspace:
    """Session binding of one triple to its device state (reference 97-130).

    The device session (problem upload, operators staged for the kernel) is
    built on first use per arithmetic flavour and reused across MPC steps;
    `set_row_data` swaps in the per-step operand as in the reference.
    """

    def __init__(self, triple: PhiTriple, col_solvers, spec: ProblemSpec,
                 patches=None, row_data: RowData | None = None, system: LtiSystem | None = None):
        self.triple = triple
        self.tables: LayoutTables = triple.tables
        self.col_solvers = col_solvers
        self.spec = spec
        self.rho = float(spec.rho)
        self.n_rows = self.tables.n_rows
        self.n_cols = self.tables.n_cols
        self.n_elems = self.tables.n_elems
        self.row_data = row_data
        self.patches = patches
        self.system = system
        self._sessions = {}
        self._maps = None
        self.last_device_ms = 0.0

    def set_row_data(self, row_data: RowData):
        self.row_data = row_data

    def session(self, exact: bool, device: int = 0) -> DeviceSession:
        key = (bool(exact), int(device))
        if key not in self._sessions:
            layout = DeviceLayout(self.system, self.spec, self.tables.mask,
                                  _classes_of(self.col_solvers), exact=exact)
            self._sessions[key] = DeviceSession(layout, device)
        return self._sessions[key]

    def _gathers(self, layout):
        if self._maps is None:
            self._maps = (layout.column_gather(self.tables), layout.row_gather(self.tables))
        return self._maps

    def upload_triple(self, sess: DeviceSession):
        cg, _ = self._gathers(sess.layout)
        valid = cg >= 0
        for which, arr in ((PSI, self.triple.psi_c), (LAM, self.triple.lam_c)):
            buf = np.zeros(sess.n_cell)
            buf[cg[valid]] = arr[valid]
            sess.put(which, buf)

    def download_triple(self, sess: DeviceSession):
        cg, rg = self._gathers(sess.layout)
        t = self.triple
        cvalid, rvalid = cg >= 0, rg >= 0
        cgs, rgs = np.where(cvalid, cg, 0), np.where(rvalid, rg, 0)
        for which, col_arr, row_arr in ((PSI, t.psi_c, t.psi_r), (LAM, t.lam_c, t.lam_r),
                                        (PHI, t.phi_c, t.phi_r), (PSI_PREV, t.psi_prev_c, None)):
            buf = sess.get(which)
            col_arr[:] = np.where(cvalid, buf[cgs], 0.0)
            if row_arr is not None:
                row_arr[:] = np.where(rvalid, buf[rgs], 0.0)

    def _prepare(self, strategy: ExecStrategy) -> DeviceSession:
        if self.row_data is None:
            raise ValueError("no row data set on the workspace")
        sess = self.session(strategy.exact, strategy.device)
        sess.set_x(_x_of(self.row_data, self.tables))
        self.upload_triple(sess)
        return sess

    def device_iterate(self, strategy: ExecStrategy, n: int = 1):
        """Exactly n iterations from the current triple; triple refreshed.
        Returns the (pri, dual) of the last iteration."""
        sess = self._prepare(strategy)
        hist = sess.iterate(n)
        self.last_device_ms = sess.last_timing()[0]
        self.download_triple(sess)
        return float(hist[-1, 0]), float(hist[-1, 1])

    def device_solve(self, strategy: ExecStrategy, max_iters: int, eps_pri: float, eps_dual: float):
        sess = self._prepare(strategy)
        n, hist, ok = sess.solve(max_iters, eps_pri, eps_dual)
        self.last_device_ms = sess.last_timing()[0]
        self.download_triple(sess)
        return n, [(float(p), float(d)) for p, d in hist], ok

    def close(self):
        for s in self._sessions.values():
            s.close()
        self._sessions.clear()


def admm_solve(row_data: RowData, col_solvers, triple: PhiTriple, spec: ProblemSpec,
               strategy=None, executor=None, workspace: AdmmWorkspace | None = None) -> AdmmState:
    """Consensus ADMM from the triple as passed (zero it for a cold start),
    until pri <= eps_pri and dual <= eps_dual; NotConverged at max_iters
    (reference admm.py:315-347). The whole loop runs in one device launch."""
    if executor is not None:
        strat = executor.strategy
    elif isinstance(strategy, str):
        strat = ExecStrategy(strategy)
    else:
        strat = strategy or ExecStrategy("b200")
    if workspace is None:
        workspace = AdmmWorkspace(triple, col_solvers, spec)
    workspace.set_row_data(row_data)
    n, history, ok = workspace.device_solve(strat, spec.max_iters, spec.eps_pri, spec.eps_dual)
    if executor is not None:
        executor.ledger.record_launch(n, workspace.last_device_ms)
    triple._dlmpc_ws = (workspace, strat)
    if not ok:
        raise NotConverged(history)
    return AdmmState(triple, n, history, True)


def verify_fixed_point(triple: PhiTriple, row_data: RowData, operator, spec: ProblemSpec) -> FixedPointReport:
    """Audit a solve without trusting the iteration that produced it
    (reference admm.py:417-434), on the device: the dynamics residual of the
    projected iterate through each column's restricted operator, the change
    of a fresh row solve at the final dual point, and the consensus gap; all
    within 10 x eps_pri for an accepted solve. The triple's arrays (including
    its φ) are what is audited."""
    from .sls_core import build_column_classes
    ws, strat = getattr(triple, "_dlmpc_ws", (None, ExecStrategy("b200")))
    if ws is None or ws.triple is not triple:
        ws = AdmmWorkspace(triple, build_column_classes(operator, triple.tables.mask), spec)
    ws.set_row_data(row_data)
    sess = ws._prepare(strat)
    _, rg = ws._gathers(sess.layout)
    phi = np.zeros(sess.n_cell)
    phi[rg[rg >= 0]] = triple.phi_r[rg >= 0]      # the reference audits the row layout
    dyn, res, gap = sess.audit(phi)
    return FixedPointReport(dyn, res, gap, 10.0 * spec.eps_pri)


# ---------------------------------------------------------------------------
# closed loop
# ---------------------------------------------------------------------------

_SPEC_ARRAYS = ("state_weights", "input_weights", "terminal_weights", "state_lo", "state_hi", "input_lo",
                "input_hi")


def _spec_arrays(spec: ProblemSpec):
    """Copies of the spec's arrays and scalars a cached session was built for."""
    return ([np.array(getattr(spec, n), dtype=np.float64, copy=True) for n in _SPEC_ARRAYS],
            (spec.horizon, spec.rho))


def _spec_unchanged(sess, spec: ProblemSpec) -> bool:
    """The cached session still matches `spec` (an in-place edit of its arrays
    invalidates it); array comparisons instead of re-hashing on every call."""
    arrays, scalars = sess._spec_arrays
    if scalars != (spec.horizon, spec.rho):
        return False
    return all(np.array_equal(a, getattr(spec, n)) for a, n in zip(arrays, _SPEC_ARRAYS))


def _spec_fingerprint(spec: ProblemSpec) -> bytes:
    h = hashlib.blake2b(digest_size=16)
    for name in ("state_weights", "input_weights", "terminal_weights", "state_lo",
                 "state_hi", "input_lo", "input_hi"):
        h.update(np.ascontiguousarray(getattr(spec, name), dtype=np.float64).tobytes())
    h.update(repr((spec.horizon, spec.rho)).encode())
    return h.digest()


def _plant_views(system: LtiSystem, mask: LocalityMask):
    arrs = []
    for m in (system.a, system.b):
        arrs += [m.data, m.indices, m.indptr]
    if mask.compact is not None:   # explicit masks hold immutable support tuples
        arrs += [mask.compact["ball_ptr"], mask.compact["ball_idx"]]
    return arrs, (mask.n_rows, mask.n_cols, mask.d, mask.d_row, mask.d_col)


def _plant_arrays(system: LtiSystem, mask: LocalityMask):
    """Copies of what a cached session was built from besides the spec: the
    plant's CSR arrays (A, B) and the locality structure. The reference
    rebuilds its operators on every dlmpc_simulate call (admm.py:470-475), so
    an in-place edit of any of these between calls must not hit a stale
    session."""
    arrs, key = _plant_views(system, mask)
    return [np.array(a, copy=True) for a in arrs], key


def _plant_unchanged(sess, system: LtiSystem, mask: LocalityMask) -> bool:
    arrs, key = sess._plant
    cur, cur_key = _plant_views(system, mask)
    return key == cur_key and len(arrs) == len(cur) and \
        all(a.shape == np.shape(b) and np.array_equal(a, b) for a, b in zip(arrs, cur))


class DlmpcSession:
    """Precomputed closed-loop session on one GPU: the reference's
    `precompute_global` (dynamics operator, column solvers) plus the device
    upload, reusable across `simulate` calls with different x0."""

    def __init__(self, system: LtiSystem, spec: ProblemSpec, mask: LocalityMask,
                 strategy="b200", tile_cols: int | None = None):
        strat = ExecStrategy(strategy) if isinstance(strategy, str) else strategy
        self.system, self.spec, self.mask, self.strategy = system, spec, mask, strat
        t0 = time.perf_counter()
        # class-deduplicated column operators from the structural builder:
        # the same bits as the reference's per-column reduction, O(classes)
        # factorizations instead of O(N) (sls_core.py:253-289)
        self.classes = build_column_classes_structural(system, spec.horizon, mask)
        self.layout = DeviceLayout(system, spec, mask, self.classes, exact=strat.exact,
                                   tile_cols=tile_cols)
        self.device = DeviceSession(self.layout, strat.device)
        self.precompute_s = time.perf_counter() - t0
        self._fp = _spec_fingerprint(spec)
        self._spec_arrays = _spec_arrays(spec)
        self._plant = _plant_arrays(system, mask)

    def simulate(self, x0, t_sim: int, warm_start: bool = True):
        """Closed loop on device; returns (Trajectory, device_ms)."""
        out = self.device.simulate(x0, t_sim, self.spec.max_iters, self.spec.eps_pri,
                                   self.spec.eps_dual, warm_start=warm_start, cold_start=True)
        traj = Trajectory(out["states"], out["inputs"], out["step_iterations"])
        return traj, self.device.last_timing()[0]

    def simulate_audited(self, x0, t_sim: int, warm_start: bool, ledger):
        """The closed loop one MPC step per launch with the on-device
        fixed-point audit after every solve (reference admm.py:506-513)."""
        x = np.asarray(x0, dtype=np.float64)
        states, inputs, iters = [x], [], []
        worst = {"dynamics_residual": 0.0, "resolve_residual": 0.0, "consensus_gap": 0.0}
        for step in range(t_sim):
            try:
                out = self.device.simulate(x, 1, self.spec.max_iters, self.spec.eps_pri, self.spec.eps_dual,
                                           warm_start=warm_start, cold_start=(step == 0 or not warm_start))
            except (NotConverged, RowInfeasible) as err:
                err.step = step
                raise
            ledger.record_launch(out["step_iterations"][0], self.device.last_timing()[0])
            for key, v in zip(worst, self.device.audit()):
                worst[key] = max(worst[key], v)
            x = out["states"][1]
            states.append(x)
            inputs.append(out["inputs"][0])
            iters.append(out["step_iterations"][0])
        return Trajectory(np.array(states), np.array(inputs), iters), worst

    def close(self):
        self.device.close()


_SESSIONS = {}


def _cached_session(system, spec, mask, strat):
    key = (id(system), id(spec), id(mask), strat.variant, strat.device)
    hit = _SESSIONS.get(key)
    if hit is not None:
        ref_sys, ref_spec, ref_mask, sess = hit
        if ref_sys() is system and ref_spec() is spec and ref_mask() is mask \
                and _spec_unchanged(sess, spec) and _plant_unchanged(sess, system, mask):
            return sess, True
        sess.close()
        del _SESSIONS[key]
    sess = DlmpcSession(system, spec, mask, strat)
    if len(_SESSIONS) > 8:
        for k in list(_SESSIONS)[:4]:
            _SESSIONS.pop(k)[3].close()
    _SESSIONS[key] = (weakref.ref(system), weakref.ref(spec), weakref.ref(mask), sess)
    return sess, False


def dlmpc_simulate(system: LtiSystem, spec: ProblemSpec, mask: LocalityMask,
                   x0: np.ndarray, t_sim: int, strategy="b200",
                   warm_start: bool = True, audit: bool = False):
    """Closed-loop MPC (reference admm.py:437-540): t_sim times row data,
    ADMM solve, control extraction and plant step -- all in one persistent
    device launch. Returns (Trajectory, RunReport); raises NotConverged /
    RowInfeasible carrying the failing step like the reference."""
    from .report import PHASES, RunReport

    x0 = np.asarray(x0, dtype=np.float64)
    if x0.shape != (system.n_states,):
        raise ValueError("x0 length must equal the global state dimension")
    if t_sim < 1:
        raise ValueError("t_sim must be >= 1")
    strat = ExecStrategy(strategy) if isinstance(strategy, str) else strategy
    total_start = time.perf_counter()
    phases = dict.fromkeys(PHASES, 0.0)
    start = time.perf_counter()
    executor = Executor(strat)
    phases["setup"] = time.perf_counter() - start
    start = time.perf_counter()
    sess, _ = _cached_session(system, spec, mask, strat)
    phases["precompute_global"] = time.perf_counter() - start
    start = time.perf_counter()
    audit_worst = None
    try:
        if not audit:
            traj, dev_ms = sess.simulate(x0, t_sim, warm_start)
            executor.ledger.record_launch(sum(traj.step_iterations), dev_ms)
        else:
            traj, audit_worst = sess.simulate_audited(x0, t_sim, warm_start, executor.ledger)
            dev_ms = executor.ledger.device_time_ms
    finally:
        phases["optimize"] = time.perf_counter() - start
    report = RunReport(
        scenario={"strategy": strat.variant, "worker_count": executor.workers, "t_sim": t_sim,
                  "warm_start": warm_start, "rho": spec.rho, "eps": spec.eps_pri,
                  "device_ms": dev_ms},
        phase_times_ms={k: v * 1e3 for k, v in phases.items()},
        per_step_iters=list(traj.step_iterations),
        ledger=executor.ledger,
        closed_loop_cost=closed_loop_cost(traj),
        converged_all_steps=True,
        total_wall_ms=(time.perf_counter() - total_start) * 1e3,
        audit_worst=audit_worst,
    )
    return traj, report
