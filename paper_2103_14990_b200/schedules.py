"""The reference's four device schedules and scalar stage functions, on the GPU.

The reference package models the paper's GPU schemes (arXiv 2103.14990
§III) as CPU thread-pool schedules over its dual padded layout
(`strategies.py:262-314`, `admm.py:153-270`, `sls_core.py:352-518`):

  naive / padded  per iteration 4 stage launches + 4 host syncs
  fused           Φ launch, host sync, combined column launch, flag read
  patch-local     one column-patch launch, pointer swap, flag read

`ScheduleEngine` runs those schedules for real on the B200
(`csrc/dlmpc_schedules.cuh`): the state is the reference's own padded
layouts in device memory, each stage is one kernel launch, each host sync a
stream synchronisation and each flag read a 16-byte read of the reduced
residual pair -- so the reference's `SyncLedger` counts real events, and the
arithmetic is the reference's bit for bit (every schedule reproduces the
reference's iterates exactly).

The scalar functions (`phi_row_solve`, `psi_column_solve`, `lambda_update`,
`column_residuals`, `extract_control`, `step_dynamics`; admm.py:28-74,
350-369) are device operators too (`dlmpc_op_*`). There is no CPU path.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from .device import _SchedProblem, _i32p, _i64p, _f64p, load_library
from .errors import DeviceError, RowInfeasible

# stage kernels (include/dlmpc.h DLMPC_STAGE_*)
(STAGE_PHI_ROWS, STAGE_PHI_ROWS_PADDED, STAGE_EXCHANGE_PHI, STAGE_PSI_COLS, STAGE_LAMBDA_COLS,
 STAGE_LAMBDA_ELEMS, STAGE_CONV_COLS, STAGE_EXCHANGE_PSI_LAM, STAGE_FUSED_COLS, STAGE_PATCH_COLS,
 STAGE_PATCH_COLS_PADDED) = range(11)
# arrays (DLMPC_SCHED_*)
(A_PHI_R, A_PSI_R, A_LAM_R, A_PHI_C, A_PSI_C, A_LAM_C, A_PSI_PREV_C, A_PRI_C, A_DUAL_C, A_A_PAD, A_ADA,
 A_ROW_W, A_ROW_LO, A_ROW_HI) = range(14)

TRIPLE_ARRAYS = (("phi_r", A_PHI_R), ("psi_r", A_PSI_R), ("lam_r", A_LAM_R), ("phi_c", A_PHI_C),
                 ("psi_c", A_PSI_C), ("lam_c", A_LAM_C), ("psi_prev_c", A_PSI_PREV_C))

DEVICE_SCHEDULES = ("naive", "padded", "fused", "patch-local")


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _check_global(rc, what):
    if rc != 0:
        lib = load_library()
        raise DeviceError(f"{what}: {lib.dlmpc_global_error().decode()} (status {rc})")


def _classes_of(col_solvers):
    from .sls_core import ColumnClasses
    if isinstance(col_solvers, ColumnClasses):
        return col_solvers
    cc = getattr(col_solvers, "classes", None)
    return cc if cc is not None else ColumnClasses.from_precomps(col_solvers)


def patch_tables(tables, patches):
    """Concatenated patch tables (reference AdmmWorkspace._build_patch_tables,
    admm.py:139-151): member rows, the column's slot in each, ownership."""
    members = [np.asarray(p.member_rows, dtype=np.int64) for p in patches]
    lens = np.array([m.size for m in members], dtype=np.int64)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    rows = np.concatenate(members) if members else np.zeros(0, np.int64)
    slot = np.concatenate([tables.col_slot_in_row[c, :lens[c]] for c in range(len(patches))]).astype(np.int32)
    owned = (tables.owner_col[rows] == np.repeat(np.arange(len(patches)), lens)).astype(np.int32)
    return off, rows, slot, owned


class ScheduleEngine:
    """Device state + stage kernels of one workspace (reference layouts)."""

    def __init__(self, tables, col_solvers, rho: float, patches=None, device: int = 0):
        self._lib = load_library()
        self._h = None
        self.tables = t = tables
        self.device = int(device)
        self.n_rows, self.n_cols, self.d_row, self.d_col = t.n_rows, t.n_cols, t.d_row, t.d_col
        self.n_elems = int(t.n_elems)
        keep = {}
        keep["row_len"] = _c(t.row_len, np.int32)
        keep["col_len"] = _c(t.col_len, np.int32)
        keep["rs"] = _c(t.rs, np.int64)
        keep["c2r"] = _c(np.where(t.col_valid, t.c2r_flat, -1), np.int64)
        keep["r2c"] = _c(np.where(t.row_valid, t.r2c_flat, -1), np.int64)
        keep["ef"] = _c(t.elem_flat_col, np.int64)
        if col_solvers is not None:
            cc = _classes_of(col_solvers)
            gs = [np.ascontiguousarray(k.g, dtype=np.float64) for k in cc.classes]
            ps = [np.ascontiguousarray(k.projector, dtype=np.float64) for k in cc.classes]
            keep["col_class"] = _c(cc.col_class, np.int32)
            keep["class_m"] = np.array([g.shape[0] for g in gs], dtype=np.int32)
            keep["class_s"] = np.array([g.shape[1] for g in gs], dtype=np.int32)
            keep["g_off"] = np.concatenate([[0], np.cumsum([g.size for g in gs])]).astype(np.int64)
            keep["g_pool"] = _c(np.concatenate([g.ravel() for g in gs]) if gs else np.zeros(1), np.float64)
            keep["p_off"] = np.concatenate([[0], np.cumsum([p.size for p in ps])]).astype(np.int64)
            keep["p_pool"] = _c(np.concatenate([p.ravel() for p in ps]) if ps else np.zeros(1), np.float64)
            rhs = [np.asarray(cc.reduced_rhs(c), dtype=np.float64) for c in range(t.n_cols)]
            keep["rhs_off"] = np.concatenate([[0], np.cumsum([r.size for r in rhs])]).astype(np.int64)
            keep["rhs_pool"] = _c(np.concatenate(rhs) if rhs else np.zeros(1), np.float64)
            n_classes = len(gs)
        else:   # row stages only (e.g. the audit's fresh Φ)
            keep["col_class"] = np.zeros(t.n_cols, np.int32)
            keep["class_m"] = keep["class_s"] = np.zeros(1, np.int32)
            keep["g_off"] = keep["p_off"] = np.zeros(1, np.int64)
            keep["g_pool"] = keep["p_pool"] = np.zeros(1)
            keep["rhs_off"] = np.zeros(t.n_cols + 1, np.int64)
            keep["rhs_pool"] = np.zeros(1)
            n_classes = 0
        self.has_columns = col_solvers is not None
        if patches is None:
            from .strategies import build_patches
            patches = build_patches(t)
        po, prw, pslot, pown = patch_tables(t, patches)
        keep.update(po=po, prw=prw, pslot=pslot, pown=pown)
        pr = _SchedProblem()
        pr.n_rows, pr.n_cols, pr.d_row, pr.d_col = self.n_rows, self.n_cols, self.d_row, self.d_col
        pr.n_elems, pr.rho = self.n_elems, float(rho)
        pr.row_len, pr.col_len = _p(keep["row_len"], C.c_int32), _p(keep["col_len"], C.c_int32)
        pr.rs, pr.c2r_flat, pr.r2c_flat = (_p(keep[k], C.c_int64) for k in ("rs", "c2r", "r2c"))
        pr.elem_flat_col = _p(keep["ef"], C.c_int64)
        pr.n_classes = n_classes
        pr.col_class, pr.class_m, pr.class_s = (_p(keep[k], C.c_int32) for k in ("col_class", "class_m", "class_s"))
        pr.class_g_off, pr.class_p_off, pr.col_rhs_off = (_p(keep[k], C.c_int64) for k in ("g_off", "p_off", "rhs_off"))
        pr.g_pool, pr.p_pool, pr.rhs_pool = (_p(keep[k], C.c_double) for k in ("g_pool", "p_pool", "rhs_pool"))
        pr.n_patch = int(prw.size)
        pr.patch_off, pr.patch_rows = _p(po, C.c_int64), _p(prw, C.c_int64)
        pr.patch_slot, pr.patch_owned = _p(pslot, C.c_int32), _p(pown, C.c_int32)
        h = C.c_void_p()
        _check_global(self._lib.dlmpc_sched_create(C.byref(pr), self.device, C.byref(h)), "dlmpc_sched_create")
        self._h = h
        self.duplicated_rows_per_iter = int(prw.size) - int(np.unique(prw).size) if prw.size else 0

    # -- plumbing ---------------------------------------------------------------
    def _check(self, rc, what):
        if rc != 0:
            raise DeviceError(f"{what}: {self._lib.dlmpc_sched_last_error(self._h).decode()} (status {rc})")
        return rc

    def close(self):
        if self._h is not None:
            self._lib.dlmpc_sched_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:   # noqa: BLE001 -- interpreter teardown
            pass

    def put(self, which, arr):
        a = _c(arr, np.float64)
        self._check(self._lib.dlmpc_sched_put(self._h, which, _p(a, C.c_double)), "dlmpc_sched_put")

    def get(self, which, out):
        """Device array into `out` (C-contiguous float64, written in place)."""
        if out.flags.c_contiguous and out.dtype == np.float64:
            self._check(self._lib.dlmpc_sched_get(self._h, which, _p(out, C.c_double)), "dlmpc_sched_get")
        else:
            tmp = np.empty(out.shape)
            self._check(self._lib.dlmpc_sched_get(self._h, which, _p(tmp, C.c_double)), "dlmpc_sched_get")
            out[...] = tmp

    def push_triple(self, triple):
        for name, which in TRIPLE_ARRAYS:
            self.put(which, getattr(triple, name))

    def pull_triple(self, triple):
        for name, which in TRIPLE_ARRAYS:
            self.get(which, getattr(triple, name))

    def push_row_data(self, rd):
        self.put(A_A_PAD, rd.a_pad)
        self.put(A_ADA, rd.a_dot_a)
        self.put(A_ROW_W, rd.weight)
        self.put(A_ROW_LO, rd.lo)
        self.put(A_ROW_HI, rd.hi)

    def set_costs(self, weight, lo, hi):
        self.put(A_ROW_W, weight)
        self.put(A_ROW_LO, lo)
        self.put(A_ROW_HI, hi)

    def set_x(self, x):
        """Row data of the measured state on the device (sls_core.py:330-349)."""
        x = _c(x, np.float64)
        bad = C.c_int64(-1)
        rc = self._lib.dlmpc_sched_set_x(self._h, _p(x, C.c_double), x.size, C.byref(bad))
        if rc == 2:
            raise RowInfeasible(int(bad.value))
        self._check(rc, "dlmpc_sched_set_x")

    def stage(self, stage, lo, hi):
        self._check(self._lib.dlmpc_sched_stage(self._h, int(stage), int(lo), int(hi)), "dlmpc_sched_stage")

    def sync(self):
        self._check(self._lib.dlmpc_sched_sync(self._h), "dlmpc_sched_sync")

    def read_residuals(self):
        out = np.zeros(2)
        self._check(self._lib.dlmpc_sched_read_residuals(self._h, _p(out, C.c_double)), "dlmpc_sched_read_residuals")
        return float(out[0]), float(out[1])

    def phi_compute(self, lo, hi):
        out = np.zeros((hi - lo, self.d_row))
        if hi > lo:
            self._check(self._lib.dlmpc_sched_phi_compute(self._h, int(lo), int(hi), _p(out, C.c_double)),
                        "dlmpc_sched_phi_compute")
        return out

    def swap_rows(self):
        self._check(self._lib.dlmpc_sched_swap_rows(self._h), "dlmpc_sched_swap_rows")


# ---------------------------------------------------------------------------
# the reference's scalar stage functions as device operators
# ---------------------------------------------------------------------------
def op_phi_rows(a, v, ada, weight, lo, hi, rho, lengths=None, device=0):
    """Batched phi_row_solve: rows of a / v (n x d), each of length lengths[i]."""
    a, v = _c(np.atleast_2d(a), np.float64), _c(np.atleast_2d(v), np.float64)
    n, d = a.shape
    ln = _c(np.full(n, d) if lengths is None else lengths, np.int32)
    ada, w, lo, hi = (_c(np.broadcast_to(z, (n,)), np.float64) for z in (ada, weight, lo, hi))
    out = np.zeros((n, d))
    lib = load_library()
    _check_global(lib.dlmpc_op_phi_rows(int(device), n, d, _p(ln, C.c_int32), _p(a, C.c_double),
                                        _p(v, C.c_double), _p(ada, C.c_double), _p(w, C.c_double),
                                        _p(lo, C.c_double), _p(hi, C.c_double), float(rho),
                                        _p(out, C.c_double)), "dlmpc_op_phi_rows")
    return out


def op_psi_cols(g, projector, rhs, k, device=0):
    """Batched psi_column_solve: g (n x m x s), projector (n x s x m), rhs (n x m), k (n x s)."""
    g, P = _c(g, np.float64), _c(projector, np.float64)
    rhs, k = _c(rhs, np.float64), _c(k, np.float64)
    n, m, s = g.shape
    out = np.zeros((n, s))
    lib = load_library()
    _check_global(lib.dlmpc_op_psi_cols(int(device), n, m, s, _p(g, C.c_double), _p(P, C.c_double),
                                        _p(rhs, C.c_double), _p(k, C.c_double), _p(out, C.c_double)),
                  "dlmpc_op_psi_cols")
    return out


def op_lambda(lam, phi, psi, device=0):
    lam, phi, psi = (_c(z, np.float64) for z in (lam, phi, psi))
    out = np.zeros(lam.shape)
    lib = load_library()
    _check_global(lib.dlmpc_op_lambda(int(device), lam.size, _p(lam, C.c_double), _p(phi, C.c_double),
                                      _p(psi, C.c_double), _p(out, C.c_double)), "dlmpc_op_lambda")
    return out


def op_residuals(phi, psi, prev, lengths, rho, device=0):
    """Per row of phi/psi/prev (n x d) over its first lengths[i] entries:
    (max|phi - psi|, rho * max|psi - prev|)."""
    phi, psi, prev = (_c(np.atleast_2d(z), np.float64) for z in (phi, psi, prev))
    n, d = phi.shape
    ln = _c(lengths, np.int32)
    out = np.zeros((n, 2))
    lib = load_library()
    _check_global(lib.dlmpc_op_residuals(int(device), n, d, _p(ln, C.c_int32), _p(phi, C.c_double),
                                         _p(psi, C.c_double), _p(prev, C.c_double), float(rho),
                                         _p(out, C.c_double)), "dlmpc_op_residuals")
    return out


def op_row_dots(vals, idx, lengths, x, device=0):
    """out[i] = ascending sum_j vals[i, j] * x[idx[i, j]] over j < lengths[i]."""
    vals, idx = _c(np.atleast_2d(vals), np.float64), _c(np.atleast_2d(idx), np.int64)
    x = _c(x, np.float64)
    n, d = vals.shape
    ln = _c(lengths, np.int32)
    out = np.zeros(n)
    lib = load_library()
    _check_global(lib.dlmpc_op_row_dots(int(device), n, d, _p(ln, C.c_int32), _p(vals, C.c_double),
                                        _p(idx, C.c_int64), x.size, _p(x, C.c_double), _p(out, C.c_double)),
                  "dlmpc_op_row_dots")
    return out


def op_plant_step(a, b, x, u, device=0):
    """x+ = A x + B u with scipy's CSR accumulation order (admm.py:363-369)."""
    a, b = a.tocsr(), b.tocsr()
    x, u = _c(x, np.float64), _c(u, np.float64)
    ap, ai, av = _c(a.indptr, np.int64), _c(a.indices, np.int32), _c(a.data, np.float64)
    bp, bi, bv = _c(b.indptr, np.int64), _c(b.indices, np.int32), _c(b.data, np.float64)
    out = np.zeros(a.shape[0])
    if u.size == 0:
        u = np.zeros(1)
    lib = load_library()
    _check_global(lib.dlmpc_op_plant_step(int(device), a.shape[0], b.shape[1], _p(ap, C.c_int64), _p(ai, C.c_int32),
                                          _p(av, C.c_double), _p(bp, C.c_int64), _p(bi, C.c_int32),
                                          _p(bv, C.c_double), _p(x, C.c_double), _p(u, C.c_double),
                                          _p(out, C.c_double)), "dlmpc_op_plant_step")
    return out
