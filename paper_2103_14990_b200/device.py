"""ctypes binding of libdlmpc.so (include/dlmpc.h) and the device session.

The shared library is built in-tree (`build.py`, `__graft_entry__.build`)
and loaded from this package directory. If it is missing or no CUDA device
is visible, every entry point raises `DeviceError` -- there is no CPU path.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .errors import DeviceError, NotConverged, RowInfeasible

_LIB_PATH = os.environ.get("DLMPC_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                          "libdlmpc.so")

DLMPC_OK, DLMPC_NOT_CONVERGED, DLMPC_ROW_INFEASIBLE = 0, 1, 2
DLMPC_BAD_ARGUMENT, DLMPC_CUDA_ERROR, DLMPC_NO_DEVICE = 3, 4, 5
PSI, LAM, PSI_PREV, PHI, LAM_PREV, S_ROW, X, ADA = range(8)

_P = C.POINTER
_i32p, _i64p, _f64p = _P(C.c_int32), _P(C.c_int64), _P(C.c_double)


class _Problem(C.Structure):
    _fields_ = [
        ("n_sub", C.c_int32), ("n_rows", C.c_int32), ("n_cols", C.c_int32), ("n_inputs", C.c_int32),
        ("s_pad", C.c_int32), ("horizon", C.c_int32), ("exact", C.c_int32), ("contiguous", C.c_int32),
        ("own_sub_lo", C.c_int32), ("own_sub_hi", C.c_int32), ("own_col_lo", C.c_int32), ("own_col_hi", C.c_int32),
        ("rho", C.c_double),
        ("row_start", _i64p), ("ball_ptr", _i64p), ("ball_idx", _i32p), ("ball_off", _i32p),
        ("state_start", _i32p), ("state_count", _i32p), ("sub_first_bad", _i32p),
        ("d_pad", C.c_int32), ("supp_col", _i32p), ("supp_off", _i32p), ("supp_len", _i32p),
        ("row_w", _f64p), ("row_lo", _f64p), ("row_hi", _f64p),
        ("col_owner", _i32p), ("col_len", _i32p), ("col_class", _i32p), ("col_vec", _i32p),
        ("col_irow", _i32p), ("col_rowbase", _i64p),
        ("n_classes", C.c_int32), ("class_s", _i32p), ("class_n0", _i32p), ("class_ldn", _i32p),
        ("class_null_off", _i64p), ("null_pool", _f64p),
        ("n_vec", C.c_int32), ("q_pool", _f64p),
        ("class_m", _i32p), ("class_g_off", _i64p), ("class_p_off", _i64p),
        ("g_pool", _f64p), ("p_pool", _f64p), ("m_pad", C.c_int32), ("rhs_pool", _f64p),
        ("ref_pos", _i32p),
        ("n_tiles", C.c_int32), ("tile_cols", C.c_int32),
        ("tile_class", _i32p), ("tile_first", _i32p), ("tile_count", _i32p), ("tile_colv", _i32p),
        ("a_ptr", _i64p), ("a_idx", _i32p), ("a_val", _f64p),
        ("b_ptr", _i64p), ("b_idx", _i32p), ("b_val", _f64p),
        ("input_owner", _i32p), ("input_local", _i32p),
        ("class_ntouch", _i32p), ("class_g0_off", _i64p), ("g0_pool", _f64p),
        ("class_perm_off", _i64p), ("perm_pool", _i32p), ("col_pin", _i32p),
        ("grid_ctas", C.c_int32),
    ]


EXPORTS = ("dlmpc_create", "dlmpc_destroy", "dlmpc_last_error", "dlmpc_global_error",
           "dlmpc_set_x", "dlmpc_solve", "dlmpc_iterate", "dlmpc_simulate",
           "dlmpc_simulate_device", "dlmpc_get", "dlmpc_put", "dlmpc_zero",
           "dlmpc_last_timing", "dlmpc_stream", "dlmpc_synchronize", "dlmpc_info", "dlmpc_plan_flags",
           "dlmpc_phase_times", "dlmpc_audit", "dlmpc_get_cols", "dlmpc_put_cols",
           "dlmpc_finish_step", "dlmpc_set_halo", "dlmpc_halo_pack", "dlmpc_halo_unpack",
           "dlmpc_iterate_async", "dlmpc_halo_pack_async", "dlmpc_halo_unpack_async", "dlmpc_set_stream",
           "dlmpc_fp64_peak",
           "dlmpc_sched_create", "dlmpc_sched_destroy", "dlmpc_sched_last_error", "dlmpc_sched_put",
           "dlmpc_sched_get", "dlmpc_sched_set_x", "dlmpc_sched_stage", "dlmpc_sched_sync",
           "dlmpc_sched_read_residuals", "dlmpc_sched_phi_compute", "dlmpc_sched_swap_rows",
           "dlmpc_op_phi_rows", "dlmpc_op_psi_cols", "dlmpc_op_lambda", "dlmpc_op_residuals",
           "dlmpc_op_row_dots", "dlmpc_op_plant_step",
           "dlmpc_dist_alloc", "dlmpc_dist_setup", "dlmpc_dist_solve", "dlmpc_multi_solve",
           "dlmpc_ipc_get", "dlmpc_ipc_open", "dlmpc_ipc_close")


class _SchedProblem(C.Structure):
    _fields_ = [
        ("n_rows", C.c_int32), ("n_cols", C.c_int32), ("d_row", C.c_int32), ("d_col", C.c_int32),
        ("n_elems", C.c_int64), ("rho", C.c_double),
        ("row_len", _i32p), ("col_len", _i32p), ("rs", _i64p), ("c2r_flat", _i64p), ("r2c_flat", _i64p),
        ("elem_flat_col", _i64p),
        ("n_classes", C.c_int32), ("col_class", _i32p), ("class_m", _i32p), ("class_s", _i32p),
        ("class_g_off", _i64p), ("g_pool", _f64p), ("class_p_off", _i64p), ("p_pool", _f64p),
        ("col_rhs_off", _i64p), ("rhs_pool", _f64p),
        ("n_patch", C.c_int64), ("patch_off", _i64p), ("patch_rows", _i64p), ("patch_slot", _i32p),
        ("patch_owned", _i32p),
        ("row_w", _f64p), ("row_lo", _f64p), ("row_hi", _f64p),
    ]

_lib = None


def library_path() -> str:
    return _LIB_PATH


def load_library():
    """Load libdlmpc.so (raises DeviceError if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise DeviceError(f"{_LIB_PATH} is missing: run `python build.py` (or "
                          f"__graft_entry__.build()) to compile the CUDA library")
    lib = C.CDLL(_LIB_PATH)
    vp = C.c_void_p
    lib.dlmpc_create.argtypes = [_P(_Problem), C.c_int, _P(vp)]
    lib.dlmpc_destroy.argtypes = [vp]
    lib.dlmpc_destroy.restype = None
    lib.dlmpc_last_error.argtypes = [vp]
    lib.dlmpc_last_error.restype = C.c_char_p
    lib.dlmpc_global_error.restype = C.c_char_p
    lib.dlmpc_set_x.argtypes = [vp, _f64p, _i64p]
    lib.dlmpc_solve.argtypes = [vp, C.c_int, C.c_double, C.c_double, _i32p, _f64p]
    lib.dlmpc_iterate.argtypes = [vp, C.c_int, _f64p]
    lib.dlmpc_simulate.argtypes = [vp, _f64p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                   _f64p, _f64p, _i32p, _i32p, _i64p, _i32p, _f64p]
    lib.dlmpc_simulate_device.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                          C.c_double, vp, vp, vp, vp]
    lib.dlmpc_get.argtypes = [vp, C.c_int, _f64p]
    lib.dlmpc_put.argtypes = [vp, C.c_int, _f64p]
    lib.dlmpc_zero.argtypes = [vp]
    lib.dlmpc_last_timing.argtypes = [vp, _P(C.c_float), _i32p]
    lib.dlmpc_stream.argtypes = [vp]
    lib.dlmpc_stream.restype = vp
    lib.dlmpc_synchronize.argtypes = [vp]
    lib.dlmpc_info.argtypes = [vp, _i64p]
    lib.dlmpc_plan_flags.argtypes = [vp, _i64p, C.c_int]
    lib.dlmpc_phase_times.argtypes = [vp, _P(C.c_uint64), C.c_int]
    lib.dlmpc_audit.argtypes = [vp, _f64p, _f64p]
    lib.dlmpc_get_cols.argtypes = [vp, C.c_int, C.c_int, C.c_int, vp]
    lib.dlmpc_put_cols.argtypes = [vp, C.c_int, C.c_int, C.c_int, vp]
    lib.dlmpc_finish_step.argtypes = [vp, _f64p, _f64p]
    lib.dlmpc_set_halo.argtypes = [vp, _i64p, C.c_int64, _i64p, C.c_int64]
    lib.dlmpc_halo_pack.argtypes = [vp, vp]
    lib.dlmpc_halo_unpack.argtypes = [vp, vp]
    lib.dlmpc_iterate_async.argtypes = [vp, C.c_int, vp]
    lib.dlmpc_halo_pack_async.argtypes = [vp, vp]
    lib.dlmpc_halo_unpack_async.argtypes = [vp, vp]
    lib.dlmpc_set_stream.argtypes = [vp, vp]
    lib.dlmpc_fp64_peak.argtypes = [C.c_int, _f64p]
    lib.dlmpc_sched_create.argtypes = [_P(_SchedProblem), C.c_int, _P(vp)]
    lib.dlmpc_sched_destroy.argtypes = [vp]
    lib.dlmpc_sched_destroy.restype = None
    lib.dlmpc_sched_last_error.argtypes = [vp]
    lib.dlmpc_sched_last_error.restype = C.c_char_p
    lib.dlmpc_sched_put.argtypes = [vp, C.c_int, _f64p]
    lib.dlmpc_sched_get.argtypes = [vp, C.c_int, _f64p]
    lib.dlmpc_sched_set_x.argtypes = [vp, _f64p, C.c_int64, _i64p]
    lib.dlmpc_sched_stage.argtypes = [vp, C.c_int, C.c_int64, C.c_int64]
    lib.dlmpc_sched_sync.argtypes = [vp]
    lib.dlmpc_sched_read_residuals.argtypes = [vp, _f64p]
    lib.dlmpc_sched_phi_compute.argtypes = [vp, C.c_int64, C.c_int64, _f64p]
    lib.dlmpc_sched_swap_rows.argtypes = [vp]
    lib.dlmpc_op_phi_rows.argtypes = [C.c_int, C.c_int, C.c_int, _i32p, _f64p, _f64p, _f64p, _f64p, _f64p,
                                      _f64p, C.c_double, _f64p]
    lib.dlmpc_op_psi_cols.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _f64p, _f64p, _f64p, _f64p, _f64p]
    lib.dlmpc_op_lambda.argtypes = [C.c_int, C.c_int64, _f64p, _f64p, _f64p, _f64p]
    lib.dlmpc_op_residuals.argtypes = [C.c_int, C.c_int, C.c_int, _i32p, _f64p, _f64p, _f64p, C.c_double, _f64p]
    lib.dlmpc_op_row_dots.argtypes = [C.c_int, C.c_int, C.c_int, _i32p, _f64p, _i64p, C.c_int64, _f64p, _f64p]
    lib.dlmpc_op_plant_step.argtypes = [C.c_int, C.c_int, C.c_int, _i64p, _i32p, _f64p, _i64p, _i32p, _f64p,
                                        _f64p, _f64p, _f64p]
    lib.dlmpc_dist_alloc.argtypes = [vp, C.c_int, _P(vp)]
    lib.dlmpc_dist_setup.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int64, _i64p, _i64p, _i32p,
                                     _P(vp), _P(vp), _P(vp), C.c_uint32, _P(vp), _P(vp)]
    lib.dlmpc_dist_solve.argtypes = [vp, C.c_int, C.c_double, C.c_double, _i32p, _f64p]
    lib.dlmpc_multi_solve.argtypes = [_P(vp), C.c_int, C.c_int, C.c_double, C.c_double, _i32p, _f64p]
    lib.dlmpc_ipc_get.argtypes = [vp, vp]
    lib.dlmpc_ipc_open.argtypes = [vp, C.c_int, _P(vp)]
    lib.dlmpc_ipc_close.argtypes = [vp]
    _lib = lib
    return lib


def fp64_peak_tflops(device: int = 0) -> float:
    """Measured FP64 DMMA peak of `device` (TFLOP/s), for roofline fractions."""
    lib = load_library()
    out = C.c_double(0.0)
    if lib.dlmpc_fp64_peak(int(device), C.byref(out)) != 0:
        raise DeviceError("dlmpc_fp64_peak: " + lib.dlmpc_global_error().decode())
    return float(out.value)


def multi_solve(sessions, max_iters, eps_pri, eps_dual):
    """The one-GPU test of the device exchange: the ranks' sessions as slices
    of ONE cooperative launch -> (iterations, history, converged)."""
    lib = load_library()
    hs = (C.c_void_p * len(sessions))(*[s._h for s in sessions])
    hist = np.zeros(2 * max_iters)
    n = C.c_int32(0)
    rc = lib.dlmpc_multi_solve(hs, len(sessions), int(max_iters), float(eps_pri), float(eps_dual), C.byref(n),
                               hist.ctypes.data_as(_f64p))
    if rc not in (DLMPC_OK, DLMPC_NOT_CONVERGED):
        raise DeviceError(f"dlmpc_multi_solve failed ({rc}): {lib.dlmpc_last_error(sessions[0]._h).decode()}")
    k = int(n.value)
    return k, hist[:2 * k].reshape(k, 2), rc == DLMPC_OK


def ipc_handle(dev_ptr: int) -> bytes:
    lib = load_library()
    buf = C.create_string_buffer(64)
    if lib.dlmpc_ipc_get(C.c_void_p(dev_ptr), buf) != 0:
        raise DeviceError("dlmpc_ipc_get: " + lib.dlmpc_global_error().decode())
    return buf.raw


def ipc_open(handle: bytes, device: int) -> int:
    lib = load_library()
    out = C.c_void_p()
    if lib.dlmpc_ipc_open(C.create_string_buffer(handle, 64), int(device), C.byref(out)) != 0:
        raise DeviceError("dlmpc_ipc_open: " + lib.dlmpc_global_error().decode())
    return int(out.value)


def ipc_close(dev_ptr: int):
    load_library().dlmpc_ipc_close(C.c_void_p(dev_ptr))


def _ptr(a, ctype):
    if a is None:
        return None
    return a.ctypes.data_as(_P(ctype))


class DeviceSession:
    """One uploaded problem (a `dlmpc_handle`) on one GPU."""

    def __init__(self, layout, device: int = 0, grid_ctas: int = 0):
        lib = load_library()
        self.layout = L = layout
        self._keep = []

        def arr(name, dtype):
            v = getattr(L, name, None)
            if v is None:
                return None
            a = np.ascontiguousarray(v, dtype=dtype)
            self._keep.append(a)
            return a

        i32 = lambda n: _ptr(arr(n, np.int32), C.c_int32)
        i64 = lambda n: _ptr(arr(n, np.int64), C.c_int64)
        f64 = lambda n: _ptr(arr(n, np.float64), C.c_double)
        p = _Problem()
        p.n_sub, p.n_rows, p.n_cols, p.n_inputs = L.n_sub, L.n_rows, L.n_cols, L.n_inputs
        p.s_pad, p.horizon, p.exact, p.contiguous = L.s_pad, L.horizon, int(L.exact), int(L.contiguous)
        p.rho = L.rho
        p.grid_ctas = int(grid_ctas)
        p.own_sub_lo, p.own_sub_hi = L.own_sub
        p.own_col_lo, p.own_col_hi = L.own_cols
        p.row_start, p.ball_ptr = i64("row_start"), i64("ball_ptr")
        p.ball_idx, p.ball_off = i32("ball_idx"), i32("ball_off")
        p.state_start, p.state_count, p.sub_first_bad = i32("state_start"), i32("state_count"), i32("sub_first_bad")
        p.row_w, p.row_lo, p.row_hi = f64("row_w"), f64("row_lo"), f64("row_hi")
        p.col_owner, p.col_len, p.col_class, p.col_vec = i32("col_owner"), i32("col_len"), i32("col_class"), i32("col_vec")
        p.col_irow, p.col_rowbase = i32("col_irow"), i64("col_rowbase")
        p.d_pad, p.supp_col, p.supp_off, p.supp_len = L.d_pad, i32("supp_col"), i32("supp_off"), i32("supp_len")
        p.n_classes = L.n_classes
        p.class_s, p.class_n0, p.class_ldn = i32("class_s"), i32("class_n0"), i32("class_ldn")
        p.class_null_off, p.null_pool = i64("class_null_off"), f64("null_pool")
        p.n_vec, p.q_pool = L.n_vec, f64("q_pool")
        p.class_m = i32("class_m")
        if L.exact:
            p.class_g_off, p.class_p_off = i64("class_g_off"), i64("class_p_off")
            p.g_pool, p.p_pool = f64("g_pool"), f64("p_pool")
        p.m_pad, p.rhs_pool, p.ref_pos = L.m_pad, f64("rhs_pool"), i32("ref_pos")
        p.n_tiles, p.tile_cols = L.n_tiles, L.tile_cols
        p.tile_class, p.tile_first, p.tile_count, p.tile_colv = (
            i32("tile_class"), i32("tile_first"), i32("tile_count"), i32("tile_colv"))
        p.a_ptr, p.a_idx, p.a_val = i64("a_ptr"), i32("a_idx"), f64("a_val")
        p.b_ptr, p.b_idx, p.b_val = i64("b_ptr"), i32("b_idx"), f64("b_val")
        p.input_owner, p.input_local = i32("input_owner"), i32("input_local")
        p.class_ntouch, p.class_g0_off, p.g0_pool = i32("class_ntouch"), i64("class_g0_off"), f64("g0_pool")
        p.class_perm_off, p.perm_pool, p.col_pin = i64("class_perm_off"), i32("perm_pool"), i32("col_pin")
        h = C.c_void_p()
        rc = lib.dlmpc_create(C.byref(p), int(device), C.byref(h))
        self._keep = []
        if rc != DLMPC_OK:
            raise DeviceError(f"dlmpc_create failed ({rc}): {lib.dlmpc_global_error().decode()}")
        self._lib, self._h = lib, h
        self.device = int(device)
        self.n_cell = L.n_cols * L.s_pad

    # -- lifecycle --------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            self._lib.dlmpc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc, what):
        if rc in (DLMPC_OK, DLMPC_NOT_CONVERGED, DLMPC_ROW_INFEASIBLE):
            return rc
        msg = self._lib.dlmpc_last_error(self._h).decode()
        if rc == DLMPC_BAD_ARGUMENT:
            raise ValueError(f"{what}: {msg}")
        raise DeviceError(f"{what} failed ({rc}): {msg}")

    # -- entry points -----------------------------------------------------------
    def set_x(self, x):
        """Load a measured state; raises RowInfeasible like precompute_row_data."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        bad = C.c_int64(-1)
        rc = self._check(self._lib.dlmpc_set_x(self._h, _ptr(x, C.c_double), C.byref(bad)), "dlmpc_set_x")
        if rc == DLMPC_ROW_INFEASIBLE:
            raise RowInfeasible(int(bad.value))

    def solve(self, max_iters, eps_pri, eps_dual):
        """Returns (iterations, history (n x 2), converged)."""
        hist = np.zeros(2 * max_iters)
        it = C.c_int32(0)
        rc = self._check(self._lib.dlmpc_solve(self._h, int(max_iters), float(eps_pri), float(eps_dual),
                                               C.byref(it), _ptr(hist, C.c_double)), "dlmpc_solve")
        n = int(it.value)
        return n, hist[:2 * n].reshape(n, 2), rc == DLMPC_OK

    def iterate(self, n=1):
        hist = np.zeros(2 * n)
        self._check(self._lib.dlmpc_iterate(self._h, int(n), _ptr(hist, C.c_double)), "dlmpc_iterate")
        return hist.reshape(n, 2)

    def simulate(self, x0, t_sim, max_iters, eps_pri, eps_dual, warm_start=True, cold_start=True):
        """Closed loop on device. Returns dict(states, inputs, step_iterations)
        or raises NotConverged / RowInfeasible with the failing step."""
        L = self.layout
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        states = np.empty((t_sim + 1, L.n_cols))     # every row written on success
        inputs = np.empty((t_sim, L.n_inputs))
        iters = np.empty(t_sim, dtype=np.int32)
        fstep, fit = C.c_int32(-1), C.c_int32(0)
        bad = C.c_int64(-1)
        # the failing step's residual history (written on NotConverged only):
        # one buffer per session instead of a fresh 2 * max_iters array per call
        fhist = getattr(self, "_fhist", None)
        if fhist is None or fhist.size < 2 * max_iters:
            fhist = self._fhist = np.zeros(2 * max_iters)
        rc = self._check(self._lib.dlmpc_simulate(
            self._h, _ptr(x0, C.c_double), int(t_sim), int(bool(warm_start)), int(bool(cold_start)),
            int(max_iters), float(eps_pri), float(eps_dual), _ptr(states, C.c_double),
            _ptr(inputs, C.c_double), _ptr(iters, C.c_int32), C.byref(fstep), C.byref(bad),
            C.byref(fit), _ptr(fhist, C.c_double)), "dlmpc_simulate")
        if rc == DLMPC_ROW_INFEASIBLE:
            err = RowInfeasible(int(bad.value))
            err.step = int(fstep.value)
            raise err
        if rc == DLMPC_NOT_CONVERGED:
            n = int(fit.value)
            raise NotConverged([tuple(r) for r in fhist[:2 * n].reshape(n, 2)], step=int(fstep.value))
        return {"states": states, "inputs": inputs, "step_iterations": [int(v) for v in iters]}

    def simulate_device(self, x0_ptr, t_sim, max_iters, eps_pri, eps_dual, states_ptr, inputs_ptr,
                        iters_ptr, status_ptr, warm_start=True, cold_start=True):
        """Closed loop with device pointers (ints); asynchronous on the handle's stream."""
        self._check(self._lib.dlmpc_simulate_device(
            self._h, C.c_void_p(x0_ptr), int(t_sim), int(bool(warm_start)), int(bool(cold_start)),
            int(max_iters), float(eps_pri), float(eps_dual), C.c_void_p(states_ptr),
            C.c_void_p(inputs_ptr), C.c_void_p(iters_ptr), C.c_void_p(status_ptr)), "dlmpc_simulate_device")

    def get(self, which):
        L = self.layout
        n = {S_ROW: L.n_rows, X: L.n_cols, ADA: L.n_sub}.get(which, self.n_cell)
        out = np.zeros(n)
        self._check(self._lib.dlmpc_get(self._h, int(which), _ptr(out, C.c_double)), "dlmpc_get")
        return out

    def put(self, which, values):
        v = np.ascontiguousarray(values, dtype=np.float64).ravel()
        if v.size != self.n_cell:
            raise ValueError("internal-layout array has the wrong size")
        self._check(self._lib.dlmpc_put(self._h, int(which), _ptr(v, C.c_double)), "dlmpc_put")

    def audit(self, phi=None):
        """(dynamics_residual, resolve_residual, consensus_gap) of the current
        iterate; `phi` (internal layout) overrides the last iteration's φ."""
        out = np.zeros(3)
        ph = None if phi is None else np.ascontiguousarray(phi, dtype=np.float64)
        self._check(self._lib.dlmpc_audit(self._h, _ptr(ph, C.c_double), _ptr(out, C.c_double)),
                    "dlmpc_audit")
        return float(out[0]), float(out[1]), float(out[2])

    def get_cols(self, which, c0, n, out=None):
        """ψ or λ of columns [c0, c0+n) of the current iterate (internal layout)."""
        out = np.empty(n * self.layout.s_pad) if out is None else out
        self._check(self._lib.dlmpc_get_cols(self._h, int(which), int(c0), int(n), out.ctypes.data),
                    "dlmpc_get_cols")
        return out

    def put_cols(self, which, c0, n, values):
        v = np.ascontiguousarray(values, dtype=np.float64)
        self._check(self._lib.dlmpc_put_cols(self._h, int(which), int(c0), int(n), v.ctypes.data),
                    "dlmpc_put_cols")

    # -- graph-partitioned solve with the exchange on the device -----------------
    def dist_alloc(self, world):
        """Exchange state for `world` ranks -> the 7 device pointers a
        neighbour needs (ψ0, ψ1, λ0, λ1, halo counter, slot table, residual counter)."""
        out = (C.c_void_p * 7)()
        self._check(self._lib.dlmpc_dist_alloc(self._h, int(world), out), "dlmpc_dist_alloc")
        return [int(v or 0) for v in out]

    def dist_setup(self, rank, world, send_src, send_dst, send_peer, peer_bufs, halo_per_iter, all_bufs):
        """peer_bufs: per destination peer its dist_alloc pointers; all_bufs:
        per rank its dist_alloc pointers (slot table and residual counter)."""
        n_peers = len(peer_bufs)
        self._dist_keep = [np.ascontiguousarray(send_src, dtype=np.int64),
                           np.ascontiguousarray(send_dst, dtype=np.int64),
                           np.ascontiguousarray(send_peer, dtype=np.int32)]
        arr = lambda vals: (C.c_void_p * max(1, len(vals)))(*[C.c_void_p(v) for v in vals])
        psi = arr([b[k] for b in peer_bufs for k in (0, 1)])
        lam = arr([b[k] for b in peer_bufs for k in (2, 3)])
        flag = arr([b[4] for b in peer_bufs])
        slots = arr([b[5] for b in all_bufs])
        rflag = arr([b[6] for b in all_bufs])
        self._dist_ptrs = (psi, lam, flag, slots, rflag)
        src, dst, peer = self._dist_keep
        self._check(self._lib.dlmpc_dist_setup(self._h, int(rank), int(world), n_peers, int(src.size),
                                               _ptr(src, C.c_int64), _ptr(dst, C.c_int64), _ptr(peer, C.c_int32),
                                               psi, lam, flag, C.c_uint32(int(halo_per_iter)), slots, rflag),
                    "dlmpc_dist_setup")

    def dist_solve(self, max_iters, eps_pri, eps_dual):
        """One partitioned solve, exchange on the device -> (iterations, history, converged)."""
        hist = np.zeros(2 * max_iters)
        n = C.c_int32(0)
        rc = self._check(self._lib.dlmpc_dist_solve(self._h, int(max_iters), float(eps_pri), float(eps_dual),
                                                    C.byref(n), _ptr(hist, C.c_double)), "dlmpc_dist_solve")
        k = int(n.value)
        return k, hist[:2 * k].reshape(k, 2), rc == DLMPC_OK

    def set_halo(self, send_cells, recv_cells):
        """Register the partitioned path's halo cell lists (internal layout)."""
        self._send = np.ascontiguousarray(send_cells, dtype=np.int64)
        self._recv = np.ascontiguousarray(recv_cells, dtype=np.int64)
        self._check(self._lib.dlmpc_set_halo(self._h, _ptr(self._send, C.c_int64), int(self._send.size),
                                             _ptr(self._recv, C.c_int64), int(self._recv.size)),
                    "dlmpc_set_halo")

    def halo_pack(self, out_ptr):
        """Pack the current (ψ, λ) of the send cells into `out_ptr` (host or
        device address, 2*n_send doubles)."""
        self._check(self._lib.dlmpc_halo_pack(self._h, C.c_void_p(out_ptr)), "dlmpc_halo_pack")

    def halo_unpack(self, in_ptr):
        self._check(self._lib.dlmpc_halo_unpack(self._h, C.c_void_p(in_ptr)), "dlmpc_halo_unpack")

    # asynchronous forms (device buffers, enqueued on the session's stream)
    def iterate_async(self, n, resid_ptr):
        """n iterations without a stop test; the last (pri, dual) to device
        memory at `resid_ptr` (2 doubles). No host synchronisation."""
        self._check(self._lib.dlmpc_iterate_async(self._h, int(n), C.c_void_p(resid_ptr)), "dlmpc_iterate_async")

    def halo_pack_async(self, out_ptr):
        self._check(self._lib.dlmpc_halo_pack_async(self._h, C.c_void_p(out_ptr)), "dlmpc_halo_pack_async")

    def halo_unpack_async(self, in_ptr):
        self._check(self._lib.dlmpc_halo_unpack_async(self._h, C.c_void_p(in_ptr)), "dlmpc_halo_unpack_async")

    def set_stream(self, stream_ptr):
        """Run on an external CUDA stream (int handle; None = the session's
        own; 0, the legacy default stream, is passed as cudaStreamLegacy)."""
        if stream_ptr is None:
            h = None
        else:
            h = int(stream_ptr) or 1   # cudaStreamLegacy
        self._check(self._lib.dlmpc_set_stream(self._h, C.c_void_p(h)), "dlmpc_set_stream")

    def finish_step(self):
        """(u, x_next) for the loaded x after host-driven iterations."""
        u = np.zeros(self.layout.n_inputs)
        xn = np.zeros(self.layout.n_cols)
        self._check(self._lib.dlmpc_finish_step(self._h, _ptr(u, C.c_double), _ptr(xn, C.c_double)),
                    "dlmpc_finish_step")
        return u, xn

    def zero(self):
        self._check(self._lib.dlmpc_zero(self._h), "dlmpc_zero")

    def synchronize(self):
        self._check(self._lib.dlmpc_synchronize(self._h), "dlmpc_synchronize")

    @property
    def stream(self):
        return self._lib.dlmpc_stream(self._h)

    def last_timing(self):
        ms, n = C.c_float(0), C.c_int32(0)
        self._lib.dlmpc_last_timing(self._h, C.byref(ms), C.byref(n))
        return float(ms.value), int(n.value)

    def phase_times(self, reset=True):
        """Per-CTA per-phase SM cycles (profiling build), shape (grid, 16)."""
        g = self.info()["grid"]
        out = np.zeros(16 * g, dtype=np.uint64)
        self._check(self._lib.dlmpc_phase_times(self._h, out.ctypes.data_as(_P(C.c_uint64)), int(reset)),
                    "dlmpc_phase_times")
        return out.reshape(g, 16)

    def info(self):
        out = np.zeros(9, dtype=np.int64)
        self._lib.dlmpc_info(self._h, _ptr(out, C.c_int64))
        keys = ("n_rows", "n_cols", "s_pad", "n_sub", "grid", "tile_cols", "smem_bytes", "mode", "units")
        d = dict(zip(keys, (int(v) for v in out)))
        d["mode"] = ("patch", "twophase", "exact", "stream")[d["mode"]]
        fl = np.zeros(5, dtype=np.int64)
        self._lib.dlmpc_plan_flags(self._h, _ptr(fl, C.c_int64), 5)
        d.update(zip(("cache_phi", "fuse_steps", "rb_gemv", "stash_bufs", "pairs"), (int(v) for v in fl)))
        return d
