/*
 * dlmpc.h -- C ABI of the B200 DLMPC ADMM hot path (libdlmpc.so).
 *
 * This is the device boundary that replaces the reference's per-iteration
 * execution layer (L3 in SURVEY.md §1):
 *
 *   reference interface                                   replaced by
 *   ---------------------------------------------------   ---------------------------
 *   admm_solve loop          admm.py:315-347              dlmpc_solve
 *   Executor.run_iteration   strategies.py:249-260        dlmpc_iterate
 *   precompute_row_data      sls_core.py:330-349          dlmpc_set_x
 *   PhiTriple (state arrays) sls_core.py:415-438          dlmpc_get / dlmpc_put / dlmpc_zero
 *   AdmmWorkspace.__init__   admm.py:106-127              dlmpc_create
 *   dlmpc_simulate loop      admm.py:486-520              dlmpc_simulate
 *   extract_control          admm.py:350-360              (inside dlmpc_simulate)
 *   step_dynamics            admm.py:363-369              (inside dlmpc_simulate)
 *
 * All pointers in the structs below are HOST pointers that must stay valid
 * only for the duration of the call; the library copies what it needs into
 * device memory it owns. No torch types cross this boundary. A handle is
 * bound to one device and one CUDA stream and is not thread-safe.
 *
 * Status codes map one to one to the Python exceptions of errors.py
 * (reference errors.py:8-62): DLMPC_NOT_CONVERGED -> NotConverged,
 * DLMPC_ROW_INFEASIBLE -> RowInfeasible; every other nonzero code is a
 * DeviceError / ValueError with dlmpc_last_error() text.
 */
#ifndef DLMPC_H
#define DLMPC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  DLMPC_OK = 0,
  DLMPC_NOT_CONVERGED = 1,   /* iteration cap reached (admm.py:342-343)        */
  DLMPC_ROW_INFEASIBLE = 2,  /* zero state on a row whose bounds exclude zero  */
  DLMPC_BAD_ARGUMENT = 3,
  DLMPC_CUDA_ERROR = 4,
  DLMPC_NO_DEVICE = 5
};

/* which array dlmpc_get/dlmpc_put address (internal column layout, n_cols x s_pad) */
enum {
  DLMPC_PSI = 0,       /* ψ, current iterate                          */
  DLMPC_LAM = 1,       /* λ, current iterate                          */
  DLMPC_PSI_PREV = 2,  /* ψ before the last iteration (psi_prev_c)    */
  DLMPC_PHI = 3,       /* φ of the last iteration (phi_c)             */
  DLMPC_LAM_PREV = 4,  /* λ before the last iteration                 */
  DLMPC_S_ROW = 5,     /* per-row Φ scale of the last iteration (n_rows, internal order) */
  DLMPC_X = 6,         /* measured state currently loaded (n_x)       */
  DLMPC_ADA = 7        /* per-subsystem ||a||^2 for the loaded state  */
};

/*
 * Problem description. Internal layouts (built by devlayout.py):
 *  - rows are grouped by owning subsystem: subsystem i owns internal rows
 *    [row_start[i], row_start[i+1]) in ascending reference-row order;
 *  - column c (= global state c, owner col_owner[c]) stores its support as
 *    the concatenation, over ball members i of the owner (ascending), of the
 *    rows of i; entry (row of i with local index l, column c) lives at
 *    c*s_pad + ball_off[e] + l where e is the (i -> owner) edge of the ball CSR;
 *  - the Ψ operator of every column class is stored padded for the FP64
 *    tensor-core fragments (see devlayout.py).
 */
typedef struct dlmpc_problem {
  int32_t n_sub, n_rows, n_cols, n_inputs, s_pad, horizon;
  int32_t exact;          /* 1: reference arithmetic bit for bit; 0: fast path  */
  int32_t contiguous;     /* 1: every ball is a contiguous id range (chains)    */
  /* owned range for graph-partitioned runs: only these subsystems / columns
   * are solved (and enter the residuals); the rest is a read-only halo.
   * own_sub_hi <= own_sub_lo means "everything". */
  int32_t own_sub_lo, own_sub_hi, own_col_lo, own_col_hi;
  double rho;
  /* subsystems */
  const int64_t* row_start;      /* [n_sub+1] */
  const int64_t* ball_ptr;       /* [n_sub+1] */
  const int32_t* ball_idx;       /* [nnz_ball] ascending per node            */
  const int32_t* ball_off;       /* [nnz_ball] offset of node i's rows inside column support of ball_idx[e] */
  const int32_t* state_start;    /* [n_sub] */
  const int32_t* state_count;    /* [n_sub] */
  const int32_t* sub_first_bad;  /* [n_sub] lowest reference row of the node whose bounds exclude 0, or -1 */
  int32_t d_pad;                 /* padded row-support length (>= max supp_len)  */
  const int32_t* supp_col;       /* [n_sub*d_pad] row-support columns, ascending  */
  const int32_t* supp_off;       /* [n_sub*d_pad] block offset of the node's rows in each of those columns */
  const int32_t* supp_len;       /* [n_sub] row-support length (= d_row of the node's rows) */
  /* rows, internal order */
  const double* row_w;           /* [n_rows] */
  const double* row_lo;
  const double* row_hi;
  /* columns */
  const int32_t* col_owner;      /* [n_cols] */
  const int32_t* col_len;        /* [n_cols] */
  const int32_t* col_class;      /* [n_cols] */
  const int32_t* col_vec;        /* [n_cols] index into q_pool / rhs_pool */
  const int32_t* col_irow;       /* [n_sub*s_pad] internal row per support slot (NULL if contiguous) */
  const int64_t* col_rowbase;    /* [n_cols] internal row of support slot 0 (contiguous supports) */
  /* column classes (fast path operators) */
  int32_t n_classes;
  const int32_t* class_s;        /* [n_classes] support length                   */
  const int32_t* class_n0;       /* null-space dimension                         */
  const int32_t* class_ldn;      /* leading dimension of the padded operator     */
  const int64_t* class_null_off; /* [n_classes+1] offsets (doubles) into null_pool */
  const double* null_pool;       /* per class: [round8(s) x ldn], zero padded     */
  int32_t n_vec;
  const double* q_pool;          /* [n_vec x s_pad] particular solutions          */
  /* exact path operators (reference support order) */
  const int32_t* class_m;        /* rows of the reduced operator g               */
  const int64_t* class_g_off;    /* [n_classes+1] offsets into g_pool ([m x s])   */
  const int64_t* class_p_off;    /* [n_classes+1] offsets into p_pool ([s x m])   */
  const double* g_pool;
  const double* p_pool;
  int32_t m_pad;
  const double* rhs_pool;        /* [n_vec x m_pad] reduced rhs                   */
  const int32_t* ref_pos;        /* [n_sub*s_pad] internal slot of reference slot p */
  /* tiles of the column stage */
  int32_t n_tiles, tile_cols;    /* tile_cols in {8,16}                           */
  const int32_t* tile_class;     /* [n_tiles] */
  const int32_t* tile_first;     /* [n_tiles] first index into tile_colv          */
  const int32_t* tile_count;     /* [n_tiles] */
  const int32_t* tile_colv;      /* [n_cols] columns sorted by class              */
  /* plant (CSR, reference column order) for the on-device closed loop */
  const int64_t* a_ptr; const int32_t* a_idx; const double* a_val;   /* n_cols rows  */
  const int64_t* b_ptr; const int32_t* b_idx; const double* b_val;   /* n_cols rows  */
  const int32_t* input_owner;    /* [n_inputs] */
  const int32_t* input_local;    /* [n_inputs] local row index of input k at t=0 */
  /* audit (optional, NULL disables dlmpc_audit): per class the touched-rows
   * operator g0 [ntouch x s] in reference support order and the support
   * permutation (reference slot -> internal slot); per column the rhs0 pin */
  const int32_t* class_ntouch;
  const int64_t* class_g0_off;   /* [n_classes+1] */
  const double* g0_pool;
  const int64_t* class_perm_off; /* [n_classes+1] */
  const int32_t* perm_pool;
  const int32_t* col_pin;        /* [n_cols] row of rhs0 = 1 among the touched rows, -1 if none */
  /* CTAs of the persistent kernel (0: one per SM). The one-GPU test of the
   * device-side exchange runs the ranks of a partitioned solve as slices of
   * one cooperative grid (dlmpc_multi_solve), so each rank plans for its slice. */
  int32_t grid_ctas;
} dlmpc_problem;

typedef struct dlmpc_handle dlmpc_handle;

/* Upload a problem and allocate all device state (zeroed). */
int dlmpc_create(const dlmpc_problem* prob, int device, dlmpc_handle** out);
void dlmpc_destroy(dlmpc_handle* h);
const char* dlmpc_last_error(const dlmpc_handle* h);
/* Library-wide error text for failures before a handle exists. */
const char* dlmpc_global_error(void);

/* Load a measured state: ||a||^2 per subsystem on device and the row
 * feasibility check of sls_core.py:346-348. *bad_row = first infeasible
 * reference row or -1; returns DLMPC_ROW_INFEASIBLE in that case. */
int dlmpc_set_x(dlmpc_handle* h, const double* x, int64_t* bad_row);

/* ADMM from the current iterate until both residuals are within tolerance
 * (admm.py:336-343). hist receives 2*iters doubles (pri, dual). */
int dlmpc_solve(dlmpc_handle* h, int max_iters, double eps_pri, double eps_dual,
                int* iters, double* hist);

/* Exactly n iterations, no convergence stop (Executor.run_iteration x n). */
int dlmpc_iterate(dlmpc_handle* h, int n, double* hist);

/* Closed loop of t_sim MPC steps fully on device (admm.py:486-520):
 * row data, solve, control extraction and plant step per step in one
 * persistent launch. states: (t_sim+1) x n_cols, inputs: t_sim x n_inputs,
 * step_iters: t_sim. On failure *fail_step is the step, *bad_row the row
 * (RowInfeasible) and fail_hist receives the failing step's history
 * (2*max_iters doubles, *fail_iters entries valid). cold_start zeroes the
 * iterate first (a fresh PhiTriple, admm.py:466). */
int dlmpc_simulate(dlmpc_handle* h, const double* x0, int t_sim, int warm_start, int cold_start,
                   int max_iters, double eps_pri, double eps_dual,
                   double* states, double* inputs, int* step_iters,
                   int* fail_step, int64_t* bad_row, int* fail_iters, double* fail_hist);

/* Same closed loop with x0 and all outputs already in device memory
 * (device pointers); nothing is copied and the call does not synchronise. */
int dlmpc_simulate_device(dlmpc_handle* h, const double* x0_dev, int t_sim, int warm_start,
                          int cold_start, int max_iters, double eps_pri, double eps_dual,
                          double* states_dev, double* inputs_dev, int* step_iters_dev,
                          int* status_dev);

/* Fixed-point audit of the current iterate (reference verify_fixed_point,
 * admm.py:417-434): out[0] dynamics residual max|g0 ψ - rhs0|, out[1]
 * re-solve residual max|Φ(current duals) - φ|, out[2] consensus gap
 * max|φ - ψ|. φ is the last iteration's (phi_host == NULL) or a caller's
 * φ in internal layout. Needs the audit tables of dlmpc_problem. */
int dlmpc_audit(dlmpc_handle* h, const double* phi_host, double* out3);

/* Column ranges of the current ψ / λ (internal layout, host or device
 * pointers): the per-iteration halo exchange of the partitioned path. */
int dlmpc_get_cols(dlmpc_handle* h, int which, int c0, int n, double* dst);
int dlmpc_put_cols(dlmpc_handle* h, int which, int c0, int n, const double* src);

/* Halo exchange of the partitioned path (one rank's sub-problem): register
 * the internal cells this rank sends (concatenated over destination ranks)
 * and receives (over source ranks) once, then every iteration pack the
 * current (ψ, λ) of the send cells into `out` [2*n_send doubles, pairs
 * interleaved] and unpack a received message `in` [2*n_recv] into the halo
 * cells. Pointers may be host or device memory; both calls synchronise.
 * Replaces the reference's shared-memory triple, which every worker reads
 * in place (admm.py:186-253: there is no exchange on one host). */
int dlmpc_set_halo(dlmpc_handle* h, const int64_t* send_cells, int64_t n_send,
                   const int64_t* recv_cells, int64_t n_recv);
int dlmpc_halo_pack(dlmpc_handle* h, double* out);
int dlmpc_halo_unpack(dlmpc_handle* h, const double* in);

/* Asynchronous forms for the multi-GPU driver (all enqueued on the handle's
 * stream, no host synchronisation): n host-driven iterations without a stop
 * test, the last iteration's (pri, dual) maxima copied to resid_dev (2
 * doubles, device memory); pack / unpack of the halo with device buffers.
 * Replace the per-iteration round trips of dlmpc_iterate / dlmpc_halo_pack /
 * dlmpc_halo_unpack (reference: the coordinator's run_iteration ->
 * reduce_convergence, strategies.py:178-183, 249-260). */
int dlmpc_iterate_async(dlmpc_handle* h, int n, double* resid_dev);
int dlmpc_halo_pack_async(dlmpc_handle* h, double* out_dev);
int dlmpc_halo_unpack_async(dlmpc_handle* h, const double* in_dev);
/* Run the handle's work on an external CUDA stream (e.g. the framework's
 * current stream, so its collectives order against the kernels); NULL
 * restores the handle's own stream. Synchronises the previous stream. */
int dlmpc_set_stream(dlmpc_handle* h, void* stream);

/* After host-driven iterations: control extraction (admm.py:350-360) and
 * plant step (admm.py:363-369) for the loaded x; u_out [n_inputs],
 * x_next_out [n_cols] (valid for owned states). */
int dlmpc_finish_step(dlmpc_handle* h, double* u_out, double* x_next_out);

/* Copy an internal-layout array to/from host memory. */
int dlmpc_get(dlmpc_handle* h, int which, double* dst);
int dlmpc_put(dlmpc_handle* h, int which, const double* src);
int dlmpc_zero(dlmpc_handle* h);

/* Device time (ms, CUDA events on the handle's stream) of the last
 * solve / iterate / simulate launch, and the number of kernels it launched. */
int dlmpc_last_timing(const dlmpc_handle* h, float* ms, int* launches);
/* The CUDA stream of the handle (cudaStream_t as void*). */
void* dlmpc_stream(dlmpc_handle* h);
int dlmpc_synchronize(dlmpc_handle* h);
/* Per-CTA per-phase device nanoseconds accumulated by a profiling build
 * (-DDLMPC_PHASE_TIMING; zeros otherwise): out[grid*16] SM cycles; reset
 * clears them. Per iteration: 0 Φ, 1 Ψ prologue, 2 GEMM 1, 3 GEMM 2,
 * 4 epilogue, 5 residual publish, 6 grid barrier, 7 stop test; per MPC step:
 * 8 row data + barrier, 9 Φ metadata cache, 10 control + plant, 11 barrier. */
int dlmpc_phase_times(dlmpc_handle* h, uint64_t* out, int reset);
/* Shape info: n_rows, n_cols, s_pad, n_sub, grid CTAs, tile_cols, smem bytes,
 * kernel mode (0 patch, 1 two-phase, 2 exact, 3 stream), work units. */
int dlmpc_info(const dlmpc_handle* h, int64_t* out9);
/* Kernel plan flags, the first n of: Φ metadata cached per CTA, fused
 * MPC-step transitions (closed loops), register-blocked GEMV pair, ψ/λ
 * staging buffers, K-split CTA pairs. No reference counterpart. */
int dlmpc_plan_flags(const dlmpc_handle* h, int64_t* out, int n);

/* ------------------------------------------------------------------------
 * The reference's device schedules (strategies.py:44-314: naive, padded,
 * fused, patch-local), executed on the GPU over the reference's own dual
 * padded layout (sls_core.py:352-518) with the reference's arithmetic bit for
 * bit. The host (strategies.Executor) drives one iteration as the reference's
 * coordinator does; every stage is one kernel launch on the handle's stream,
 * dlmpc_sched_sync is a host sync and dlmpc_sched_read_residuals the flag
 * read, so the reference's SyncLedger counts real events.
 * ---------------------------------------------------------------------- */
typedef struct dlmpc_sched dlmpc_sched;

typedef struct dlmpc_sched_problem {
  int32_t n_rows, n_cols, d_row, d_col;
  int64_t n_elems;
  double rho;
  const int32_t* row_len;        /* [n_rows]  LayoutTables.row_len                     */
  const int32_t* col_len;        /* [n_cols]  LayoutTables.col_len                     */
  const int64_t* rs;             /* [n_rows*d_row] column of each row slot, -1 past the support */
  const int64_t* c2r_flat;       /* [n_cols*d_col] row-layout twin, -1 past the support */
  const int64_t* r2c_flat;       /* [n_rows*d_row] column-layout twin, -1 past the support */
  const int64_t* elem_flat_col;  /* [n_elems] valid column-layout cells                */
  int32_t n_classes;
  const int32_t* col_class;      /* [n_cols] operator class                           */
  const int32_t* class_m;        /* [n_classes] constraint rows                       */
  const int32_t* class_s;        /* [n_classes] support length                        */
  const int64_t* class_g_off; const double* g_pool;   /* g [m x s] per class           */
  const int64_t* class_p_off; const double* p_pool;   /* projector [s x m] per class   */
  const int64_t* col_rhs_off; const double* rhs_pool; /* [n_cols+1] offsets, rhs [m]   */
  int64_t n_patch;               /* 0: no patch tables (patch-local unavailable)      */
  const int64_t* patch_off;      /* [n_cols+1] (admm.py:139-151)                      */
  const int64_t* patch_rows;     /* member rows of each column patch                  */
  const int32_t* patch_slot;     /* the column's slot in each member row               */
  const int32_t* patch_owned;    /* 1: the column publishes the row (owner_col)        */
  const double* row_w; const double* row_lo; const double* row_hi;   /* [n_rows] or NULL (put later) */
} dlmpc_sched_problem;

enum {   /* arrays of dlmpc_sched_get / dlmpc_sched_put */
  DLMPC_SCHED_PHI_R = 0, DLMPC_SCHED_PSI_R = 1, DLMPC_SCHED_LAM_R = 2, DLMPC_SCHED_PHI_C = 3,
  DLMPC_SCHED_PSI_C = 4, DLMPC_SCHED_LAM_C = 5, DLMPC_SCHED_PSI_PREV_C = 6, DLMPC_SCHED_PRI_C = 7,
  DLMPC_SCHED_DUAL_C = 8, DLMPC_SCHED_A_PAD = 9, DLMPC_SCHED_ADA = 10, DLMPC_SCHED_ROW_W = 11,
  DLMPC_SCHED_ROW_LO = 12, DLMPC_SCHED_ROW_HI = 13   /* row data of the current step (RowData) */
};

enum {   /* stage kernels of dlmpc_sched_stage (AdmmWorkspace, admm.py:153-270) */
  DLMPC_STAGE_PHI_ROWS = 0,          /* phi_rows, exact-size items (naive)             */
  DLMPC_STAGE_PHI_ROWS_PADDED = 1,   /* phi_rows, longest-vector items (padded)        */
  DLMPC_STAGE_EXCHANGE_PHI = 2,      /* exchange_phi_to_col                            */
  DLMPC_STAGE_PSI_COLS = 3,          /* psi_cols                                       */
  DLMPC_STAGE_LAMBDA_COLS = 4,       /* lambda_cols                                    */
  DLMPC_STAGE_LAMBDA_ELEMS = 5,      /* lambda_elems                                   */
  DLMPC_STAGE_CONV_COLS = 6,         /* conv_cols (+ the global maxima)                */
  DLMPC_STAGE_EXCHANGE_PSI_LAM = 7,  /* exchange_psi_lam_to_row                        */
  DLMPC_STAGE_FUSED_COLS = 8,        /* fused_cols (paper §III-C)                      */
  DLMPC_STAGE_PATCH_COLS = 9,        /* patch_cols (paper §III-D)                      */
  DLMPC_STAGE_PATCH_COLS_PADDED = 10
};

int dlmpc_sched_create(const dlmpc_sched_problem* prob, int device, dlmpc_sched** out);
void dlmpc_sched_destroy(dlmpc_sched* h);
const char* dlmpc_sched_last_error(const dlmpc_sched* h);
int dlmpc_sched_put(dlmpc_sched* h, int which, const double* src);
int dlmpc_sched_get(dlmpc_sched* h, int which, double* dst);
/* precompute_row_data (sls_core.py:330-349) on device: a_pad, ||a||^2 for x;
 * DLMPC_ROW_INFEASIBLE with *bad_row = the lowest infeasible row */
int dlmpc_sched_set_x(dlmpc_sched* h, const double* x, int64_t n_x, int64_t* bad_row);
/* one stage launch over items [lo, hi) (rows, columns or elements), async */
int dlmpc_sched_stage(dlmpc_sched* h, int stage, int64_t lo, int64_t hi);
int dlmpc_sched_sync(dlmpc_sched* h);
/* the reduced (pri, dual) of the residual stages since the last read
 * (reduce_residuals, admm.py:269-270); resets the maxima */
int dlmpc_sched_read_residuals(dlmpc_sched* h, double* pri_dual);
/* AdmmWorkspace._phi_compute (admm.py:155-166): rows [lo, hi) into out, state untouched */
int dlmpc_sched_phi_compute(dlmpc_sched* h, int64_t lo, int64_t hi, double* out);
/* swap_row_buffers (admm.py:255-259): the patch scatter's buffers become current */
int dlmpc_sched_swap_rows(dlmpc_sched* h);

/* The reference's scalar stage functions as device operators over n
 * independent items (host pointers, synchronous):
 *   dlmpc_op_phi_rows     phi_row_solve     admm.py:28-51   (items of length len[i], stride d)
 *   dlmpc_op_psi_cols     psi_column_solve  admm.py:54-60   (per item g [m x s], P [s x m], rhs [m], k [s])
 *   dlmpc_op_lambda       lambda_update     admm.py:63-67
 *   dlmpc_op_residuals    column_residuals  admm.py:69-74   (out2: pri, dual per item)
 *   dlmpc_op_row_dots     extract_control   admm.py:350-360 (ascending gather-dots)
 *   dlmpc_op_plant_step   step_dynamics     admm.py:363-369 (CSR A x + B u, scipy's order) */
int dlmpc_op_phi_rows(int device, int n, int d, const int32_t* len, const double* a, const double* v,
                      const double* ada, const double* w, const double* lo, const double* hi, double rho,
                      double* out);
int dlmpc_op_psi_cols(int device, int n, int m, int s, const double* g, const double* P, const double* rhs,
                      const double* k, double* out);
int dlmpc_op_lambda(int device, int64_t n, const double* lam, const double* phi, const double* psi, double* out);
int dlmpc_op_residuals(int device, int n, int d, const int32_t* len, const double* phi, const double* psi,
                       const double* prev, double rho, double* out2);
int dlmpc_op_row_dots(int device, int n, int d, const int32_t* len, const double* vals, const int64_t* idx,
                      int64_t n_x, const double* x, double* out);
int dlmpc_op_plant_step(int device, int n_x, int n_u, const int64_t* a_ptr, const int32_t* a_idx,
                        const double* a_val, const int64_t* b_ptr, const int32_t* b_idx, const double* b_val,
                        const double* x, const double* u, double* out);

/* ------------------------------------------------------------------------
 * Graph-partitioned solve with the exchange ON THE DEVICE (replaces the
 * host-driven per-iteration pack / send-recv / unpack / all-reduce of
 * dlmpc_iterate_async + dlmpc_halo_*; reference: there is no exchange on one
 * host, admm.py:186-253 and strategies.py:178-183). Each rank's persistent
 * kernel stores the halo cells its neighbours read straight into their ψ/λ
 * buffers (peer pointers: NVLink P2P via the IPC helpers below, or the same
 * device), bumps their arrival counters, posts its residual maxima into
 * every rank's slot table and waits for its neighbours -- one launch per
 * solve, no host involvement per iteration, the same global stop decision on
 * every rank. Non-patch kernel modes (stream, two-phase, exact).
 * ---------------------------------------------------------------------- */
/* Allocate the exchange state of a handle for `world` ranks and return the
 * device pointers a neighbour needs: out[0..6] = ψ buffer 0, ψ buffer 1,
 * λ buffer 0, λ buffer 1, halo arrival counter, residual slot table,
 * residual arrival counter. */
int dlmpc_dist_alloc(dlmpc_handle* h, int world, void** out7);
/* Wire the exchange: this rank's send list (local cells, destination cells,
 * destination peer index per entry), per peer its ψ/λ buffers (2 each) and
 * arrival counter, per rank its slot table and residual counter, and how
 * many counter increments per iteration this rank receives (the CTAs of all
 * its sending neighbours). Pointers are device addresses (peer or local). */
int dlmpc_dist_setup(dlmpc_handle* h, int rank, int world, int n_peers, int64_t n_send,
                     const int64_t* send_src, const int64_t* send_dst, const int32_t* send_peer,
                     void* const* peer_psi, void* const* peer_lam, void* const* peer_flag,
                     uint32_t halo_per_iter, void* const* all_slots, void* const* all_rflag);
/* One partitioned solve (every rank calls it; ranks on different GPUs run
 * concurrently). Same results as dlmpc_solve: iterations, global history. */
int dlmpc_dist_solve(dlmpc_handle* h, int max_iters, double eps_pri, double eps_dual, int* iters, double* hist);
/* The one-GPU test: the n ranks' handles (same device, same kernel mode)
 * as slices of ONE cooperative launch; iters / hist as dlmpc_dist_solve. */
int dlmpc_multi_solve(dlmpc_handle* const* hs, int n, int max_iters, double eps_pri, double eps_dual,
                      int* iters, double* hist);
/* CUDA IPC of device allocations for the multi-process exchange (64-byte
 * handles). */
int dlmpc_ipc_get(const void* dev_ptr, void* handle64);
int dlmpc_ipc_open(const void* handle64, int device, void** dev_ptr);
int dlmpc_ipc_close(void* dev_ptr);

/* Measured FP64 tensor-core (DMMA m8n8k4) peak of `device` in TFLOP/s: the
 * denominator of bench.py's FP64 roofline fraction (no reference counterpart;
 * MEASURED_PEAKS.json has HBM and bf16 only). */
int dlmpc_fp64_peak(int device, double* tflops);

#ifdef __cplusplus
}
#endif
#endif /* DLMPC_H */
