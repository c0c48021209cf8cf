// dlmpc_schedules.cuh -- the reference's four device schedules, executed on
// the B200 (included by dlmpc.cu; C ABI `dlmpc_sched_*` / `dlmpc_op_*` in
// include/dlmpc.h).
//
// The reference (strategies.py:44-314) MODELS the paper's GPU schemes as CPU
// thread-pool schedules over the dual padded layout (sls_core.py:415-518):
//
//   naive / padded  4 stage launches and 4 host syncs per iteration:
//                   Φ rows | exchange | Ψ columns | Λ elements | residuals |
//                   exchange (strategies.py:283-296); naive items loop over
//                   their exact support length, padded ones over the longest
//                   vector (the paper's §III-B)
//   fused           Φ launch, host sync, exchange, one combined column launch
//                   (Ψ + Λ + residuals + scatter to rows), flag read (§III-C)
//   patch-local     one launch: every column recomputes Φ of its support rows
//                   (duplicated work), publishes the rows it owns, then Ψ, Λ,
//                   residuals and a scatter into the alternate row buffers;
//                   pointer swap; flag read (§III-D)
//
// Here those schedules run for real: every stage is a kernel launch on the
// handle's stream, every host sync a stream synchronisation, every flag read
// a 16-byte device->host read of the residual pair, so the reference's
// SyncLedger counts real events. The state is the reference's own layout
// (φ, ψ, λ row- and column-major, padding exactly zero) and the arithmetic is
// the reference's bit for bit: ascending Φ dots, numpy pairwise Ψ sums, no
// FMA -- every schedule reproduces the reference's iterates exactly.
//
// The production path is the persistent kernel (dlmpc_device.cuh); these
// schedules are the drop-in for the reference's ExecStrategy variants and the
// B200 measurement of the paper's scheme comparison.
#pragma once

namespace dlmpc {
namespace sched {

struct RefDev {
  int n_rows, n_cols, d_row, d_col;
  long long n_elems;
  double rho;
  const int* row_len; const int* col_len;
  const long long* rs;          // [n_rows*d_row] column of row slot k, -1 past the support
  const long long* c2r;         // [n_cols*d_col] flat row-layout twin, -1 past the support
  const long long* r2c;         // [n_rows*d_row] flat column-layout twin, -1 past the support
  const long long* elem_flat;   // [n_elems] valid column-layout cells
  const int* col_class; const int* class_m;
  const long long* g_off; const double* g_pool;   // per class g [m x s], s = the column's support length
  const long long* p_off; const double* p_pool;   // per class projector [s x m]
  const long long* rhs_off; const double* rhs_pool;   // per column rhs [m]
  const long long* patch_off;   // [n_cols+1] into patch_rows (patch-local)
  const long long* patch_rows;  // member rows of each column's patch (its support rows)
  const int* patch_slot;        // the column's slot inside each member row
  const int* patch_owned;       // 1: the column publishes that row (its canonical owner)
  // iterates (reference padded layouts) and per-step row data
  double* phi_r; double* psi_r; double* lam_r; double* psi_r_nx; double* lam_r_nx;
  double* phi_c; double* psi_c; double* lam_c; double* prev_c; double* pri_c; double* dual_c;
  double* a_pad; double* ada; double* w; double* lo; double* hi;   // row data of the current step
  unsigned long long* resid;    // [2] residual maxima (ordered bits, NaN wins)
  int* bad;                     // RowInfeasible: lowest infeasible row
};

// np.clip semantics (NaN propagates)
__device__ __forceinline__ double clip_nan(double y0, double lo, double hi) {
  return y0 != y0 ? y0 : fmin(fmax(y0, lo), hi);
}

// One row's Φ (AdmmWorkspace._phi_compute, admm.py:155-166) for the whole
// padded width: v = ψ - λ, c = ascending_dot(v, a) (sls_core.py:37-47),
// y0 = ρc / (ρ + 2w‖a‖²), y = clip(y0, lo, hi), scale = (y - c)/‖a‖² (0 when
// ‖a‖² = 0), out = v + scale·a. PADDED: the dot walks all d_row slots (the
// longest vector, §III-B); otherwise the row's own length, then the padding's
// +0 products as one +0 (bitwise the same sum).
template <bool PADDED, class Out>
__device__ __forceinline__ void phi_row(const RefDev& R, long long r, const double* psi_r, const double* lam_r,
                                        const Out& out) {
  const int D = R.d_row;
  const int n = PADDED ? D : R.row_len[r];
  const double* a = R.a_pad + r * D;
  const double* ps = psi_r + r * D;
  const double* lm = lam_r + r * D;
  double c = 0.0;
  for (int j = 0; j < n; ++j) {
    const double p = __dmul_rn(__dsub_rn(ps[j], lm[j]), a[j]);
    c = j == 0 ? p : __dadd_rn(c, p);
  }
  if (!PADDED && n < D) c = n == 0 ? 0.0 : __dadd_rn(c, 0.0);
  const double ada = R.ada[r];
  const double den = __dadd_rn(R.rho, __dmul_rn(__dmul_rn(2.0, R.w[r]), ada));
  const double y = clip_nan(__ddiv_rn(__dmul_rn(R.rho, c), den), R.lo[r], R.hi[r]);
  const double scale = ada > 0.0 ? __ddiv_rn(__dsub_rn(y, c), ada) : 0.0;
  for (int j = 0; j < D; ++j) out(j, __dadd_rn(__dsub_rn(ps[j], lm[j]), __dmul_rn(scale, a[j])));
}

template <bool PADDED>
__global__ void phi_rows_kernel(RefDev R, long long lo, long long hi, double* dst) {
  for (long long r = lo + blockIdx.x * (long long)blockDim.x + threadIdx.x; r < hi;
       r += (long long)gridDim.x * blockDim.x) {
    double* o = (dst ? dst : R.phi_r) + r * R.d_row;
    phi_row<PADDED>(R, r, R.psi_r, R.lam_r, [o](int j, double v) { o[j] = v; });
  }
}

// φ_c = φ_r.flat[c2r] (sls_core.py:442-446); padding 0
__global__ void exchange_phi_kernel(RefDev R) {
  const long long n = (long long)R.n_cols * R.d_col;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
    const long long s = R.c2r[q];
    R.phi_c[q] = s >= 0 ? R.phi_r[s] : 0.0;
  }
}

// ψ_r, λ_r = ψ_c, λ_c gathered by r2c (sls_core.py:448-456)
__global__ void exchange_psi_lam_kernel(RefDev R) {
  const long long n = (long long)R.n_rows * R.d_row;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
    const long long s = R.r2c[q];
    R.psi_r[q] = s >= 0 ? R.psi_c[s] : 0.0;
    R.lam_r[q] = s >= 0 ? R.lam_c[s] : 0.0;
  }
}

// Ψ of column c by one block (admm.py:174-186): k = φ + λ; r = rhs - Σpw g∘k
// (per constraint row, numpy pairwise over the support); ψ_prev ← ψ;
// ψ = k + Σpw P∘r. `sm`: k [s] then r [m].
__device__ void psi_column(const RefDev& R, int c, double* sm) {
  const int s = R.col_len[c];
  const int cls = R.col_class[c];
  const int m = R.class_m[cls];
  const double* g = R.g_pool + R.g_off[cls];
  const double* P = R.p_pool + R.p_off[cls];
  const double* rhs = R.rhs_pool + R.rhs_off[c];
  double* k = sm;
  double* res = sm + s;
  const long long base = (long long)c * R.d_col;
  for (int j = threadIdx.x; j < s; j += blockDim.x) k[j] = __dadd_rn(R.phi_c[base + j], R.lam_c[base + j]);
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x)
    res[i] = __dsub_rn(rhs[i], pairwise_sum(ProdRow{g + (size_t)i * s, k}, 0, s));
  __syncthreads();
  for (int j = threadIdx.x; j < s; j += blockDim.x) {
    R.prev_c[base + j] = R.psi_c[base + j];
    R.psi_c[base + j] = __dadd_rn(k[j], pairwise_sum(ProdRow{P + (size_t)j * m, res}, 0, m));
  }
  __syncthreads();
}

// λ_c += φ_c - ψ_c over the whole padded column (admm.py:205-207)
__device__ __forceinline__ void lambda_column(const RefDev& R, int c) {
  const long long base = (long long)c * R.d_col;
  for (int j = threadIdx.x; j < R.d_col; j += blockDim.x)
    R.lam_c[base + j] = __dadd_rn(R.lam_c[base + j], __dsub_rn(R.phi_c[base + j], R.psi_c[base + j]));
}

// pri_c = max|φ - ψ|, dual_c = ρ·max|ψ - ψ_prev| over the padded column
// (admm.py:214-217), and the global maxima (reduce_residuals, 269-270) by an
// ordered-bit atomicMax (NaN wins, as np.max). One block per column.
__device__ void conv_column(const RefDev& R, int c, double* red) {
  const long long base = (long long)c * R.d_col;
  double p = 0.0, d = 0.0;
  for (int j = threadIdx.x; j < R.d_col; j += blockDim.x) {
    p = rmax(p, __dsub_rn(R.phi_c[base + j], R.psi_c[base + j]));
    d = rmax(d, __dsub_rn(R.psi_c[base + j], R.prev_c[base + j]));
  }
  for (int o = 16; o > 0; o >>= 1) {
    p = rmax(p, __shfl_xor_sync(0xffffffffu, p, o));
    d = rmax(d, __shfl_xor_sync(0xffffffffu, d, o));
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) { red[2 * warp] = p; red[2 * warp + 1] = d; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < nw; ++q) { p = rmax(p, red[2 * q]); d = rmax(d, red[2 * q + 1]); }
    const double dual = __dmul_rn(R.rho, d);
    R.pri_c[c] = p;
    R.dual_c[c] = dual;
    atomicMax(R.resid, static_cast<unsigned long long>(__double_as_longlong(p) & 0x7fffffffffffffffLL));
    atomicMax(R.resid + 1, static_cast<unsigned long long>(__double_as_longlong(dual) & 0x7fffffffffffffffLL));
  }
  __syncthreads();
}

// scatter of one column's ψ, λ into a row layout (sls_core.py:458-472)
__device__ __forceinline__ void scatter_column(const RefDev& R, int c, double* psi_dst, double* lam_dst) {
  const long long base = (long long)c * R.d_col;
  for (int j = threadIdx.x; j < R.col_len[c]; j += blockDim.x) {
    const long long t = R.c2r[base + j];
    psi_dst[t] = R.psi_c[base + j];
    lam_dst[t] = R.lam_c[base + j];
  }
}

__global__ void psi_cols_kernel(RefDev R, int lo, int hi) {
  extern __shared__ double sm[];
  for (int c = lo + blockIdx.x; c < hi; c += gridDim.x) psi_column(R, c, sm);
}

__global__ void lambda_cols_kernel(RefDev R, int lo, int hi) {
  for (int c = lo + blockIdx.x; c < hi; c += gridDim.x) lambda_column(R, c);
}

// element-parallel Λ over the valid cells (admm.py:209-212, naive/padded)
__global__ void lambda_elems_kernel(RefDev R, long long lo, long long hi) {
  for (long long e = lo + blockIdx.x * (long long)blockDim.x + threadIdx.x; e < hi;
       e += (long long)gridDim.x * blockDim.x) {
    const long long q = R.elem_flat[e];
    R.lam_c[q] = __dadd_rn(R.lam_c[q], __dsub_rn(R.phi_c[q], R.psi_c[q]));
  }
}

__global__ void conv_cols_kernel(RefDev R, int lo, int hi) {
  __shared__ double red[64];
  for (int c = lo + blockIdx.x; c < hi; c += gridDim.x) conv_column(R, c, red);
}

// the combined kernel (admm.py:219-225, paper §III-C)
__global__ void fused_cols_kernel(RefDev R, int lo, int hi) {
  extern __shared__ double sm[];
  __shared__ double red[64];
  for (int c = lo + blockIdx.x; c < hi; c += gridDim.x) {
    psi_column(R, c, sm);
    lambda_column(R, c);
    __syncthreads();
    conv_column(R, c, red);
    scatter_column(R, c, R.psi_r, R.lam_r);
    __syncthreads();
  }
}

// the column patch (admm.py:227-253, paper §III-D): Φ of every member row
// recomputed from the CURRENT row layout (the duplicated work), the column's
// φ entries assembled, the owned rows published to φ_r, then Ψ, Λ, the
// residuals and a scatter into the alternate row buffers.
template <bool PADDED>
__global__ void patch_cols_kernel(RefDev R, int lo, int hi) {
  extern __shared__ double sm[];
  __shared__ double red[64];
  for (int c = lo + blockIdx.x; c < hi; c += gridDim.x) {
    const long long a = R.patch_off[c], b = R.patch_off[c + 1];
    for (long long q = a + threadIdx.x; q < b; q += blockDim.x) {
      const long long r = R.patch_rows[q];
      const int slot = R.patch_slot[q];
      const bool own = R.patch_owned[q] != 0;
      double* phic = R.phi_c + (long long)c * R.d_col + (q - a);
      double* phir = R.phi_r + r * R.d_row;
      phi_row<PADDED>(R, r, R.psi_r, R.lam_r, [=](int j, double v) {
        if (j == slot) *phic = v;
        if (own) phir[j] = v;
      });
    }
    __syncthreads();
    psi_column(R, c, sm);
    lambda_column(R, c);
    __syncthreads();
    conv_column(R, c, red);
    scatter_column(R, c, R.psi_r_nx, R.lam_r_nx);
    __syncthreads();
  }
}

// per-step row data (sls_core.py:330-349): a_pad = x[rs] (0 past the
// support), ‖a‖² ascending over the padded row, RowInfeasible scan
__global__ void set_x_kernel(RefDev R, const double* x) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < R.n_rows;
       r += (long long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int k = 0; k < R.d_row; ++k) {
      const long long col = R.rs[r * R.d_row + k];
      const double v = col >= 0 ? x[col] : 0.0;
      R.a_pad[r * R.d_row + k] = v;
      const double p = __dmul_rn(v, v);
      acc = k == 0 ? p : __dadd_rn(acc, p);
    }
    R.ada[r] = acc;
    if (acc == 0.0 && (R.lo[r] > 0.0 || R.hi[r] < 0.0)) atomicMin(R.bad, static_cast<int>(r));
  }
}

// ---- standalone stage operators (the reference's scalar functions) --------

// phi_row_solve (admm.py:28-51) over n independent rows of width d:
// v given, ‖a‖² = 0 returns v unchanged (infeasible rows are rejected on the
// host before the launch, as the reference raises before computing).
__global__ void op_phi_rows_kernel(int n, int d, const int* len, const double* a, const double* v,
                                   const double* ada, const double* w, const double* lo, const double* hi,
                                   double rho, double* out) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const double* ar = a + (size_t)r * d;
    const double* vr = v + (size_t)r * d;
    double* o = out + (size_t)r * d;
    const int L = len[r];
    if (ada[r] == 0.0) {
      for (int j = 0; j < d; ++j) o[j] = vr[j];
      continue;
    }
    double c = 0.0;
    for (int j = 0; j < L; ++j) {
      const double p = __dmul_rn(vr[j], ar[j]);
      c = j == 0 ? p : __dadd_rn(c, p);
    }
    const double den = __dadd_rn(rho, __dmul_rn(__dmul_rn(2.0, w[r]), ada[r]));
    const double y0 = __ddiv_rn(__dmul_rn(rho, c), den);
    // Python min(max(y0, lo), hi): max(NaN, lo) keeps NaN, min(NaN, hi) too
    const double y = y0 != y0 ? y0 : fmin(fmax(y0, lo[r]), hi[r]);
    const double scale = __ddiv_rn(__dsub_rn(y, c), ada[r]);
    for (int j = 0; j < L; ++j) o[j] = __dadd_rn(vr[j], __dmul_rn(scale, ar[j]));
  }
}

// psi_column_solve (admm.py:54-60) for n columns with their own operators
__global__ void op_psi_cols_kernel(int n, int m, int s, const double* g, const double* P, const double* rhs,
                                   const double* k, double* out) {
  extern __shared__ double sm[];
  double* res = sm;
  for (int c = blockIdx.x; c < n; c += gridDim.x) {
    const double* gc = g + (size_t)c * m * s;
    const double* pc = P + (size_t)c * s * m;
    const double* kc = k + (size_t)c * s;
    for (int i = threadIdx.x; i < m; i += blockDim.x)
      res[i] = __dsub_rn(rhs[(size_t)c * m + i], pairwise_sum(ProdRow{gc + (size_t)i * s, kc}, 0, s));
    __syncthreads();
    for (int j = threadIdx.x; j < s; j += blockDim.x)
      out[(size_t)c * s + j] = __dadd_rn(kc[j], pairwise_sum(ProdRow{pc + (size_t)j * m, res}, 0, m));
    __syncthreads();
  }
}

// lambda_update (admm.py:63-67)
__global__ void op_lambda_kernel(long long n, const double* lam, const double* phi, const double* psi, double* out) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x)
    out[q] = __dadd_rn(lam[q], __dsub_rn(phi[q], psi[q]));
}

// column_residuals (admm.py:69-74) for n columns of length len[c] (row stride d)
__global__ void op_residuals_kernel(int n, int d, const int* len, const double* phi, const double* psi,
                                    const double* prev, double rho, double* out) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    double p = 0.0, q = 0.0;
    bool first = true;
    for (int j = 0; j < len[c]; ++j) {
      const double a = fabs(__dsub_rn(phi[(size_t)c * d + j], psi[(size_t)c * d + j]));
      const double b = fabs(__dsub_rn(psi[(size_t)c * d + j], prev[(size_t)c * d + j]));
      p = first ? a : rmax(p, a);
      q = first ? b : rmax(q, b);
      first = false;
    }
    out[2 * c] = p;
    out[2 * c + 1] = __dmul_rn(rho, q);
  }
}

// ascending gather-dots: out[i] = Σ↑ vals[i, j] * x[idx[i, j]], j < len[i]
// (extract_control, admm.py:350-360)
__global__ void op_row_dots_kernel(int n, int d, const int* len, const double* vals, const long long* idx,
                                   const double* x, double* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int j = 0; j < len[i]; ++j) {
      const double p = __dmul_rn(vals[(size_t)i * d + j], x[idx[(size_t)i * d + j]]);
      acc = j == 0 ? p : __dadd_rn(acc, p);
    }
    out[i] = acc;
  }
}

// step_dynamics (admm.py:363-369): scipy's csr_matvec order for A x and B u
// (y[i] = 0; y[i] += a_ij x_j in index order), then the elementwise sum
__global__ void op_plant_kernel(int n, const long long* ap, const int* ai, const double* av, const long long* bp,
                                const int* bi, const double* bv, const double* x, const double* u, double* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double ya = 0.0, yb = 0.0;
    for (long long q = ap[i]; q < ap[i + 1]; ++q) ya = __dadd_rn(ya, __dmul_rn(av[q], x[ai[q]]));
    for (long long q = bp[i]; q < bp[i + 1]; ++q) yb = __dadd_rn(yb, __dmul_rn(bv[q], u[bi[q]]));
    out[i] = __dadd_rn(ya, yb);
  }
}

}  // namespace sched
}  // namespace dlmpc
