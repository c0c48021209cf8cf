// dlmpc.cu -- B200 (sm_100a) implementation of the DLMPC ADMM hot path.
//
// One persistent cooperative kernel runs a whole solve (or a whole closed
// loop of MPC steps) per launch. Per ADMM iteration:
//
//   Φ row stage   (reference admm.py:155-170)   one warp per subsystem; lanes
//                 walk the subsystem's rows; each row reads its d-hop
//                 neighbourhood of ψ,λ as contiguous per-column segments
//                 (block layout, see dlmpc.h) and produces the scalar Φ scale
//                 s_r = (clip(y0) - c_r)/||a||^2. φ itself is never stored:
//                 φ(r,c) = (ψ-λ)(r,c) + s_r·x_c is rebuilt where it is used.
//   grid barrier
//   Ψ/Λ/conv      (admm.py:174-217) tiles of TC same-class columns per CTA:
//                 k = φ+λ staged in shared memory, ψ' = q + N(Nᵀk) as two
//                 FP64 tensor-core GEMMs (mma.sync m8n8k4 f64; tcgen05 has no
//                 f64 kind) against the class's null-space basis N, which is
//                 staged in shared memory once per launch; then λ' = λ+(φ-ψ'),
//                 the residual maxima, and the write of (ψ',λ') into the other
//                 ping-pong buffer (which is the Ψ/Λ col->row exchange: the
//                 next Φ stage reads the column layout directly).
//   grid barrier  + global max of (pri, dual) via 64-bit atomicMax on the
//                 ordered bit pattern of non-negative doubles; every CTA reads
//                 the same two words and takes the same stop decision.
//
// EXACT=true replaces the Ψ GEMMs by the reference's dense form
// k + P(rhs - g k) with numpy's pairwise summation order and disables FMA
// contraction everywhere (__dmul_rn/__dadd_rn), which makes every iterate
// bit-identical to the reference's `sequential` schedule.
#include "../../include/dlmpc.h"

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <climits>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

namespace cg = cooperative_groups;

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kBadNone = 0x7f7f7f7f;   // cudaMemset(0x7f) pattern = "no infeasible row"

struct DevProblem {
  int n_sub, n_rows, n_cols, n_inputs, s_pad, exact, contiguous, d_row;
  double rho;
  const int64_t* row_start; const int64_t* ball_ptr; const int* ball_idx; const int* ball_off;
  const int* state_start; const int* state_count; const int* sub_first_bad;
  const double* row_w; const double* row_lo; const double* row_hi;
  const int* col_owner; const int* col_len; const int* col_class; const int* col_vec; const int* col_irow;
  int n_classes; const int* class_s; const int* class_n0; const int* class_ldn;
  const int64_t* class_null_off; const double* null_pool; const double* q_pool;
  const int* class_m; const int64_t* class_g_off; const int64_t* class_p_off;
  const double* g_pool; const double* p_pool; int m_pad; const double* rhs_pool; const int* ref_pos;
  int n_tiles, tile_cols; const int* tile_class; const int* tile_first; const int* tile_count;
  const int* tile_colv;
  const int64_t* a_ptr; const int* a_idx; const double* a_val;
  const int64_t* b_ptr; const int* b_idx; const double* b_val;
  const int* input_owner; const int* input_local;
  // mutable device state
  double* psi[2]; double* lam[2]; double* s_row; double* ada; double* x[2]; double* u;
  unsigned long long* resid;   // [2 * resid_cap] residual maxima per iteration
  int resid_cap;
  int* ctl;                    // [8]: 0 status, 1 fail step, 2/3 bad-row slots, 4 cur buffer, 5 fail iters
  // shared-memory plan (doubles)
  int resident_class, res_rows, res_ldn;
  int s8_max, n08_max, ldk, split_max;
  int off_k, off_y, off_yp, off_red, off_ex;
};

struct RunArgs {
  int t_sim, closed_loop, warm_start, cold_start, max_iters, stop_on_conv;
  double eps_pri, eps_dual;
  double* hist;        // [2*max_iters] history of the current / failing step
  int* step_iters;     // [t_sim]
  double* states;      // [(t_sim+1) * n_cols] (closed loop)
  double* inputs;      // [t_sim * n_inputs]
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

// numpy pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
// pairwise_sum_DOUBLE) of the rounded products a[i]*b[i], i < n.
// The reference's Ψ reductions `.sum(axis=2)` (admm.py:184, 186) use it.
template <class F>
__device__ double pairwise_sum(const F& f, int lo, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, f(lo + i));
    return r;
  }
  if (n <= 128) {
    double r0 = f(lo), r1 = f(lo + 1), r2 = f(lo + 2), r3 = f(lo + 3);
    double r4 = f(lo + 4), r5 = f(lo + 5), r6 = f(lo + 6), r7 = f(lo + 7);
    int i = 8;
    const int stop = n - (n % 8);
    for (; i < stop; i += 8) {
      r0 = __dadd_rn(r0, f(lo + i));     r1 = __dadd_rn(r1, f(lo + i + 1));
      r2 = __dadd_rn(r2, f(lo + i + 2)); r3 = __dadd_rn(r3, f(lo + i + 3));
      r4 = __dadd_rn(r4, f(lo + i + 4)); r5 = __dadd_rn(r5, f(lo + i + 5));
      r6 = __dadd_rn(r6, f(lo + i + 6)); r7 = __dadd_rn(r7, f(lo + i + 7));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3)),
                           __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
    for (; i < n; ++i) res = __dadd_rn(res, f(lo + i));
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pairwise_sum(f, lo, n2), pairwise_sum(f, lo + n2, n - n2));
}

struct ProdRow {   // g[i][j] * v[j]
  const double* row; const double* v;
  __device__ double operator()(int j) const { return __dmul_rn(row[j], v[j]); }
};
struct ProdStrided {  // P[j][i] * r[i] with P row-major [s][m]
  const double* row; const double* r;
  __device__ double operator()(int i) const { return __dmul_rn(row[i], r[i]); }
};

__device__ __forceinline__ double block_max(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double m = 0.0;
  if (threadIdx.x < 32) {
    m = threadIdx.x < kWarps ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  }
  return m;   // valid in thread 0
}

// ||a||^2 of every subsystem's rows (reference sls_core.py:338-339; all rows
// of a subsystem share the support, hence a_pad and a_dot_a) and the
// RowInfeasible scan of sls_core.py:346-348.
__device__ void row_data_stage(const DevProblem& P, const double* x, int* bad_slot) {
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, GT = gridDim.x * blockDim.x;
  for (int i = gt; i < P.n_sub; i += GT) {
    double acc = 0.0;
    bool first = true;
    int len = 0;
    for (long long e = P.ball_ptr[i]; e < P.ball_ptr[i + 1]; ++e) {
      const int j = P.ball_idx[e];
      const int c0 = P.state_start[j], nc = P.state_count[j];
      for (int c = c0; c < c0 + nc; ++c) {
        const double xc = ld_cg(x + c);
        const double pr = __dmul_rn(xc, xc);
        acc = first ? pr : __dadd_rn(acc, pr);
        first = false;
      }
      len += nc;
    }
    if (len < P.d_row) acc = __dadd_rn(acc, 0.0);   // the padded slots of a_pad
    P.ada[i] = acc;
    if (acc == 0.0 && P.sub_first_bad[i] >= 0) atomicMin(bad_slot, P.sub_first_bad[i]);
  }
}

// Φ row stage: s_r for every row.
template <bool EXACT>
__device__ void phi_stage(const DevProblem& P, int b, const double* x) {
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kWarps + (threadIdx.x >> 5), GW = gridDim.x * kWarps;
  const double* psi = P.psi[b];
  const double* lam = P.lam[b];
  const double rho = P.rho;
  for (int i = gw; i < P.n_sub; i += GW) {
    const long long r0 = P.row_start[i];
    const int nr = static_cast<int>(P.row_start[i + 1] - r0);
    const long long e0 = P.ball_ptr[i], e1 = P.ball_ptr[i + 1];
    const double ada = ld_cg(P.ada + i);
    for (int l = lane; l < nr; l += 32) {
      double acc = 0.0;
      bool first = true;
      int len = 0;
      for (long long e = e0; e < e1; ++e) {
        const int j = P.ball_idx[e];
        const int off = P.ball_off[e] + l;
        const int c0 = P.state_start[j], nc = P.state_count[j];
        len += nc;
        for (int c = c0; c < c0 + nc; ++c) {
          const size_t pos = static_cast<size_t>(c) * P.s_pad + off;
          const double v = __dsub_rn(ld_cg(psi + pos), ld_cg(lam + pos));
          const double xc = ld_cg(x + c);
          if (EXACT) {
            const double pr = __dmul_rn(v, xc);
            acc = first ? pr : __dadd_rn(acc, pr);
            first = false;
          } else {
            acc = fma(v, xc, acc);
          }
        }
      }
      if (EXACT && len < P.d_row) acc = __dadd_rn(acc, 0.0);
      const long long ir = r0 + l;
      const double w = P.row_w[ir];
      const double y0 = __ddiv_rn(__dmul_rn(rho, acc),
                                  __dadd_rn(rho, __dmul_rn(__dmul_rn(2.0, w), ada)));
      const double y = fmin(fmax(y0, P.row_lo[ir]), P.row_hi[ir]);
      P.s_row[ir] = ada > 0.0 ? __ddiv_rn(__dsub_rn(y, acc), ada) : 0.0;
    }
  }
}

__device__ __forceinline__ long long support_row(const DevProblem& P, int owner, int p) {
  if (P.contiguous) return P.row_start[P.ball_idx[P.ball_ptr[owner]]] + p;
  return P.col_irow[static_cast<size_t>(owner) * P.s_pad + p];
}

template <bool EXACT>
__device__ __forceinline__ double make_phi(double v, double s, double xc) {
  return EXACT ? __dadd_rn(v, __dmul_rn(s, xc)) : fma(s, xc, v);
}

// Ψ/Λ/residual column stage, fast path: tiles of TC columns, FP64 DMMA.
template <int TC>
__device__ void column_stage_fast(const DevProblem& P, int b, const double* x, int it,
                                  double* smem, const double* nsm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tig = lane & 3;
  double* kb = smem + P.off_k;
  double* yb = smem + P.off_y;
  double* yp = smem + P.off_yp;
  double* red = smem + P.off_red;
  const int ldk = P.ldk;
  const double* psi = P.psi[b];
  const double* lam = P.lam[b];
  double* psi_n = P.psi[b ^ 1];
  double* lam_n = P.lam[b ^ 1];
  double pri_m = 0.0, dual_m = 0.0;
  for (int tile = blockIdx.x; tile < P.n_tiles; tile += gridDim.x) {
    const int k = P.tile_class[tile];
    const int first = P.tile_first[tile];
    const int nt = P.tile_count[tile];
    const int S = P.class_s[k], S8 = (S + 7) & ~7;
    const int n0 = P.class_n0[k], n08 = (n0 + 7) & ~7;
    const int ldn = P.class_ldn[k];
    const double* nop = (k == P.resident_class) ? nsm : P.null_pool + P.class_null_off[k];
    // prologue: K[p][t] = φ + λ  (admm.py:183), zero padded to S8 x TC
    for (int idx = tid; idx < TC * S8; idx += kThreads) {
      const int t = idx / S8, p = idx - t * S8;
      double kv = 0.0;
      if (t < nt && p < S) {
        const int c = P.tile_colv[first + t];
        const size_t pos = static_cast<size_t>(c) * P.s_pad + p;
        const double ps = ld_cg(psi + pos), lm = ld_cg(lam + pos);
        const double s = ld_cg(P.s_row + support_row(P, P.col_owner[c], p));
        const double phi = make_phi<false>(__dsub_rn(ps, lm), s, ld_cg(x + c));
        kv = __dadd_rn(phi, lm);
      }
      kb[p * ldk + t] = kv;
    }
    __syncthreads();
    // GEMM 1: Y[a][t] = sum_p N[p][a] K[p][t]   (M = n0, N = TC, K = S)
    const int mt1 = n08 >> 3, ntn = TC >> 3, ks1 = S8 >> 2;
    const int pairs1 = mt1 * ntn;
    int split = 1;
    while (pairs1 * split < kWarps && split < P.split_max) split <<= 1;
    for (int u = warp; u < pairs1 * split; u += kWarps) {
      const int pair = u % pairs1, sl = u / pairs1;
      const int mt = pair / ntn, nn = pair - mt * ntn;
      double c0 = 0.0, c1 = 0.0;
      for (int ks = sl; ks < ks1; ks += split) {
        const int p = ks * 4 + tig;
        dmma(c0, c1, nop[p * ldn + mt * 8 + g], kb[p * ldk + nn * 8 + g]);
      }
      double* dst = (split == 1) ? yb : yp + static_cast<size_t>(sl) * P.n08_max * ldk;
      dst[(mt * 8 + g) * ldk + nn * 8 + 2 * tig] = c0;
      dst[(mt * 8 + g) * ldk + nn * 8 + 2 * tig + 1] = c1;
    }
    __syncthreads();
    if (split > 1) {
      for (int idx = tid; idx < n08 * TC; idx += kThreads) {
        const int a = idx / TC, t = idx - a * TC;
        double v = yp[a * ldk + t];
        for (int sl = 1; sl < split; ++sl) v += yp[static_cast<size_t>(sl) * P.n08_max * ldk + a * ldk + t];
        yb[a * ldk + t] = v;
      }
      __syncthreads();
    }
    // GEMM 2: O[p][t] = sum_a N[p][a] Y[a][t]   (M = S, N = TC, K = n0) -> kb
    const int mt2 = S8 >> 3, ks2 = n08 >> 2;
    for (int u = warp; u < mt2 * ntn; u += kWarps) {
      const int mt = u / ntn, nn = u - mt * ntn;
      double c0 = 0.0, c1 = 0.0;
      for (int ks = 0; ks < ks2; ++ks) {
        const int a = ks * 4 + tig;
        dmma(c0, c1, nop[(mt * 8 + g) * ldn + a], yb[a * ldk + nn * 8 + g]);
      }
      kb[(mt * 8 + g) * ldk + nn * 8 + 2 * tig] = c0;
      kb[(mt * 8 + g) * ldk + nn * 8 + 2 * tig + 1] = c1;
    }
    __syncthreads();
    // epilogue: ψ' = q + O, λ' = λ + (φ - ψ'), residual maxima (admm.py:186, 207, 216-217)
    for (int idx = tid; idx < nt * S; idx += kThreads) {
      const int t = idx / S, p = idx - t * S;
      const int c = P.tile_colv[first + t];
      const size_t pos = static_cast<size_t>(c) * P.s_pad + p;
      const double ps = ld_cg(psi + pos), lm = ld_cg(lam + pos);
      const double s = ld_cg(P.s_row + support_row(P, P.col_owner[c], p));
      const double phi = make_phi<false>(__dsub_rn(ps, lm), s, ld_cg(x + c));
      const double pn = P.q_pool[static_cast<size_t>(P.col_vec[c]) * P.s_pad + p] + kb[p * ldk + t];
      const double d = __dsub_rn(phi, pn);
      psi_n[pos] = pn;
      lam_n[pos] = __dadd_rn(lm, d);
      pri_m = fmax(pri_m, fabs(d));
      dual_m = fmax(dual_m, fabs(__dsub_rn(pn, ps)));
    }
    __syncthreads();
  }
  const double bp = block_max(pri_m, red);
  const double bd = block_max(dual_m, red);
  if (tid == 0) {
    atomicMax(P.resid + 2 * it, static_cast<unsigned long long>(__double_as_longlong(bp)));
    atomicMax(P.resid + 2 * it + 1, static_cast<unsigned long long>(__double_as_longlong(bd)));
  }
}

// Ψ/Λ/residual column stage, exact path: one column per CTA at a time, the
// reference's dense projector with numpy's pairwise order.
__device__ void column_stage_exact(const DevProblem& P, int b, const double* x, int it,
                                   double* smem) {
  const int tid = threadIdx.x;
  const int sp = P.s_pad;
  double* phi_s = smem + P.off_ex;          // internal order
  double* lam_s = phi_s + sp;
  double* psi_s = lam_s + sp;
  double* kref = psi_s + sp;                // reference order
  double* pnew = kref + sp;                 // internal order
  double* res_s = pnew + sp;                // [m_pad]
  double* red = smem + P.off_red;
  const double* psi = P.psi[b];
  const double* lam = P.lam[b];
  double* psi_n = P.psi[b ^ 1];
  double* lam_n = P.lam[b ^ 1];
  double pri_m = 0.0, dual_m = 0.0;
  for (int c = blockIdx.x; c < P.n_cols; c += gridDim.x) {
    const int owner = P.col_owner[c];
    const int k = P.col_class[c];
    const int S = P.class_s[k], m = P.class_m[k];
    const double* gk = P.g_pool + P.class_g_off[k];
    const double* pk = P.p_pool + P.class_p_off[k];
    const double* rhs = P.rhs_pool + static_cast<size_t>(P.col_vec[c]) * P.m_pad;
    const int* rp = P.ref_pos + static_cast<size_t>(owner) * sp;
    const double xc = ld_cg(x + c);
    for (int p = tid; p < S; p += kThreads) {
      const size_t pos = static_cast<size_t>(c) * sp + p;
      const double ps = ld_cg(psi + pos), lm = ld_cg(lam + pos);
      const double s = ld_cg(P.s_row + support_row(P, owner, p));
      phi_s[p] = make_phi<true>(__dsub_rn(ps, lm), s, xc);
      lam_s[p] = lm;
      psi_s[p] = ps;
    }
    __syncthreads();
    for (int q = tid; q < S; q += kThreads) kref[q] = __dadd_rn(phi_s[rp[q]], lam_s[rp[q]]);
    __syncthreads();
    for (int i = tid; i < m; i += kThreads)
      res_s[i] = __dsub_rn(rhs[i], pairwise_sum(ProdRow{gk + static_cast<size_t>(i) * S, kref}, 0, S));
    __syncthreads();
    for (int q = tid; q < S; q += kThreads)
      pnew[rp[q]] = __dadd_rn(kref[q],
                              pairwise_sum(ProdStrided{pk + static_cast<size_t>(q) * m, res_s}, 0, m));
    __syncthreads();
    for (int p = tid; p < S; p += kThreads) {
      const size_t pos = static_cast<size_t>(c) * sp + p;
      const double pn = pnew[p];
      const double d = __dsub_rn(phi_s[p], pn);
      psi_n[pos] = pn;
      lam_n[pos] = __dadd_rn(lam_s[p], d);
      pri_m = fmax(pri_m, fabs(d));
      dual_m = fmax(dual_m, fabs(__dsub_rn(pn, psi_s[p])));
    }
    __syncthreads();
  }
  const double bp = block_max(pri_m, red);
  const double bd = block_max(dual_m, red);
  if (tid == 0) {
    atomicMax(P.resid + 2 * it, static_cast<unsigned long long>(__double_as_longlong(bp)));
    atomicMax(P.resid + 2 * it + 1, static_cast<unsigned long long>(__double_as_longlong(bd)));
  }
}

// u_k = ascending dot of φ_r[input row k, t=0] with x (admm.py:350-360);
// φ is rebuilt from the iterate the last Φ stage read (buffer pb).
template <bool EXACT>
__device__ void control_stage(const DevProblem& P, int pb, const double* x) {
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, GT = gridDim.x * blockDim.x;
  for (int k = gt; k < P.n_inputs; k += GT) {
    const int i = P.input_owner[k], l = P.input_local[k];
    const double s = ld_cg(P.s_row + P.row_start[i] + l);
    double acc = 0.0;
    bool first = true;
    for (long long e = P.ball_ptr[i]; e < P.ball_ptr[i + 1]; ++e) {
      const int j = P.ball_idx[e];
      const int off = P.ball_off[e] + l;
      const int c0 = P.state_start[j], nc = P.state_count[j];
      for (int c = c0; c < c0 + nc; ++c) {
        const size_t pos = static_cast<size_t>(c) * P.s_pad + off;
        const double xc = ld_cg(x + c);
        const double phi = make_phi<EXACT>(__dsub_rn(ld_cg(P.psi[pb] + pos), ld_cg(P.lam[pb] + pos)), s, xc);
        const double pr = __dmul_rn(phi, xc);
        acc = first ? pr : __dadd_rn(acc, pr);
        first = false;
      }
    }
    P.u[k] = acc;
  }
}

// x+ = A x + B u on the plant's CSR rows (admm.py:363-369: scipy csr_matvec
// accumulates from 0 in stored order without FMA, then the two vectors add).
__device__ void plant_stage(const DevProblem& P, const double* x, double* xn) {
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, GT = gridDim.x * blockDim.x;
  for (int r = gt; r < P.n_cols; r += GT) {
    double ax = 0.0, bu = 0.0;
    for (long long q = P.a_ptr[r]; q < P.a_ptr[r + 1]; ++q) ax = __dadd_rn(ax, __dmul_rn(P.a_val[q], ld_cg(x + P.a_idx[q])));
    for (long long q = P.b_ptr[r]; q < P.b_ptr[r + 1]; ++q) bu = __dadd_rn(bu, __dmul_rn(P.b_val[q], ld_cg(P.u + P.b_idx[q])));
    xn[r] = __dadd_rn(ax, bu);
  }
}

__device__ void zero_iterate(const DevProblem& P, int b) {
  const size_t n = static_cast<size_t>(P.n_cols) * P.s_pad;
  const size_t gt = blockIdx.x * blockDim.x + threadIdx.x, GT = gridDim.x * blockDim.x;
  for (size_t q = gt; q < n; q += GT) { P.psi[b][q] = 0.0; P.lam[b][q] = 0.0; }
}

template <int TC, bool EXACT>
__global__ void __launch_bounds__(kThreads, 1) dlmpc_persistent(DevProblem P, RunArgs R) {
  extern __shared__ __align__(16) double smem[];
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x;
  const bool leader = blockIdx.x == 0 && tid == 0;
  // Stage the dominant class's null-space operator into shared memory once.
  const double* nsm = nullptr;
  if (!EXACT && P.resident_class >= 0) {
    const double* src = P.null_pool + P.class_null_off[P.resident_class];
    const int n = P.res_rows * P.res_ldn;
    for (int q = tid; q < n; q += kThreads) smem[q] = src[q];
    nsm = smem;
  }
  int b = P.ctl[4];
  const size_t gt = blockIdx.x * blockDim.x + tid, GT = gridDim.x * blockDim.x;
  for (int step = 0; step < R.t_sim; ++step) {
    const double* x = P.x[R.closed_loop ? (step & 1) : 0];
    int* bad_slot = P.ctl + 2 + (step & 1);
    for (size_t q = gt; q < static_cast<size_t>(2 * R.max_iters); q += GT) P.resid[q] = 0ull;
    if (R.closed_loop) {
      row_data_stage(P, x, bad_slot);
      if ((R.cold_start && step == 0) || !R.warm_start) zero_iterate(P, b);
    }
    grid.sync();
    if (R.closed_loop) {
      const int bad = *reinterpret_cast<volatile int*>(bad_slot);
      if (bad != kBadNone) {
        if (leader) { P.ctl[0] = DLMPC_ROW_INFEASIBLE; P.ctl[1] = step; P.ctl[5] = 0; P.ctl[4] = b; }
        return;
      }
      if (leader) P.ctl[2 + ((step + 1) & 1)] = kBadNone;
    }
    int it = 0;
    bool conv = false;
    while (it < R.max_iters) {
      phi_stage<EXACT>(P, b, x);
      grid.sync();
      if (EXACT) column_stage_exact(P, b, x, it, smem);
      else column_stage_fast<TC>(P, b, x, it, smem, nsm);
      grid.sync();
      b ^= 1;
      const double pri = __longlong_as_double(static_cast<long long>(__ldcg(P.resid + 2 * it)));
      const double dual = P.rho * __longlong_as_double(static_cast<long long>(__ldcg(P.resid + 2 * it + 1)));
      if (leader) { R.hist[2 * it] = pri; R.hist[2 * it + 1] = dual; }
      ++it;
      if (R.stop_on_conv && pri <= R.eps_pri && dual <= R.eps_dual) { conv = true; break; }
    }
    if (leader) R.step_iters[step] = it;
    if (R.stop_on_conv && !conv) {
      if (leader) { P.ctl[0] = DLMPC_NOT_CONVERGED; P.ctl[1] = step; P.ctl[5] = it; P.ctl[4] = b; }
      return;
    }
    if (R.closed_loop) {
      if (step == 0) {
        for (size_t q = gt; q < static_cast<size_t>(P.n_cols); q += GT) R.states[q] = x[q];
      }
      control_stage<EXACT>(P, b ^ 1, x);
      grid.sync();
      double* xn = P.x[(step + 1) & 1];
      plant_stage(P, x, xn);
      for (size_t q = gt; q < static_cast<size_t>(P.n_cols); q += GT)
        R.states[static_cast<size_t>(step + 1) * P.n_cols + q] = xn[q];
      for (size_t q = gt; q < static_cast<size_t>(P.n_inputs); q += GT)
        R.inputs[static_cast<size_t>(step) * P.n_inputs + q] = P.u[q];
      grid.sync();
    }
  }
  if (leader) { P.ctl[0] = DLMPC_OK; P.ctl[4] = b; }
}

// Row data for the solve API (dlmpc_set_x): a plain launch.
__global__ void set_x_kernel(DevProblem P) {
  row_data_stage(P, P.x[0], P.ctl + 2);
}

// φ of the last iteration, internal column layout (for dlmpc_get(DLMPC_PHI)).
template <bool EXACT>
__global__ void phi_materialize_kernel(DevProblem P, int pb, double* out) {
  const size_t n = static_cast<size_t>(P.n_cols) * P.s_pad;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n; q += (size_t)gridDim.x * blockDim.x) {
    const int c = static_cast<int>(q / P.s_pad), p = static_cast<int>(q % P.s_pad);
    double v = 0.0;
    if (p < P.col_len[c]) {
      const double s = P.s_row[support_row(P, P.col_owner[c], p)];
      v = make_phi<EXACT>(__dsub_rn(P.psi[pb][q], P.lam[pb][q]), s, P.x[0][c]);
    }
    out[q] = v;
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

thread_local std::string g_global_error;

}  // namespace

struct dlmpc_handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  DevProblem P{};
  std::vector<void*> allocs;
  std::string err;
  int grid = 0, smem_bytes = 0, sm_count = 0;
  int max_iters_cap = 0;
  double* d_hist = nullptr; int* d_step_iters = nullptr;
  double* d_states = nullptr; double* d_inputs = nullptr; int states_cap = 0;
  float last_ms = 0.f; int last_launches = 0;
  double* d_scratch = nullptr;
};

namespace {

int fail(dlmpc_handle* h, int code, const std::string& msg) {
  if (h) h->err = msg; else g_global_error = msg;
  return code;
}

#define CUDA_OR_FAIL(h, expr)                                                        \
  do {                                                                               \
    cudaError_t e_ = (expr);                                                         \
    if (e_ != cudaSuccess)                                                           \
      return fail((h), DLMPC_CUDA_ERROR, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

template <class T>
int upload(dlmpc_handle* h, const T* src, size_t n, const T** dst) {
  *dst = nullptr;
  if (src == nullptr || n == 0) return DLMPC_OK;
  void* p = nullptr;
  CUDA_OR_FAIL(h, cudaMalloc(&p, n * sizeof(T)));
  h->allocs.push_back(p);
  CUDA_OR_FAIL(h, cudaMemcpy(p, src, n * sizeof(T), cudaMemcpyHostToDevice));
  *dst = static_cast<const T*>(p);
  return DLMPC_OK;
}

template <class T>
int alloc(dlmpc_handle* h, size_t n, T** dst) {
  void* p = nullptr;
  CUDA_OR_FAIL(h, cudaMalloc(&p, (n ? n : 1) * sizeof(T)));
  h->allocs.push_back(p);
  CUDA_OR_FAIL(h, cudaMemset(p, 0, (n ? n : 1) * sizeof(T)));
  *dst = static_cast<T*>(p);
  return DLMPC_OK;
}

using KernelFn = void (*)(DevProblem, RunArgs);

KernelFn pick_kernel(const DevProblem& P) {
  if (P.exact) return dlmpc_persistent<8, true>;
  switch (P.tile_cols) {
    case 8: return dlmpc_persistent<8, false>;
    case 16: return dlmpc_persistent<16, false>;
    default: return dlmpc_persistent<32, false>;
  }
}

int ensure_run_buffers(dlmpc_handle* h, int max_iters, int t_sim) {
  if (max_iters > h->max_iters_cap) {
    if (h->d_hist) cudaFree(h->d_hist);
    if (h->P.resid) cudaFree(h->P.resid);
    CUDA_OR_FAIL(h, cudaMalloc(&h->d_hist, sizeof(double) * 2 * max_iters));
    CUDA_OR_FAIL(h, cudaMalloc(&h->P.resid, sizeof(unsigned long long) * 2 * max_iters));
    h->max_iters_cap = max_iters;
    h->P.resid_cap = max_iters;
  }
  if (t_sim > h->states_cap) {
    if (h->d_step_iters) cudaFree(h->d_step_iters);
    if (h->d_states) cudaFree(h->d_states);
    if (h->d_inputs) cudaFree(h->d_inputs);
    CUDA_OR_FAIL(h, cudaMalloc(&h->d_step_iters, sizeof(int) * t_sim));
    CUDA_OR_FAIL(h, cudaMalloc(&h->d_states, sizeof(double) * (size_t)(t_sim + 1) * h->P.n_cols));
    CUDA_OR_FAIL(h, cudaMalloc(&h->d_inputs, sizeof(double) * (size_t)t_sim * (h->P.n_inputs ? h->P.n_inputs : 1)));
    h->states_cap = t_sim;
  }
  return DLMPC_OK;
}

int launch(dlmpc_handle* h, const RunArgs& R) {
  KernelFn fn = pick_kernel(h->P);
  DevProblem P = h->P;
  RunArgs Rc = R;
  void* args[] = {&P, &Rc};
  CUDA_OR_FAIL(h, cudaEventRecord(h->ev0, h->stream));
  CUDA_OR_FAIL(h, cudaLaunchCooperativeKernel(reinterpret_cast<void*>(fn), dim3(h->grid), dim3(kThreads),
                                              args, static_cast<size_t>(h->smem_bytes), h->stream));
  CUDA_OR_FAIL(h, cudaEventRecord(h->ev1, h->stream));
  h->last_launches = 1;
  return DLMPC_OK;
}

int finish_timing(dlmpc_handle* h) {
  CUDA_OR_FAIL(h, cudaEventSynchronize(h->ev1));
  CUDA_OR_FAIL(h, cudaEventElapsedTime(&h->last_ms, h->ev0, h->ev1));
  return DLMPC_OK;
}

int read_ctl(dlmpc_handle* h, int* ctl) {
  CUDA_OR_FAIL(h, cudaMemcpyAsync(ctl, h->P.ctl, sizeof(int) * 8, cudaMemcpyDeviceToHost, h->stream));
  CUDA_OR_FAIL(h, cudaStreamSynchronize(h->stream));
  return DLMPC_OK;
}

}  // namespace

extern "C" {

const char* dlmpc_global_error(void) { return g_global_error.c_str(); }
const char* dlmpc_last_error(const dlmpc_handle* h) { return h ? h->err.c_str() : g_global_error.c_str(); }

int dlmpc_create(const dlmpc_problem* pr, int device, dlmpc_handle** out) {
  if (!pr || !out) return fail(nullptr, DLMPC_BAD_ARGUMENT, "null argument");
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(nullptr, DLMPC_NO_DEVICE, "no CUDA device visible");
  if (device < 0 || device >= ndev) return fail(nullptr, DLMPC_BAD_ARGUMENT, "device out of range");
  if (pr->tile_cols != 8 && pr->tile_cols != 16 && pr->tile_cols != 32)
    return fail(nullptr, DLMPC_BAD_ARGUMENT, "tile_cols must be 8, 16 or 32");
  auto* h = new dlmpc_handle();
  h->device = device;
  if (cudaSetDevice(device) != cudaSuccess) { delete h; return fail(nullptr, DLMPC_CUDA_ERROR, "cudaSetDevice failed"); }
  int rc = DLMPC_OK;
#define UP(field, n) do { if ((rc = upload(h, pr->field, (size_t)(n), &P.field)) != DLMPC_OK) goto bad; } while (0)
  {
    DevProblem& P = h->P;
    P.n_sub = pr->n_sub; P.n_rows = pr->n_rows; P.n_cols = pr->n_cols; P.n_inputs = pr->n_inputs;
    P.s_pad = pr->s_pad; P.exact = pr->exact; P.contiguous = pr->contiguous; P.rho = pr->rho;
    P.n_classes = pr->n_classes; P.m_pad = pr->m_pad; P.n_tiles = pr->n_tiles; P.tile_cols = pr->tile_cols;
    const size_t nb = (size_t)pr->ball_ptr[pr->n_sub];
    int d_row = 0;
    for (int i = 0; i < pr->n_sub; ++i) {
      int len = 0;
      for (long long e = pr->ball_ptr[i]; e < pr->ball_ptr[i + 1]; ++e) len += pr->state_count[pr->ball_idx[e]];
      if (len > d_row) d_row = len;
    }
    P.d_row = d_row;
    UP(row_start, pr->n_sub + 1); UP(ball_ptr, pr->n_sub + 1); UP(ball_idx, nb); UP(ball_off, nb);
    UP(state_start, pr->n_sub); UP(state_count, pr->n_sub); UP(sub_first_bad, pr->n_sub);
    UP(row_w, pr->n_rows); UP(row_lo, pr->n_rows); UP(row_hi, pr->n_rows);
    UP(col_owner, pr->n_cols); UP(col_len, pr->n_cols); UP(col_class, pr->n_cols); UP(col_vec, pr->n_cols);
    if (!pr->contiguous) UP(col_irow, (size_t)pr->n_sub * pr->s_pad);
    UP(class_s, pr->n_classes); UP(class_n0, pr->n_classes); UP(class_ldn, pr->n_classes);
    UP(class_null_off, pr->n_classes + 1);
    UP(null_pool, pr->class_null_off[pr->n_classes]);
    UP(q_pool, (size_t)pr->n_vec * pr->s_pad);
    if (pr->exact) {
      UP(class_m, pr->n_classes); UP(class_g_off, pr->n_classes + 1); UP(class_p_off, pr->n_classes + 1);
      UP(g_pool, pr->class_g_off[pr->n_classes]); UP(p_pool, pr->class_p_off[pr->n_classes]);
      UP(rhs_pool, (size_t)pr->n_vec * pr->m_pad); UP(ref_pos, (size_t)pr->n_sub * pr->s_pad);
    }
    UP(tile_class, pr->n_tiles); UP(tile_first, pr->n_tiles); UP(tile_count, pr->n_tiles); UP(tile_colv, pr->n_cols);
    UP(a_ptr, pr->n_cols + 1); UP(a_idx, pr->a_ptr[pr->n_cols]); UP(a_val, pr->a_ptr[pr->n_cols]);
    UP(b_ptr, pr->n_cols + 1); UP(b_idx, pr->b_ptr[pr->n_cols]); UP(b_val, pr->b_ptr[pr->n_cols]);
    UP(input_owner, pr->n_inputs); UP(input_local, pr->n_inputs);
    const size_t ncell = (size_t)pr->n_cols * pr->s_pad;
    for (int q = 0; q < 2; ++q) {
      if ((rc = alloc(h, ncell, &P.psi[q])) != DLMPC_OK) goto bad;
      if ((rc = alloc(h, ncell, &P.lam[q])) != DLMPC_OK) goto bad;
      if ((rc = alloc(h, (size_t)pr->n_cols, &P.x[q])) != DLMPC_OK) goto bad;
    }
    if ((rc = alloc(h, (size_t)pr->n_rows, &P.s_row)) != DLMPC_OK) goto bad;
    if ((rc = alloc(h, (size_t)pr->n_sub, &P.ada)) != DLMPC_OK) goto bad;
    if ((rc = alloc(h, (size_t)(pr->n_inputs ? pr->n_inputs : 1), &P.u)) != DLMPC_OK) goto bad;
    if ((rc = alloc(h, 8, &P.ctl)) != DLMPC_OK) goto bad;
    if ((rc = alloc(h, ncell, &h->d_scratch)) != DLMPC_OK) goto bad;
    if (cudaMemset(P.ctl + 2, 0x7f, sizeof(int) * 2) != cudaSuccess) { rc = fail(h, DLMPC_CUDA_ERROR, "memset"); goto bad; }

    // shared-memory plan (doubles): [resident operator][K/O tile][Y][Y partials][reductions][exact scratch]
    int s8_max = 8, n08_max = 8, split_max = 1, res = -1, res_cols = 0;
    std::vector<int> cls_cols(pr->n_classes, 0);
    for (int c = 0; c < pr->n_cols; ++c) cls_cols[pr->col_class[c]]++;
    const int tc = pr->tile_cols;
    for (int k = 0; k < pr->n_classes; ++k) {
      const int s8 = (pr->class_s[k] + 7) & ~7, n08 = (pr->class_n0[k] + 7) & ~7;
      if (s8 > s8_max) s8_max = s8;
      if (n08 > n08_max) n08_max = n08;
      const int pairs1 = (n08 / 8) * (tc / 8);
      int sp = 1;
      while (pairs1 * sp < kWarps && sp < 4) sp <<= 1;
      if (sp > split_max) split_max = sp;
      if (cls_cols[k] > res_cols) { res_cols = cls_cols[k]; res = k; }
    }
    int ldk = tc; while (ldk % 16 != 4) ++ldk;
    P.s8_max = s8_max; P.n08_max = n08_max; P.ldk = ldk; P.split_max = split_max;
    const long long opt_limit = 220 * 1024;
    long long tile_d = (long long)s8_max * ldk + (long long)n08_max * ldk * (1 + (split_max > 1 ? split_max : 0));
    long long res_d = 0;
    if (!pr->exact && res >= 0) {
      res_d = (long long)((pr->class_s[res] + 7) & ~7) * pr->class_ldn[res];
      if ((res_d + tile_d + 64) * 8 > opt_limit) { res = -1; res_d = 0; }
    }
    P.resident_class = pr->exact ? -1 : res;
    P.res_rows = res >= 0 ? ((pr->class_s[res] + 7) & ~7) : 0;
    P.res_ldn = res >= 0 ? pr->class_ldn[res] : 0;
    long long off = (res_d + 1) & ~1LL;
    P.off_k = (int)off; off += (long long)s8_max * ldk;
    P.off_y = (int)off; off += (long long)n08_max * ldk;
    P.off_yp = (int)off; off += split_max > 1 ? (long long)split_max * n08_max * ldk : 0;
    P.off_red = (int)off; off += 64;
    P.off_ex = (int)off;
    if (pr->exact) { P.off_k = P.off_y = P.off_yp = 0; P.off_red = 0; P.off_ex = 64; off = 64 + 5LL * pr->s_pad + pr->m_pad; }
    h->smem_bytes = (int)(off * 8);
    if (h->smem_bytes > opt_limit) { rc = fail(h, DLMPC_BAD_ARGUMENT, "tile does not fit in shared memory"); goto bad; }
    KernelFn fn = pick_kernel(P);
    if (cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                             h->smem_bytes) != cudaSuccess) { rc = fail(h, DLMPC_CUDA_ERROR, "smem attribute"); goto bad; }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, reinterpret_cast<const void*>(fn), kThreads,
                                                      h->smem_bytes) != cudaSuccess || per_sm < 1) {
      rc = fail(h, DLMPC_CUDA_ERROR, "kernel cannot be resident"); goto bad;
    }
    cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, device);
    h->grid = h->sm_count;   // one CTA per SM: operator staged once per SM
    if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&h->ev0) != cudaSuccess || cudaEventCreate(&h->ev1) != cudaSuccess) {
      rc = fail(h, DLMPC_CUDA_ERROR, "stream/event creation failed"); goto bad;
    }
    if ((rc = ensure_run_buffers(h, 64, 1)) != DLMPC_OK) goto bad;
  }
#undef UP
  *out = h;
  return DLMPC_OK;
bad:
  g_global_error = h->err;
  dlmpc_destroy(h);
  return rc;
}

void dlmpc_destroy(dlmpc_handle* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (void* p : h->allocs) cudaFree(p);
  if (h->d_hist) cudaFree(h->d_hist);
  if (h->P.resid) cudaFree(h->P.resid);
  if (h->d_step_iters) cudaFree(h->d_step_iters);
  if (h->d_states) cudaFree(h->d_states);
  if (h->d_inputs) cudaFree(h->d_inputs);
  if (h->ev0) cudaEventDestroy(h->ev0);
  if (h->ev1) cudaEventDestroy(h->ev1);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

int dlmpc_set_x(dlmpc_handle* h, const double* x, int64_t* bad_row) {
  if (!h || !x) return fail(h, DLMPC_BAD_ARGUMENT, "null argument");
  cudaSetDevice(h->device);
  CUDA_OR_FAIL(h, cudaMemcpyAsync(h->P.x[0], x, sizeof(double) * h->P.n_cols, cudaMemcpyHostToDevice, h->stream));
  CUDA_OR_FAIL(h, cudaMemsetAsync(h->P.ctl + 2, 0x7f, sizeof(int), h->stream));
  set_x_kernel<<<(h->P.n_sub + 255) / 256, 256, 0, h->stream>>>(h->P);
  CUDA_OR_FAIL(h, cudaGetLastError());
  int ctl[8];
  if (int rc = read_ctl(h, ctl)) return rc;
  if (bad_row) *bad_row = ctl[2] == kBadNone ? -1 : ctl[2];
  return ctl[2] == kBadNone ? DLMPC_OK : DLMPC_ROW_INFEASIBLE;
}

static int run_iterations(dlmpc_handle* h, int max_iters, double eps_pri, double eps_dual, int stop,
                          int* iters, double* hist) {
  cudaSetDevice(h->device);
  if (max_iters < 1) return fail(h, DLMPC_BAD_ARGUMENT, "max_iters must be >= 1");
  if (int rc = ensure_run_buffers(h, max_iters, 1)) return rc;
  RunArgs R{};
  R.t_sim = 1; R.closed_loop = 0; R.warm_start = 1; R.cold_start = 0;
  R.max_iters = max_iters; R.stop_on_conv = stop; R.eps_pri = eps_pri; R.eps_dual = eps_dual;
  R.hist = h->d_hist; R.step_iters = h->d_step_iters; R.states = h->d_states; R.inputs = h->d_inputs;
  if (int rc = launch(h, R)) return rc;
  if (int rc = finish_timing(h)) return rc;
  CUDA_OR_FAIL(h, cudaGetLastError());
  int ctl[8];
  if (int rc = read_ctl(h, ctl)) return rc;
  int n = 0;
  CUDA_OR_FAIL(h, cudaMemcpy(&n, h->d_step_iters, sizeof(int), cudaMemcpyDeviceToHost));
  if (ctl[0] == DLMPC_NOT_CONVERGED) n = ctl[5];
  if (iters) *iters = n;
  if (hist && n > 0) CUDA_OR_FAIL(h, cudaMemcpy(hist, h->d_hist, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost));
  return ctl[0];
}

int dlmpc_solve(dlmpc_handle* h, int max_iters, double eps_pri, double eps_dual, int* iters, double* hist) {
  if (!h) return fail(h, DLMPC_BAD_ARGUMENT, "null handle");
  return run_iterations(h, max_iters, eps_pri, eps_dual, 1, iters, hist);
}

int dlmpc_iterate(dlmpc_handle* h, int n, double* hist) {
  if (!h) return fail(h, DLMPC_BAD_ARGUMENT, "null handle");
  int it = 0;
  return run_iterations(h, n, 0.0, 0.0, 0, &it, hist);
}

int dlmpc_simulate_device(dlmpc_handle* h, const double* x0_dev, int t_sim, int warm_start, int cold_start,
                          int max_iters, double eps_pri, double eps_dual, double* states_dev,
                          double* inputs_dev, int* step_iters_dev, int* status_dev) {
  if (!h || !x0_dev || t_sim < 1 || max_iters < 1) return fail(h, DLMPC_BAD_ARGUMENT, "bad argument");
  cudaSetDevice(h->device);
  if (int rc = ensure_run_buffers(h, max_iters, t_sim)) return rc;
  CUDA_OR_FAIL(h, cudaMemcpyAsync(h->P.x[0], x0_dev, sizeof(double) * h->P.n_cols, cudaMemcpyDeviceToDevice, h->stream));
  CUDA_OR_FAIL(h, cudaMemsetAsync(h->P.ctl + 2, 0x7f, sizeof(int) * 2, h->stream));
  RunArgs R{};
  R.t_sim = t_sim; R.closed_loop = 1; R.warm_start = warm_start; R.cold_start = cold_start;
  R.max_iters = max_iters; R.stop_on_conv = 1; R.eps_pri = eps_pri; R.eps_dual = eps_dual;
  R.hist = h->d_hist;
  R.step_iters = step_iters_dev ? step_iters_dev : h->d_step_iters;
  R.states = states_dev ? states_dev : h->d_states;
  R.inputs = inputs_dev ? inputs_dev : h->d_inputs;
  if (int rc = launch(h, R)) return rc;
  if (status_dev) CUDA_OR_FAIL(h, cudaMemcpyAsync(status_dev, h->P.ctl, sizeof(int) * 8, cudaMemcpyDeviceToDevice, h->stream));
  CUDA_OR_FAIL(h, cudaGetLastError());
  return DLMPC_OK;
}

int dlmpc_simulate(dlmpc_handle* h, const double* x0, int t_sim, int warm_start, int cold_start,
                   int max_iters, double eps_pri, double eps_dual, double* states, double* inputs,
                   int* step_iters, int* fail_step, int64_t* bad_row, int* fail_iters, double* fail_hist) {
  if (!h || !x0 || t_sim < 1) return fail(h, DLMPC_BAD_ARGUMENT, "bad argument");
  cudaSetDevice(h->device);
  if (int rc = ensure_run_buffers(h, max_iters, t_sim)) return rc;
  CUDA_OR_FAIL(h, cudaMemcpyAsync(h->d_states, x0, sizeof(double) * h->P.n_cols, cudaMemcpyHostToDevice, h->stream));
  if (int rc = dlmpc_simulate_device(h, h->d_states, t_sim, warm_start, cold_start, max_iters, eps_pri, eps_dual,
                                     nullptr, nullptr, nullptr, nullptr)) return rc;
  if (int rc = finish_timing(h)) return rc;
  int ctl[8];
  if (int rc = read_ctl(h, ctl)) return rc;
  int done = t_sim;
  if (ctl[0] != DLMPC_OK) done = ctl[1];
  if (fail_step) *fail_step = ctl[0] == DLMPC_OK ? -1 : ctl[1];
  if (bad_row) *bad_row = ctl[0] == DLMPC_ROW_INFEASIBLE ? ctl[2 + (ctl[1] & 1)] : -1;
  if (fail_iters) *fail_iters = ctl[0] == DLMPC_NOT_CONVERGED ? ctl[5] : 0;
  if (states) CUDA_OR_FAIL(h, cudaMemcpy(states, h->d_states, sizeof(double) * (size_t)(done + 1) * h->P.n_cols, cudaMemcpyDeviceToHost));
  if (inputs && done > 0 && h->P.n_inputs > 0)
    CUDA_OR_FAIL(h, cudaMemcpy(inputs, h->d_inputs, sizeof(double) * (size_t)done * h->P.n_inputs, cudaMemcpyDeviceToHost));
  if (step_iters && done > 0) CUDA_OR_FAIL(h, cudaMemcpy(step_iters, h->d_step_iters, sizeof(int) * done, cudaMemcpyDeviceToHost));
  if (fail_hist && ctl[0] == DLMPC_NOT_CONVERGED && ctl[5] > 0)
    CUDA_OR_FAIL(h, cudaMemcpy(fail_hist, h->d_hist, sizeof(double) * 2 * ctl[5], cudaMemcpyDeviceToHost));
  return ctl[0];
}

int dlmpc_get(dlmpc_handle* h, int which, double* dst) {
  if (!h || !dst) return fail(h, DLMPC_BAD_ARGUMENT, "null argument");
  cudaSetDevice(h->device);
  int ctl[8];
  if (int rc = read_ctl(h, ctl)) return rc;
  const int b = ctl[4];
  const size_t ncell = (size_t)h->P.n_cols * h->P.s_pad;
  const double* src = nullptr;
  size_t n = ncell;
  switch (which) {
    case DLMPC_PSI: src = h->P.psi[b]; break;
    case DLMPC_LAM: src = h->P.lam[b]; break;
    case DLMPC_PSI_PREV: src = h->P.psi[b ^ 1]; break;
    case DLMPC_LAM_PREV: src = h->P.lam[b ^ 1]; break;
    case DLMPC_S_ROW: src = h->P.s_row; n = h->P.n_rows; break;
    case DLMPC_X: src = h->P.x[0]; n = h->P.n_cols; break;
    case DLMPC_ADA: src = h->P.ada; n = h->P.n_sub; break;
    case DLMPC_PHI: {
      if (h->P.exact) phi_materialize_kernel<true><<<h->sm_count * 4, 256, 0, h->stream>>>(h->P, b ^ 1, h->d_scratch);
      else phi_materialize_kernel<false><<<h->sm_count * 4, 256, 0, h->stream>>>(h->P, b ^ 1, h->d_scratch);
      CUDA_OR_FAIL(h, cudaGetLastError());
      src = h->d_scratch;
      break;
    }
    default: return fail(h, DLMPC_BAD_ARGUMENT, "unknown array id");
  }
  CUDA_OR_FAIL(h, cudaMemcpyAsync(dst, src, sizeof(double) * n, cudaMemcpyDeviceToHost, h->stream));
  CUDA_OR_FAIL(h, cudaStreamSynchronize(h->stream));
  return DLMPC_OK;
}

int dlmpc_put(dlmpc_handle* h, int which, const double* src) {
  if (!h || !src) return fail(h, DLMPC_BAD_ARGUMENT, "null argument");
  cudaSetDevice(h->device);
  int ctl[8];
  if (int rc = read_ctl(h, ctl)) return rc;
  const int b = ctl[4];
  const size_t ncell = (size_t)h->P.n_cols * h->P.s_pad;
  double* dst = nullptr;
  switch (which) {
    case DLMPC_PSI: dst = h->P.psi[b]; break;
    case DLMPC_LAM: dst = h->P.lam[b]; break;
    case DLMPC_PSI_PREV: dst = h->P.psi[b ^ 1]; break;
    case DLMPC_LAM_PREV: dst = h->P.lam[b ^ 1]; break;
    default: return fail(h, DLMPC_BAD_ARGUMENT, "array is not writable");
  }
  CUDA_OR_FAIL(h, cudaMemcpyAsync(dst, src, sizeof(double) * ncell, cudaMemcpyHostToDevice, h->stream));
  CUDA_OR_FAIL(h, cudaStreamSynchronize(h->stream));
  return DLMPC_OK;
}

int dlmpc_zero(dlmpc_handle* h) {
  if (!h) return fail(h, DLMPC_BAD_ARGUMENT, "null handle");
  cudaSetDevice(h->device);
  const size_t ncell = (size_t)h->P.n_cols * h->P.s_pad;
  for (int q = 0; q < 2; ++q) {
    CUDA_OR_FAIL(h, cudaMemsetAsync(h->P.psi[q], 0, sizeof(double) * ncell, h->stream));
    CUDA_OR_FAIL(h, cudaMemsetAsync(h->P.lam[q], 0, sizeof(double) * ncell, h->stream));
  }
  CUDA_OR_FAIL(h, cudaMemsetAsync(h->P.s_row, 0, sizeof(double) * h->P.n_rows, h->stream));
  CUDA_OR_FAIL(h, cudaStreamSynchronize(h->stream));
  return DLMPC_OK;
}

int dlmpc_last_timing(const dlmpc_handle* h, float* ms, int* launches) {
  if (!h) return DLMPC_BAD_ARGUMENT;
  if (ms) *ms = h->last_ms;
  if (launches) *launches = h->last_launches;
  return DLMPC_OK;
}

void* dlmpc_stream(dlmpc_handle* h) { return h ? static_cast<void*>(h->stream) : nullptr; }

int dlmpc_synchronize(dlmpc_handle* h) {
  if (!h) return DLMPC_BAD_ARGUMENT;
  CUDA_OR_FAIL(h, cudaStreamSynchronize(h->stream));
  return DLMPC_OK;
}

int dlmpc_info(const dlmpc_handle* h, int64_t* out) {
  if (!h || !out) return DLMPC_BAD_ARGUMENT;
  out[0] = h->P.n_rows; out[1] = h->P.n_cols; out[2] = h->P.s_pad; out[3] = h->P.n_sub;
  out[4] = h->grid; out[5] = h->P.tile_cols; out[6] = h->smem_bytes;
  return DLMPC_OK;
}

}  // extern "C"
