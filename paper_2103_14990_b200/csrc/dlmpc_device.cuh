// dlmpc_device.cuh -- device code of the DLMPC ADMM hot path (sm_100a).
//
// One persistent cooperative kernel, dlmpc_persistent<TC, MODE>, runs a whole
// solve or a whole closed loop (one launch); MODE selects the schedule:
//
//  kPatch     fast path, d-hop balls contiguous in subsystem ids (chains,
//             banded graphs), small/medium networks. Each CTA owns contiguous
//             units of subsystems; per ADMM iteration and unit it recomputes
//             the Φ scale s_r of every row its columns touch -- own rows plus a
//             d-hop halo (the paper's column patch, §III-D; reference
//             admm.py:155-170, 227-253) -- then runs the Ψ projection of its
//             columns as two FP64 tensor-core GEMMs against the class
//             null-space basis staged in shared memory, the Λ update and the
//             residual maxima (admm.py:174-217). ONE grid barrier per
//             iteration, which also publishes the global (pri, dual).
//  kPatchRb   kPatch whose chunks hold <= 2 columns (C2-sized networks): the
//             Ψ projection as a register-blocked FP64 GEMV pair (gemv_pair_rb)
//             instead of DMMA tiles that would be 3/4 empty.
//  kStream    the same algorithm restructured for large networks (>= 2 chunks
//             per CTA): Φ dots of the next iteration accumulated by the Ψ
//             epilogues (per-unit slots, deterministic), ψ/λ staged by TMA
//             bulk copies, register epilogue, hybrid warp split.
//  kTwoPhase  fast path for arbitrary graphs: a grid-wide Φ stage writes s_r
//             to global memory, barrier, class-sorted column tiles.
//  kExact     the reference's arithmetic bit for bit (dense projector, numpy
//             pairwise sums, no FMA), two-phase.
//
// φ is never stored: φ(r,c) = (ψ-λ)(r,c) + s_r·x_c is rebuilt where needed.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace cg = cooperative_groups;

namespace dlmpc {

// GEMM 1: a warp takes a whole m-row of tiles when that costs no extra round
#ifndef DLMPC_G1_MROW
#define DLMPC_G1_MROW 1
#endif
#ifndef DLMPC_STREAM_MROW
#define DLMPC_STREAM_MROW 0
#endif
#ifndef DLMPC_STREAM_KRB
// stream Φ: patch rows per thread whose loads are in flight together; 4
// covers a unit's <= 2048 patch rows in one round trip (N=1e5 642.4 -> 632.9
// us/iter against 3, bitwise the same; 2 is slower)
#define DLMPC_STREAM_KRB 4
#endif

// Optional per-phase timers (profiling build only: -DDLMPC_PHASE_TIMING).
// Thread 0 of every CTA accumulates SM-cycle deltas per phase in shared
// memory and adds them to P.phase_ns[blockIdx.x * 16 + phase] (0-7 per
// iteration, 8-15 per MPC step) when the kernel ends (round 1 added them to
// global memory at every lap: the read-modify-write put an L2 round trip into
// the next lap's interval).
#ifdef DLMPC_PHASE_TIMING
__device__ __forceinline__ unsigned long long gtimer() {   // SM cycles (globaltimer is too coarse)
  return static_cast<unsigned long long>(clock64());
}
__shared__ unsigned long long pt_sh[16];
#define PT_DECL unsigned long long pt_t0 = 0;
#define PT_START if (threadIdx.x == 0) pt_t0 = gtimer();
#define PT_LAP(P, ph) if (threadIdx.x == 0) { unsigned long long t1_ = gtimer(); pt_sh[(ph)] += t1_ - pt_t0; pt_t0 = t1_; }
#define PT_ADD(ph, v) if (threadIdx.x == 0) pt_sh[(ph)] += (v);
#define PT_INIT if (threadIdx.x == 0) for (int q_ = 0; q_ < 16; ++q_) pt_sh[q_] = 0ull;
#define PT_FLUSH(P) if (threadIdx.x == 0) for (int q_ = 0; q_ < 16; ++q_) (P).phase_ns[VBID * 16 + q_] += pt_sh[q_];
#else
#define PT_DECL
#define PT_START
#define PT_LAP(P, ph)
#define PT_ADD(ph, v)
#define PT_INIT
#define PT_FLUSH(P)
#endif

// Virtual CTA index / count of the persistent kernel: blockIdx.x / gridDim.x
// shifted by the problem's slice of the grid (P.vbase, P.vgrid), which is the
// whole grid except in the multi-rank test launch (dlmpc_multi_kernel: the
// ranks of a graph-partitioned solve as contiguous CTA slices of ONE
// cooperative grid on one GPU, so the device-side exchange is tested without
// separate launches that wait on one another). Read from the kernel
// parameters (constant bank): a per-CTA shared-memory copy measured 4%
// slower on the C4 cells.
// The production translation unit (dlmpc.cu) uses the builtins: reading the
// slice from the parameters there measured 40% slower on C2 (a codegen
// effect in the register-capped patch kernel), so only the multi-rank test
// kernel's own translation unit (dlmpc_multi.cu) defines DLMPC_VB_SHIFT.
#ifdef DLMPC_VB_SHIFT
#define VBID (static_cast<int>(blockIdx.x) - (P).vbase)
#define VGRID ((P).vgrid)
#else
#define VBID (static_cast<int>(blockIdx.x))
#define VGRID (static_cast<int>(gridDim.x))
#endif

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kBadNone = 0x7f7f7f7f;   // cudaMemset(0x7f) pattern = "no infeasible row"
constexpr int kMG1 = 4;                // m-tiles per GEMM-1 work unit
constexpr int kMG2 = 2;                // m-tiles per GEMM-2 work unit

enum Mode { kPatch = 0, kTwoPhase = 1, kExact = 2, kStream = 3,
            kPatchRb = 4 };   // kPatch with the register-blocked GEMV pair (P.rb_gemv)

struct DevProblem {
  int n_sub, n_rows, n_cols, n_inputs, s_pad, exact, contiguous, d_row;
  int own_sub_lo, own_sub_hi, own_col_lo, own_col_hi;   // owned range (graph partition)
  double rho;
  const int64_t* row_start; const int64_t* ball_ptr; const int* ball_idx; const int* ball_off;
  const int* state_start; const int* state_count; const int* sub_first_bad;
  int d_pad; const int* supp_col; const int* supp_off; const int* supp_len;
  const double* row_w; const double* row_lo; const double* row_hi;
  const int* col_owner; const int* col_len; const int* col_class; const int* col_vec; const int* col_irow;
  const int64_t* col_rowbase;
  int n_classes; const int* class_s; const int* class_n0; const int* class_ldn;
  const int64_t* class_null_off; const double* null_pool; const double* q_pool;
  const int* class_m; const int64_t* class_g_off; const int64_t* class_p_off;
  const double* g_pool; const double* p_pool; int m_pad; const double* rhs_pool; const int* ref_pos;
  int n_tiles, tile_cols; const int* tile_class; const int* tile_first; const int* tile_count;
  const int* tile_colv;
  const int64_t* a_ptr; const int* a_idx; const double* a_val;
  const int64_t* b_ptr; const int* b_idx; const double* b_val;
  const int* input_owner; const int* input_local;
  // audit tables (optional)
  const int* class_ntouch; const int64_t* class_g0_off; const double* g0_pool;
  const int64_t* class_perm_off; const int* perm_pool; const int* col_pin;
  // patch work units (built by the library at create time)
  const int* cta_unit_ptr;     // [grid+1]
  const int* unit_sub_lo;      // own subsystems [lo, hi)
  const int* unit_sub_hi;
  const int* unit_patch_lo;    // halo subsystems [lo, hi) whose rows the unit's columns touch
  const int* unit_patch_hi;
  const int* unit_chunk_ptr;   // [n_units+1]
  const int* chunk_class; const int* chunk_col0; const int* chunk_n;
  // mutable device state
  double* psi[2]; double* lam[2]; double* s_row; double* ada; double* x[2]; double* u;
  unsigned long long* resid;   // [2 * cap] residual maxima per iteration (ordered bits)
  unsigned* gbar;              // patch modes: monotonic grid-barrier arrival counter (never reset)
  int* ctl;                    // 0 status, 1 fail step, 2/3 bad-row slots, 4 cur buffer, 5 fail iters
  unsigned long long* phase_ns;   // [grid * 16] (profiling build only)
  // shared-memory plan (offsets in doubles)
  int opr_cap;                 // doubles of the per-CTA operator region at smem offset 0
  int s8_max, n08_max, ldk, ldy, split_max, patch_cap, cache_phi;
  int off_k, off_y, off_yp, off_red, off_meta, off_patch, off_phimeta, off_ex;
  int off_stash, stash_bufs;   // cp.async staging of chunk ψ,λ: [bufs][TC][2][ldk]
  // stream mode: per-unit partials of the next iteration's Φ dots. Subsystem
  // i's rows receive one partial from each unit a_i..a_i+n_i-1 whose patch
  // holds i, stored at part_off[i] + (unit - a_i) * rows_i + l; ping-pong
  // by iteration parity.
  const int64_t* part_off; const int* part_first; const int* part_n;
  double* part_buf[2];
  int off_cpatch;
  double* row_invden;          // stream mode: 1/(ρ + 2w·||a||²) per row of the current MPC step
  const int* cta_gop;          // stream mode: CTA reads its class operator from L2 (does not fit)
  int off_chtab, ch_cap;       // per-unit chunk table: [ch_cap][8] ints (k, c0, nt, S, n08, ldn)
  int off_ptab, np_cap;        // per-unit patch-subsystem table: [np_cap][6] doubles
  int tab_alt;                 // stream mode: doubles from the unit tables (chunk, patch, 1/‖a‖²) to their second copy
  int off_rowq;                // per patch row: its patch-subsystem index (int)
  int off_pada;                // per patch subsystem: ||a||^2 of this MPC step
  int off_udesc;               // two unit descriptors (16 ints each)
  int off_ublk;                // patch mode, cached single unit: unit block + per-subsystem row info
  int off_bar;                 // 3 mbarriers (ψ buffers, λ buffer)
  // stream mode, host-built control tables (one coalesced copy per unit):
  //   unit_desc [u][16] ints: own_lo, own_hi, plo, phi, prow0 (2 ints), prows, ch_a, ch_b, pt_off,
  //     nt and c0 of the first chunk, nt of the second (0 if none), -, -, -
  //   chunk_desc [ch][8 + 2*TC] ints: k, c0, nt, S, n08, ldn, paired, -, then per column slot t
  //     s0 (row of support slot 0, unit-local) and q (particular-solution vector index)
  //   unit_ptab [pt_off + q][6] doubles: (rowoff, rows, slots, own slot) ints | part_off | - | r0 | (own, -)
  const int* unit_desc; const int* chunk_desc; const double* unit_ptab;
  int ldl;                     // stream mode: row stride of the λ stash
  int warp_spec;               // stream mode: producer/consumer warp specialisation
  int small_gemv;              // patch mode: DFMA GEMV for GEMM 1 of chunks with <= 2 columns
  int rb_gemv;                 // patch mode, TC 8: register-blocked GEMV pair for chunks of <= 2 columns
  int stash_cols;              // columns per ψ,λ staging buffer (TC, or 2 with rb_gemv)
  int g1_mrow;                 // GEMM 1 by whole m-rows where it pays (DLMPC_G1_MROW=0 disables: A/B tests)
  // checked build (-DDLMPC_CHECKED, libdlmpc_checked.so): the first out-of-range
  // access is recorded here (code, then the offending index) and skipped
  int* dbg;                    // [4]: code, -, index (long long)
  // patch mode, K-split pairs: per CTA -1 or partner * 2 + half; the two CTAs
  // run the same unit on halves of the support rows and swap partial Y
  const int* cta_pair;
  unsigned* pair_flag;         // [grid] partial-Y publications (monotonic per launch)
  double* ypair;               // [grid][2][n08_max * TC] partial Y, double-buffered
  // graph-partitioned solve with the exchange on the device (P.dist, non-patch
  // modes): see dist_exchange. Peer pointers address the neighbour ranks'
  // device memory (NVLink P2P; the same device in the one-launch test).
  int dist, d_rank, d_world, d_npeer;
  long long d_nsend;
  const long long* d_send_src;       // [d_nsend] this rank's cells (internal layout)
  const long long* d_send_dst;       // [d_nsend] the destination rank's cells
  const int* d_send_peer;            // [d_nsend] destination (index into the peer tables)
  double* const* d_peer_psi;         // [d_npeer * 2] destination ψ buffers
  double* const* d_peer_lam;         // [d_npeer * 2] destination λ buffers
  unsigned* const* d_peer_flag;      // [d_npeer] their halo arrival counters
  unsigned* d_flag;                  // own halo arrival counter (monotonic, never reset)
  unsigned d_halo_per_iter;          // its increments per iteration (CTAs of all sending peers)
  unsigned long long* const* d_all_slots;   // [d_world] every rank's residual slots [2][world][2]
  unsigned* const* d_all_rflag;      // [d_world] every rank's residual arrival counter
  unsigned* d_rflag;                 // own residual arrival counter
  unsigned long long* d_slots;       // own residual slots
  int* d_abort;                      // set on an exchange timeout (all CTAs then stop)
  int vbase, vgrid;                  // this problem's CTA slice of the launch (VBID / VGRID)
  long long part_cap;          // stream mode: doubles per Φ-partials buffer
  long long smem_doubles;      // dynamic shared memory of the plan
  // patch mode, cached single unit: the closed loop's MPC-step transition
  // inside each CTA, without grid barriers (fused_transition), from per-unit
  // step-invariant tables (FuseTab) staged in shared memory at launch
  int fuse_steps;
  const int* ft_iptr; const int* ft_int;       // [n_units+1] offsets, int tables
  const int* ft_dptr; const double* ft_dbl;    // [n_units+1] offsets, A / B values
  int off_fw, ft_dcap, ft_w2cap, ft_wcap, ft_ucap;   // shared memory region and its section capacities
  // patch modes: the class sizes in shared memory (class_dims), staged at
  // launch; -1: none (other modes, or too many classes)
  int off_ctab;
};

// A unit's window for fused_transition: W = the states of its patch
// subsystems' supports, U = the inputs W's B rows reference plus the unit's
// own inputs, W2 = the states W's A rows read (all ascending). Int table:
// a header of offsets (kHeader ints), then the sections below; the double
// table holds the A values (in CSR order, per W state) then the B values.
struct FuseTab {
  enum {
    kNw, kNu, kNw2, kNa, kNint,
    kWcol,    // [nw]     r * 2 + (r is an own state)
    kW2,      // [nw2]    state
    kSupp,    // [np * d_pad] window index of each patch-subsystem support slot
    kMx,      // [nt]     window index of the single chunk's columns
    kUhead,   // [nu][4]  k * 2 + own, s_row index, support length D, entry offset
    kUent,    // [..][2]  per support slot of input k's row: ψ/λ position, column
    kAoff,    // [nw+1]   A entries of W state j, then [nw+1] its B entries
    kAent,    // [na]     W2 index
    kBent,    // [nb]     U index
    kHeader = 16
  };
};

struct RunArgs {
  int t_sim, closed_loop, warm_start, cold_start, max_iters, stop_on_conv;
  int it_base;         // iterations already run on this state (host-driven iterate calls): the
                       // stream kernel continues its Φ-dot partials instead of a full Φ
  unsigned dist_epoch;  // P.dist: iterations of the earlier launches (the counters' base)
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

// A class's sizes and basis offset: from the shared-memory table of the patch
// modes (P.off_ctab, staged at launch), else from the global tables. The
// iteration barrier's acquire invalidates L1, so right after it every global
// table load is an L2 round trip on the chunk's critical path.
struct ClassDims { int s, n0, ldn; long long off; };
__device__ __forceinline__ ClassDims class_dims(const DevProblem& P, const double* smem, int k) {
  if (P.off_ctab >= 0) {
    const int* ci = reinterpret_cast<const int*>(smem + P.off_ctab) + 4 * k;
    const long long* co = reinterpret_cast<const long long*>(smem + P.off_ctab + 2 * P.n_classes);
    return {ci[0], ci[1], ci[2], co[k]};
  }
  return {P.class_s[k], P.class_n0[k], P.class_ldn[k], P.class_null_off[k]};
}
__device__ __forceinline__ void class_table_load(const DevProblem& P, double* smem) {   // all threads
  if (P.off_ctab < 0) return;
  int* ci = reinterpret_cast<int*>(smem + P.off_ctab);
  long long* co = reinterpret_cast<long long*>(smem + P.off_ctab + 2 * P.n_classes);
  for (int k = threadIdx.x; k < P.n_classes; k += kThreads) {
    ci[4 * k] = P.class_s[k]; ci[4 * k + 1] = P.class_n0[k]; ci[4 * k + 2] = P.class_ldn[k]; ci[4 * k + 3] = 0;
    co[k] = P.class_null_off[k];
  }
}


// Bounds checks of the checked build (there is no compute-sanitizer on the
// GPU pool): DCHK(P, cond, code, idx) records the first failing (code, idx)
// in P.dbg and returns false so the caller skips the access; the host turns a
// recorded violation into DLMPC_CUDA_ERROR. In the production build it is
// the constant `true` and compiles away.
#ifdef DLMPC_CHECKED
static __device__ __noinline__ bool dchk_fail(int* dbg, int code, long long idx) {
  if (atomicCAS(dbg, 0, code) == 0) reinterpret_cast<long long*>(dbg)[1] = idx;
  return false;
}
#ifndef DLMPC_CHECKED_NODCHK
#define DCHK(P, cond, code, idx) ((cond) ? true : dchk_fail((P).dbg, (code), static_cast<long long>(idx)))
#else
#define DCHK(P, cond, code, idx) true
#endif
// the fields DCHK_CELL reads, for code that holds no DevProblem (StreamEpi)
struct CellChk { int* dbg; int own_col_lo, own_col_hi, s_pad; const int* col_len; };
#else
#define DCHK(P, cond, code, idx) true
#endif
// the owned support cell `pos` of the column layout (epilogue stores)
#define DCHK_CELL(P, pos, code)                                                                      \
  DCHK(P, (pos) >= static_cast<long long>((P).own_col_lo) * (P).s_pad &&                              \
              (pos) < static_cast<long long>((P).own_col_hi) * (P).s_pad &&                           \
              ((pos) % (P).s_pad) < (P).col_len[(pos) / (P).s_pad], code, pos)
#define DCHK_ROW(P, r, code) DCHK(P, (r) >= 0 && (r) < (P).n_rows, code, r)

__device__ __forceinline__ void cp_async16(double* smem_dst, const double* gmem_src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" :: "r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" :: "n"(N) : "memory"); }

// TMA 1-D bulk copies completing on shared-memory mbarriers (stream mode).
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile("{\n .reg .pred P1;\n LAB_WAIT:\n"
               " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
               " @P1 bra DONE;\n bra LAB_WAIT;\n DONE:\n}\n" :: "r"(smem_u32(bar)), "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// Generic-proxy global stores (the stream epilogue's ψ', λ') that other CTAs
// read with TMA bulk copies (async proxy) after the next grid barrier: the
// writers order them for the async proxy before arriving (PTX memory model,
// proxy fences).
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;\n" ::: "memory"); }

// Stage ψ,λ of nt consecutive columns starting at c0 into `st`
// ([t][ψ|λ][ldk]) with 16-byte cp.async copies (bypassing L1, like ld.cg);
// commits one group. s_pad is a multiple of 4, so sources are 16-B aligned.
__device__ __forceinline__ void stash_issue(const DevProblem& P, int c0, int nt, int S, const double* psi,
                                            const double* lam, double* st) {
  const int pairs = (S + 1) >> 1;
  const int total = nt * 2 * pairs;
  for (int q = threadIdx.x; q < total; q += blockDim.x) {
    const int t = q / (2 * pairs), r = q - t * 2 * pairs;
    const int arr = r >= pairs, pr = r - arr * pairs;
    const double* src = (arr ? lam : psi) + static_cast<size_t>(c0 + t) * P.s_pad + 2 * pr;
    cp_async16(st + (2 * t + arr) * P.ldk + 2 * pr, src);
  }
  cp_async_commit();
}

// Patch mode without staging buffers: the first chunk's ψ, λ lines into L1
// under the Φ stage (no registers held); the chunk's prologue and epilogue
// read them with plain loads. Legal right after the iteration barrier: its
// acquire invalidated L1, and buffer b is read-only until the next barrier.
__device__ __forceinline__ void chunk_prefetch_l1(const double* psi, const double* lam, int c0, int nt, int s_pad) {
  const long long n = static_cast<long long>(nt) * s_pad;   // doubles per array
  const long long lines = (n + 15) / 16;                    // 128-byte lines
  const double* b0 = psi + static_cast<long long>(c0) * s_pad;
  const double* b1 = lam + static_cast<long long>(c0) * s_pad;
  for (long long q = threadIdx.x; q < 2 * lines; q += kThreads) {
    const double* a = (q < lines ? b0 : b1) + 16 * (q < lines ? q : q - lines);
    asm volatile("prefetch.global.L1 [%0];\n" :: "l"(a));
  }
}

template <bool EXACT>
__device__ __forceinline__ double make_phi(double v, double s, double xc) {
  return EXACT ? __dadd_rn(v, __dmul_rn(s, xc)) : fma(s, xc, v);
}

// numpy pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
// pairwise_sum_DOUBLE) of rounded products f(i); the reference's Ψ
// reductions `.sum(axis=2)` (admm.py:184, 186) use it. Blocks of <= 128 are
// the 8-accumulator leaf; longer ranges split at n/2 rounded down to a
// multiple of 8 and add the two halves.
template <class F>
__device__ __forceinline__ double pairwise_leaf(const F& f, int lo, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, f(lo + i));
    return r;
  }
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

// The recursion as an explicit post-order walk (no device recursion: its
// stack depth is not statically bounded, and n >= ~900 -- the d=5, T=30
// supports -- overflowed the default per-thread stack). Depth <= 24 covers
// n < 128 * 2^23.
template <class F>
__device__ double pairwise_sum(const F& f, int lo, int n) {
  if (n <= 128) return pairwise_leaf(f, lo, n);
  int st_lo[24], st_n[24];
  double st_left[24];
  bool st_right[24];
  int top = 0;
  st_lo[0] = lo; st_n[0] = n; st_right[0] = false;
  double ret = 0.0;
  for (;;) {
    const int cl = st_lo[top], cn = st_n[top];
    if (cn > 128 && !st_right[top]) {   // descend into the left half
      int n2 = cn / 2;
      n2 -= n2 % 8;
      st_right[top] = true;
      ++top;
      st_lo[top] = cl; st_n[top] = n2; st_right[top] = false;
      continue;
    }
    ret = pairwise_leaf(f, cl, cn);     // a leaf: unwind
    for (;;) {
      if (top == 0) return ret;
      --top;
      const int pn = st_n[top];
      int n2 = pn / 2;
      n2 -= n2 % 8;
      if (st_lo[top + 1] == st_lo[top]) {   // came back from the left half: start the right one
        st_left[top] = ret;
        ++top;
        st_lo[top] = st_lo[top - 1] + n2; st_n[top] = pn - n2; st_right[top] = false;
        break;
      }
      ret = __dadd_rn(st_left[top], ret);   // came back from the right half: combine
    }
  }
}

struct ProdRow {   // row[j] * v[j]
  const double* row; const double* v;
  __device__ double operator()(int j) const { return __dmul_rn(row[j], v[j]); }
};

// Max of residual magnitudes that lets NaN win, as np.max does (reference
// admm.py:216-217, strategies.py:178-183): the operands are compared as their
// bit patterns with the sign cleared, so NaN > +inf > every finite value and
// a diverging iterate publishes NaN (the stop test `NaN <= eps` then fails
// and the solve ends in NotConverged) instead of fmax silently dropping it.
// Also |b| for free: rmax(acc, d) == max(acc, |d|) for acc >= 0.
__device__ __forceinline__ double rmax(double a, double b) {
#ifdef DLMPC_FMAX_RESID
  return fmax(a, fabs(b));
#else
  const long long ia = __double_as_longlong(a) & 0x7fffffffffffffffLL;
  const long long ib = __double_as_longlong(b) & 0x7fffffffffffffffLL;
  return __longlong_as_double(ia > ib ? ia : ib);
#endif
}

__device__ __forceinline__ double block_max(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = rmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double m = 0.0;
  if (threadIdx.x < 32) {
    m = threadIdx.x < kWarps ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) m = rmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  }
  return m;   // valid in thread 0
}

__device__ __forceinline__ void publish_residuals(const DevProblem& P, int it, double pri_m,
                                                  double dual_m, double* red) {
  for (int o = 16; o > 0; o >>= 1) {
    pri_m = rmax(pri_m, __shfl_xor_sync(0xffffffffu, pri_m, o));
    dual_m = rmax(dual_m, __shfl_xor_sync(0xffffffffu, dual_m, o));
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { red[2 * warp] = pri_m; red[2 * warp + 1] = dual_m; }
  __syncthreads();
  if (warp == 0) {
    double p = lane < kWarps ? red[2 * lane] : 0.0, d = lane < kWarps ? red[2 * lane + 1] : 0.0;
    for (int o = 16; o > 0; o >>= 1) {
      p = rmax(p, __shfl_xor_sync(0xffffffffu, p, o));
      d = rmax(d, __shfl_xor_sync(0xffffffffu, d, o));
    }
    if (lane == 0) {
      atomicMax(P.resid + 2 * it, static_cast<unsigned long long>(__double_as_longlong(p)));
      atomicMax(P.resid + 2 * it + 1, static_cast<unsigned long long>(__double_as_longlong(d)));
    }
  }
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Patch modes: the residual publish fused with the grid barrier. The block
// reduction's __syncthreads doubles as the barrier's entry; thread 0 posts
// the CTA's residual maxima, arrives on the launch-wide monotonic counter
// (release: the CTA's ψ, λ stores, ordered by that __syncthreads, and the
// two atomics become visible first) and polls it (acquire) until every CTA
// has arrived `target` times in total (wrap-safe compare). One block barrier
// less per iteration than publish_residuals + grid.sync(); the grid barrier
// itself costs ~1.2 us either way on B200 (tools/microbench/barrier_bench.cu).
__device__ __forceinline__ void publish_barrier(const DevProblem& P, unsigned long long* rs, double pri_m,
                                                double dual_m, double* red, unsigned target) {
  for (int o = 16; o > 0; o >>= 1) {
    pri_m = rmax(pri_m, __shfl_xor_sync(0xffffffffu, pri_m, o));
    dual_m = rmax(dual_m, __shfl_xor_sync(0xffffffffu, dual_m, o));
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { red[2 * warp] = pri_m; red[2 * warp + 1] = dual_m; }
  __syncthreads();
  if (warp == 0) {
    double p = lane < kWarps ? red[2 * lane] : 0.0, d = lane < kWarps ? red[2 * lane + 1] : 0.0;
    for (int o = 16; o > 0; o >>= 1) {
      p = rmax(p, __shfl_xor_sync(0xffffffffu, p, o));
      d = rmax(d, __shfl_xor_sync(0xffffffffu, d, o));
    }
    if (lane == 0) {
      atomicMax(rs, static_cast<unsigned long long>(__double_as_longlong(p)));
      atomicMax(rs + 1, static_cast<unsigned long long>(__double_as_longlong(d)));
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" :: "l"(P.gbar) : "memory");
      while (static_cast<int>(ld_acquire_u32(P.gbar) - target) < 0) {}
    }
  }
  __syncthreads();
}

// Per-MPC-step stages run a few hundred latency-bound items (subsystems,
// inputs, state rows), one warp per item: the lanes load an item's operands
// at once (one round trip), then the products are summed across the lanes in
// the reference's sequential order (warp_ordered_sum). Item q goes to CTA
// q % grid first, so the items spread over the SMs.
__device__ __forceinline__ long long wspread_first(const DevProblem& P) {
  return static_cast<long long>(threadIdx.x >> 5) * VGRID + VBID;
}
__device__ __forceinline__ long long wspread_step(const DevProblem& P) {
  return static_cast<long long>(VGRID) * (blockDim.x >> 5);
}

// acc (+)= v_0 + v_1 + ... + v_{n-1} over lanes 0..n-1, strictly in that
// order with IEEE adds; `first`: acc is not yet set (the reference starts
// from the first product, not from 0). Result in every lane.
__device__ __forceinline__ double warp_ordered_sum(double acc, bool& first, double v, int n) {
  for (int q = 0; q < n; ++q) {
    const double t = __shfl_sync(0xffffffffu, v, q);
    acc = first ? t : __dadd_rn(acc, t);
    first = false;
  }
  return acc;
}

// ||a||^2 per subsystem (reference sls_core.py:338-339: all rows of a
// subsystem share the support, hence a_pad and a_dot_a) and the RowInfeasible
// scan of sls_core.py:346-348. Strict ascending order, no FMA, in all modes.
static __device__ void row_data_stage(const DevProblem& P, const double* x, int* bad_slot) {
  const int lane = threadIdx.x & 31;
  for (long long ii = wspread_first(P); ii < P.n_sub; ii += wspread_step(P)) {
    const int i = static_cast<int>(ii);
    const int D = P.supp_len[i];
    const int* sc = P.supp_col + static_cast<size_t>(i) * P.d_pad;
    double acc = 0.0;
    bool first = true;
    for (int k0 = 0; k0 < D; k0 += 32) {
      const int kn = min(32, D - k0);
      const double xc = lane < kn ? ld_cg(x + sc[k0 + lane]) : 0.0;
      acc = warp_ordered_sum(acc, first, __dmul_rn(xc, xc), kn);
    }
    if (D < P.d_row) acc = __dadd_rn(acc, 0.0);   // the padded slots of a_pad
    if (lane == 0) {
      P.ada[i] = acc;
      if (acc == 0.0 && P.sub_first_bad[i] >= 0 && i >= P.own_sub_lo && i < P.own_sub_hi)
        atomicMin(bad_slot, P.sub_first_bad[i]);
    }
  }
}

// Φ scale of the rows of subsystem i (one warp; lanes = rows). Lane k first
// holds the k-th (column, block offset, x_c) of the shared row support; the
// row lanes then read their ψ,λ entries 8 support columns at a time.
// Calls `out(row_local, s)` for every row.
template <bool EXACT, class Out>
__device__ __forceinline__ void phi_rows_of(const DevProblem& P, int i, const double* psi,
                                            const double* lam, const double* x, const Out& out,
                                            double* inv_den_out = nullptr) {
  const int lane = threadIdx.x & 31;
  const int D = P.supp_len[i];
  const int* sc = P.supp_col + static_cast<size_t>(i) * P.d_pad;
  const int* so = P.supp_off + static_cast<size_t>(i) * P.d_pad;
  const long long r0 = P.row_start[i];
  const int nr = static_cast<int>(P.row_start[i + 1] - r0);
  const double ada = ld_cg(P.ada + i);
  const double rho = P.rho;
  for (int l0 = 0; l0 < nr; l0 += 32) {
    const int l = l0 + lane;
    const bool row_ok = l < nr;
    double w = 0.0, lo = 0.0, hi = 0.0;
    if (row_ok) { w = P.row_w[r0 + l]; lo = P.row_lo[r0 + l]; hi = P.row_hi[r0 + l]; }
    double acc = 0.0;
    bool first = true;
    for (int k0 = 0; k0 < D; k0 += 32) {
      const int kn = min(32, D - k0);
      long long base_k = 0;
      double x_k = 0.0;
      if (lane < kn) {
        const int c = sc[k0 + lane];
        base_k = static_cast<long long>(c) * P.s_pad + so[k0 + lane];
        x_k = ld_cg(x + c);
      }
      for (int u0 = 0; u0 < kn; u0 += 8) {
        double pv[8], lv[8], xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const long long bk = __shfl_sync(0xffffffffu, base_k, (u0 + u) & 31);
          xv[u] = __shfl_sync(0xffffffffu, x_k, (u0 + u) & 31);
          pv[u] = 0.0; lv[u] = 0.0;
          if (row_ok && u0 + u < kn &&
              DCHK(P, bk + l >= 0 && bk + l < static_cast<long long>(P.n_cols) * P.s_pad, 9, bk + l)) {
            pv[u] = ld_cg(psi + bk + l);
            lv[u] = ld_cg(lam + bk + l);
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (u0 + u < kn) {
            const double v = __dsub_rn(pv[u], lv[u]);
            if (EXACT) {
              const double pr = __dmul_rn(v, xv[u]);
              acc = first ? pr : __dadd_rn(acc, pr);
              first = false;
            } else {
              acc = fma(v, xv[u], acc);
            }
          }
        }
      }
    }
    if (!row_ok) continue;
    if (EXACT && D < P.d_row) acc = __dadd_rn(acc, 0.0);
    // y0 = ρc/(ρ + 2w·ada); clip; s = (y - c)/ada   (admm.py:162-166)
    const double den = __dadd_rn(rho, __dmul_rn(__dmul_rn(2.0, w), ada));
    if (inv_den_out) inv_den_out[l] = 1.0 / den;   // stream mode: later iterations multiply
    const double y0 = __ddiv_rn(__dmul_rn(rho, acc), den);
    const double y = fmin(fmax(y0, lo), hi);
    out(l, ada > 0.0 ? __ddiv_rn(__dsub_rn(y, acc), ada) : 0.0);
  }
}

// Grid-wide Φ stage of the two-phase kernels: s_r -> global s_row.
template <bool EXACT>
__device__ void phi_stage_global(const DevProblem& P, int b, const double* x) {
  const int gw = VBID * kWarps + (threadIdx.x >> 5), GW = VGRID * kWarps;
  for (int i = gw; i < P.n_sub; i += GW) {
    double* dst = P.s_row + P.row_start[i];
    phi_rows_of<EXACT>(P, i, P.psi[b], P.lam[b], x, [dst](int l, double s) { dst[l] = s; });
  }
}

// ---------------------------------------------------------------------------
// The two FP64 tensor-core GEMMs of the Ψ projection against a class's
// null-space basis N ([S8][ldn] at `nop`, smem or global):
//   GEMM 1  Y[a][t] = sum_p N[p][a] K[t][p]     (M = n0, N = TC, K = S)
//   GEMM 2  O[t][p] = sum_a N[p][a] Y[a][t]     (M = S,  N = TC, K = n0)
// K is read from kt [TC][ldk]; Y goes to yb [n08][ldy] (split-K partials in
// yp). GEMM 2 hands its accumulators to `epi` (prefetch(mt) before the k
// loop, store(mt, nn, c0, c1) after: rows mt*8+g, columns nn*8+2tig, +1).
// ---------------------------------------------------------------------------
struct NoHook { __device__ __forceinline__ void operator()() const {} };
struct CtaBar { __device__ __forceinline__ void operator()() const { __syncthreads(); } };

// named barriers (id 0 is __syncthreads)
__device__ __forceinline__ void nbar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" :: "r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;\n" :: "r"(id), "r"(n) : "memory");
}
template <int NW>
struct GroupBar {   // barrier over the first NW warps
  __device__ __forceinline__ void operator()() const { nbar_sync(1, NW * 32); }
};

// NW warps (warp ids 0..NW-1) run the GEMMs; `sync` is their barrier.
template <int TC, class Hook = NoHook, int NW = kWarps, class Sync = CtaBar, int MROW = 0>
__device__ __forceinline__ void gemm1(const DevProblem& P, int SK, int n08, int ldn, const double* nop,
                                      const double* kt, int ldk, double* yb, int ldy, double* yp,
                                      const Hook& before_sync = Hook(), const Sync& sync = Sync()) {
  constexpr int NTN = TC / 8;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tig = lane & 3;
  const int mt1 = n08 >> 3, ks1 = SK >> 2;   // SK: K extent, a multiple of 4
  // m-tiles [0, mr) by whole m-rows (patch mode, MROW): a warp takes both
  // n-tiles of an m-tile and each basis fragment feeds all NTN tiles (0.75
  // instead of 1 fragment byte per FLOP at NTN = 2). All m-tiles that way
  // when it costs no extra round, else the largest multiple of NW, the rest
  // one (m, n) tile per warp below -- the same round count as all tiles. C4
  // at N=1000: d=6,T=20 87.4 -> 77.6 us/iter, d=4,T=30 93.1 -> 84.1, d=6,T=30
  // 265 -> 249, d=5,T=10 (12 m-tiles) 27.5 -> 25.6. The stream kernel keeps MROW off (its 7 m-tiles over 16 warps
  // would lose a round; with the branch merely compiled in it measured 2-3%
  // slower). Per tile the same two chains and order as below: Y is bitwise
  // the same.
  int mr = 0;
  if (MROW && NTN > 1 && DLMPC_G1_MROW && P.g1_mrow)   // P.g1_mrow: runtime switch (tests: bitwise A/B)
    mr = (mt1 + NW - 1) / NW * NTN <= (mt1 * NTN + NW - 1) / NW ? mt1 : mt1 / NW * NW;
  else if (MROW == 2 && NTN > 1)
    mr = mt1;
  if (mr > 0) {
    for (int mt = warp; mt < mr; mt += NW) {
      double ca[NTN][2], cb[NTN][2];
#pragma unroll
      for (int nn = 0; nn < NTN; ++nn) { ca[nn][0] = ca[nn][1] = cb[nn][0] = cb[nn][1] = 0.0; }
      int ks = 0;
      for (; ks + 1 < ks1; ks += 2) {
        const int p0 = ks * 4 + tig, p1 = p0 + 4;
        const double a0 = nop[p0 * ldn + mt * 8 + g], a1 = nop[p1 * ldn + mt * 8 + g];
#pragma unroll
        for (int nn = 0; nn < NTN; ++nn) {
          dmma(ca[nn][0], ca[nn][1], a0, kt[(nn * 8 + g) * ldk + p0]);
          dmma(cb[nn][0], cb[nn][1], a1, kt[(nn * 8 + g) * ldk + p1]);
        }
      }
      if (ks < ks1) {
        const int p0 = ks * 4 + tig;
        const double a0 = nop[p0 * ldn + mt * 8 + g];
#pragma unroll
        for (int nn = 0; nn < NTN; ++nn) dmma(ca[nn][0], ca[nn][1], a0, kt[(nn * 8 + g) * ldk + p0]);
      }
#pragma unroll
      for (int nn = 0; nn < NTN; ++nn) {
        yb[(mt * 8 + g) * ldy + nn * 8 + 2 * tig] = ca[nn][0] + cb[nn][0];
        yb[(mt * 8 + g) * ldy + nn * 8 + 2 * tig + 1] = ca[nn][1] + cb[nn][1];
      }
    }
    if (mr == mt1) {
      before_sync();
      sync();
      return;
    }
  }
  if (mr > 0 || mt1 * NTN >= 12 || P.split_max == 1) {
    // enough (m, n) tiles to keep the DMMA pipe busy (or no room for split-K
    // partials): one tile per warp over the full K with two interleaved
    // accumulator chains, no split-K pass
    for (int u = warp; u < (mt1 - mr) * NTN; u += NW) {
      const int mt = mr + u / NTN, nn = u - (u / NTN) * NTN;
      double c0a = 0.0, c1a = 0.0, c0b = 0.0, c1b = 0.0;
      int ks = 0;
      for (; ks + 1 < ks1; ks += 2) {
        const int p0 = ks * 4 + tig, p1 = p0 + 4;
        const double a0 = nop[p0 * ldn + mt * 8 + g], b0 = kt[(nn * 8 + g) * ldk + p0];
        const double a1 = nop[p1 * ldn + mt * 8 + g], b1 = kt[(nn * 8 + g) * ldk + p1];
        dmma(c0a, c1a, a0, b0);
        dmma(c0b, c1b, a1, b1);
      }
      if (ks < ks1) {
        const int p0 = ks * 4 + tig;
        dmma(c0a, c1a, nop[p0 * ldn + mt * 8 + g], kt[(nn * 8 + g) * ldk + p0]);
      }
      yb[(mt * 8 + g) * ldy + nn * 8 + 2 * tig] = c0a + c0b;
      yb[(mt * 8 + g) * ldy + nn * 8 + 2 * tig + 1] = c1a + c1b;
    }
    before_sync();
    sync();
    return;
  }
  const int groups1 = (mt1 + kMG1 - 1) / kMG1;
  int split = 1;
  while (groups1 * split * 2 <= NW && split < P.split_max) split <<= 1;
  for (int u = warp; u < groups1 * split; u += NW) {
    const int grp = u / split, sl = u - grp * split;
    const int mt0 = grp * kMG1;
    double acc[kMG1][NTN][2];
#pragma unroll
    for (int m = 0; m < kMG1; ++m)
#pragma unroll
      for (int nn = 0; nn < NTN; ++nn) { acc[m][nn][0] = 0.0; acc[m][nn][1] = 0.0; }
#pragma unroll 2
    for (int ks = sl; ks < ks1; ks += split) {
      const int p = ks * 4 + tig;
      double bf[NTN];
#pragma unroll
      for (int nn = 0; nn < NTN; ++nn) bf[nn] = kt[(nn * 8 + g) * ldk + p];
#pragma unroll
      for (int m = 0; m < kMG1; ++m) {
        if (mt0 + m < mt1) {
          const double af = nop[p * ldn + (mt0 + m) * 8 + g];
#pragma unroll
          for (int nn = 0; nn < NTN; ++nn) dmma(acc[m][nn][0], acc[m][nn][1], af, bf[nn]);
        }
      }
    }
    double* dst = split == 1 ? yb : yp + static_cast<size_t>(sl) * P.n08_max * TC;
    const int ld = split == 1 ? ldy : TC;
#pragma unroll
    for (int m = 0; m < kMG1; ++m) {
      if (mt0 + m < mt1) {
#pragma unroll
        for (int nn = 0; nn < NTN; ++nn) {
          dst[((mt0 + m) * 8 + g) * ld + nn * 8 + 2 * tig] = acc[m][nn][0];
          dst[((mt0 + m) * 8 + g) * ld + nn * 8 + 2 * tig + 1] = acc[m][nn][1];
        }
      }
    }
  }
  before_sync();
  sync();
  if (split > 1) {
    for (int idx = tid; idx < n08 * TC; idx += NW * 32) {
      const int a = idx / TC, t = idx - a * TC;
      double v = yp[idx];
      for (int sl = 1; sl < split; ++sl) v += yp[static_cast<size_t>(sl) * P.n08_max * TC + idx];
      yb[a * ldy + t] = v;
    }
    sync();
  }
}

template <int TC, class Epi, int NW = kWarps>
__device__ __forceinline__ void gemm2(int S8, int n08, int ldn, const double* nop, const double* yb, int ldy,
                                      Epi& epi) {
  constexpr int NTN = TC / 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tig = lane & 3;
  const int mt2 = S8 >> 3, ks2 = n08 >> 2;
  for (int mb = warp; mb < mt2; mb += NW * kMG2) {
#pragma unroll
    for (int m = 0; m < kMG2; ++m) epi.prefetch(m, mb + m * NW);
    double acc[kMG2][NTN][2];
#pragma unroll
    for (int m = 0; m < kMG2; ++m)
#pragma unroll
      for (int nn = 0; nn < NTN; ++nn) { acc[m][nn][0] = 0.0; acc[m][nn][1] = 0.0; }
#pragma unroll 4   // 2% faster than 2 on the stream kernel; C4 cells with T >= 20 or d = 6 5-6% faster
    for (int ks = 0; ks < ks2; ++ks) {
      const int a = ks * 4 + tig;
      double bf[NTN];
#pragma unroll
      for (int nn = 0; nn < NTN; ++nn) bf[nn] = yb[a * ldy + nn * 8 + g];
#pragma unroll
      for (int m = 0; m < kMG2; ++m) {
        const int mt = mb + m * NW;
        if (mt < mt2) {
          const double af = nop[(mt * 8 + g) * ldn + a];
#pragma unroll
          for (int nn = 0; nn < NTN; ++nn) dmma(acc[m][nn][0], acc[m][nn][1], af, bf[nn]);
        }
      }
    }
    epi.before_store();
#pragma unroll
    for (int m = 0; m < kMG2; ++m) {
      const int mt = mb + m * NW;
      if (mt < mt2) {
#pragma unroll
        for (int nn = 0; nn < NTN; ++nn) epi.store(m, mt, nn, acc[m][nn][0], acc[m][nn][1]);
      }
    }
  }
}

// GEMM 2 on the m16n8k8 FP64 shape (stream mode, DLMPC_STREAM_G2M16): warp w
// takes the 16-row tile w (two of gemm2's 8-row tiles) and each k8 step is
// ONE mma per n-tile instead of eight m8n8k4 -- 4x fewer tensor instructions
// for the same FLOPs and fragment loads. Fragment layouts verified by
// tools/microbench/dmma_layout.cu (g = lane>>2, t = lane&3):
//   A (16 x 8, row): a_i = A[g + 8*(i%2)][t + 4*(i/2)];  B (8 x 8, col): b_i = B[t + 4i][g]
//   C (16 x 8): c0, c1 = C[g][2t], C[g][2t+1];  c2, c3 = C[g+8][2t], C[g+8][2t+1]
// Rows past S8 (an odd number of 8-row tiles) read zeros. The epilogue sees
// the same (m, mt, nn, c0, c1) calls as gemm2's.
__device__ __forceinline__ void dmma16(double (&c)[4], const double (&a)[4], const double (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

template <int TC, class Epi, int NW = kWarps>
__device__ __forceinline__ void gemm2_m16(int S8, int n08, int ldn, const double* nop, const double* yb, int ldy,
                                          Epi& epi) {
  constexpr int NTN = TC / 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tig = lane & 3;
  const int mt2 = S8 >> 3, mt16 = (mt2 + 1) >> 1, ks8 = n08 >> 3;
  for (int w = warp; w < mt16; w += NW) {
    const int mt0 = 2 * w, mt1 = 2 * w + 1;
    const bool hi_ok = mt1 < mt2;
    epi.prefetch(0, mt0);
    if (hi_ok) epi.prefetch(1, mt1);
    double acc[NTN][4];
#pragma unroll
    for (int nn = 0; nn < NTN; ++nn) { acc[nn][0] = acc[nn][1] = acc[nn][2] = acc[nn][3] = 0.0; }
    const double* r_lo = nop + static_cast<size_t>(mt0 * 8 + g) * ldn;
    const double* r_hi = nop + static_cast<size_t>(mt1 * 8 + g) * ldn;
#pragma unroll 2
    for (int ks = 0; ks < ks8; ++ks) {
      const int k0 = ks * 8 + tig;
      double a[4];
      a[0] = r_lo[k0];
      a[2] = r_lo[k0 + 4];
      a[1] = hi_ok ? r_hi[k0] : 0.0;
      a[3] = hi_ok ? r_hi[k0 + 4] : 0.0;
#pragma unroll
      for (int nn = 0; nn < NTN; ++nn) {
        double bf[2];
        bf[0] = yb[k0 * ldy + nn * 8 + g];
        bf[1] = yb[(k0 + 4) * ldy + nn * 8 + g];
        dmma16(acc[nn], a, bf);
      }
    }
    epi.before_store();
#pragma unroll
    for (int nn = 0; nn < NTN; ++nn) {
      epi.store(0, mt0, nn, acc[nn][0], acc[nn][1]);
      if (hi_ok) epi.store(1, mt1, nn, acc[nn][2], acc[nn][3]);
    }
  }
}

// measured (tools/lib_ab.sh, fixed 200 iterations): N=3e3 26.01 -> 25.68,
// N=1e4 72.50 -> 72.40, N=1e5 642.6 -> 640.8 us/iter
#ifndef DLMPC_STREAM_G2M16
#define DLMPC_STREAM_G2M16 1
#endif

// GEMM 1 for chunks of at most two live columns (C2-sized networks): a DFMA
// GEMV, Y[a][t] = sum_p N[p][a] K[t][p], split over support slices whose
// partials are reduced in shared memory (`part`, >= 10*n08 doubles). Lanes
// walk consecutive a (conflict free for any ldn); K is a broadcast. Columns
// t >= nt of Y are zeroed for GEMM 2. Measured 1.2 vs 1.6 us (split-K DMMA).
template <int TC>
__device__ __forceinline__ void gemv1_small(int S, int n08, int ldn, const double* nop, const double* kt, int ldk,
                                            double* part, double* yb, int ldy, int nt) {
  constexpr int PS = 5;
  const int tid = threadIdx.x;
  const int a = tid % n08, rest = tid / n08;   // n08 x (t, ps)
  const int t = rest & 1, ps = rest >> 1;
  const int pl = (S + PS - 1) / PS;
  if (ps < PS && t < nt) {
    const int p0 = ps * pl, p1 = min(S, p0 + pl);
    const double* kr = kt + t * ldk;
    double c0 = 0.0, c1 = 0.0;
    int p = p0;
    for (; p + 1 < p1; p += 2) {
      c0 = fma(nop[p * ldn + a], kr[p], c0);
      c1 = fma(nop[(p + 1) * ldn + a], kr[p + 1], c1);
    }
    if (p < p1) c0 = fma(nop[p * ldn + a], kr[p], c0);
    part[(ps * 2 + t) * n08 + a] = c0 + c1;
  }
  __syncthreads();
  for (int idx = tid; idx < n08 * TC; idx += kThreads) {
    const int aa = idx / TC, tt = idx - aa * TC;
    double v = 0.0;
    if (tt < nt)
      for (int q = 0; q < PS; ++q) v += part[(q * 2 + tt) * n08 + aa];
    yb[aa * ldy + tt] = v;
  }
  __syncthreads();
}

// Register-blocked GEMV pair for chunks of <= 2 live columns (C2-sized
// networks), no tensor cores (north_star (4): warp shuffles for the small
// dense mat-vecs). Thread (warp w, lane l = 16h + j) owns the operator block
// rows p_i = w*PB + h*RB_PL + i (i < RB_PL) x columns a_c = j*RB_AL + c
// (c < RB_AL), staged thread-major (`opT[(i*RB_AL + c)*kThreads + tid]`, see
// stage_operator_rb) so each load is conflict free and the operator is read
// exactly once per GEMV.
//   GEMV 1  Y[a][t] = sum_p N[p][a] K[t][p]: 6 partials per thread, a
//           reduce-scatter over the two p halves (one shuffle per value), then
//           the 16 warps' partials summed in shared memory (`ypart`, 16*96).
//   GEMV 2  O[t][p] = sum_a N[p][a] Y[a][t]: 14 partials per thread reduced
//           over the 16 a lanes by a reduce-scatter (15 shuffles); lane j ends
//           with O[t = j>>3][p_(j&7)] and calls epi(p, t, o) for valid p < S.
// Requires S8 <= 16*2*RB_PL (PB = ceil(S8/16) <= 14) and n08 <= 16*RB_AL.
constexpr int RB_PL = 7, RB_AL_MAX = 4;   // rows per thread; operator columns per lane (<= 4)

__device__ __forceinline__ bool rb_fits(int S8, int n08) { return S8 <= 32 * RB_PL && n08 <= 16 * RB_AL_MAX; }

// Thread-major operator copy for gemv_pair_rb (class k, at smem offset 0).
template <int RB_AL>
__device__ __forceinline__ void stage_operator_rb(const DevProblem& P, int k, double* opT) {
  const int S = P.class_s[k], n0 = P.class_n0[k], ldn = P.class_ldn[k];
  const int PB = (((S + 7) & ~7) + 15) >> 4;
  const double* src = P.null_pool + P.class_null_off[k];
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31, h = l >> 4, j = l & 15;
#pragma unroll
  for (int i = 0; i < RB_PL; ++i) {
    const int pr = h * RB_PL + i, p = w * PB + pr;
#pragma unroll
    for (int c = 0; c < RB_AL; ++c) {
      const int a = j * RB_AL + c;
      opT[(i * RB_AL + c) * kThreads + tid] = (pr < PB && p < S && a < n0) ? __ldg(src + static_cast<size_t>(p) * ldn + a) : 0.0;
    }
  }
}

template <int RB_AL>
__device__ __forceinline__ void load_operator_rb(const double* opT, double (&op)[RB_PL][RB_AL]) {
#pragma unroll
  for (int i = 0; i < RB_PL; ++i)
#pragma unroll
    for (int c = 0; c < RB_AL; ++c) op[i][c] = opT[(i * RB_AL + c) * kThreads + threadIdx.x];
}

// kf(t, p): K[t][p] for p < S (called for this thread's rows only).
template <int RB_AL, class KF, class Epi>
__device__ __forceinline__ void gemv_pair_rb(int S, const double (&op)[RB_PL][RB_AL], const KF& kf,
                                             double* ypart, double* yb2, int nt, const Epi& epi) {
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31, h = l >> 4, j = l & 15;
  const int PB = (((S + 7) & ~7) + 15) >> 4;
  const int prow0 = w * PB + h * RB_PL;   // first operator row of this thread
  const int nrow = max(0, min(RB_PL, min(PB - h * RB_PL, S - prow0)));
  // GEMV 1
  double y0[RB_AL], y1[RB_AL];
#pragma unroll
  for (int c = 0; c < RB_AL; ++c) { y0[c] = 0.0; y1[c] = 0.0; }
#pragma unroll
  for (int i = 0; i < RB_PL; ++i) {
    const double k0 = i < nrow ? kf(0, prow0 + i) : 0.0;
    const double k1 = (i < nrow && nt > 1) ? kf(1, prow0 + i) : 0.0;
#pragma unroll
    for (int c = 0; c < RB_AL; ++c) { y0[c] = fma(op[i][c], k0, y0[c]); y1[c] = fma(op[i][c], k1, y1[c]); }
  }
  // reduce-scatter over the p halves: h = 0 keeps column 0, h = 1 column 1
  // warp partials at [w][c][j][h] (h = the column kept): the 32 lanes store
  // consecutive doubles (conflict free)
  constexpr int WP = 2 * 16 * RB_AL;   // doubles per warp
#pragma unroll
  for (int c = 0; c < RB_AL; ++c) {
    const double keep = h ? y1[c] : y0[c], send = h ? y0[c] : y1[c];
    ypart[w * WP + c * 32 + j * 2 + h] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
  __syncthreads();
  if (tid < WP) {   // Y = sum over the 16 warps (fixed order) -> yb2 [t][c][j]
    double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
#pragma unroll
    for (int q = 0; q < kWarps; q += 4) {
      v0 += ypart[(q + 0) * WP + tid];
      v1 += ypart[(q + 1) * WP + tid];
      v2 += ypart[(q + 2) * WP + tid];
      v3 += ypart[(q + 3) * WP + tid];
    }
    const int c = tid >> 5, jj = (tid & 31) >> 1, t = tid & 1;
    yb2[t * (16 * RB_AL) + c * 16 + jj] = t < nt ? (v0 + v1) + (v2 + v3) : 0.0;
  }
  __syncthreads();
  // GEMV 2 (Y reads: 16 consecutive doubles per half-warp, conflict free)
  double ya[RB_AL], yc[RB_AL];
#pragma unroll
  for (int c = 0; c < RB_AL; ++c) { ya[c] = yb2[c * 16 + j]; yc[c] = yb2[16 * RB_AL + c * 16 + j]; }
  double v[16];
#pragma unroll
  for (int i = 0; i < RB_PL; ++i) {
    double o0 = 0.0, o1 = 0.0;
#pragma unroll
    for (int c = 0; c < RB_AL; ++c) { o0 = fma(op[i][c], ya[c], o0); o1 = fma(op[i][c], yc[c], o1); }
    v[i] = o0; v[8 + i] = o1;
  }
  v[7] = 0.0; v[15] = 0.0;
  // reduce-scatter over the 16 a lanes: lane j keeps index (j>>3)*8 + (j&7)
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const bool up = j & 8;
    v[k] = (up ? v[8 + k] : v[k]) + __shfl_xor_sync(0xffffffffu, up ? v[k] : v[8 + k], 8);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const bool up = j & 4;
    v[k] = (up ? v[4 + k] : v[k]) + __shfl_xor_sync(0xffffffffu, up ? v[k] : v[4 + k], 4);
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const bool up = j & 2;
    v[k] = (up ? v[2 + k] : v[k]) + __shfl_xor_sync(0xffffffffu, up ? v[k] : v[2 + k], 2);
  }
  {
    const bool up = j & 1;
    v[0] = (up ? v[1] : v[0]) + __shfl_xor_sync(0xffffffffu, up ? v[0] : v[1], 1);
  }
  const int t = j >> 3, i = j & 7;
  if (i < nrow && t < nt) epi(prow0 + i, t, v[0]);
}

// GEMM-2 epilogue of the patch/two-phase kernels: O back into kt.
struct StoreO {
  double* kt; int ldk;
  __device__ __forceinline__ void before_store() const {}
  __device__ __forceinline__ void prefetch(int, int) const {}
  __device__ __forceinline__ void store(int, int mt, int nn, double c0, double c1) const {
    const int lane = threadIdx.x & 31, g = lane >> 2, tig = lane & 3;
    kt[(nn * 8 + 2 * tig) * ldk + mt * 8 + g] = c0;
    kt[(nn * 8 + 2 * tig + 1) * ldk + mt * 8 + g] = c1;
  }
};

// ---------------------------------------------------------------------------
// Fast column chunk: TC columns of one class. The caller fills the per-column
// metadata (smem) -- m_pos[t] = column base offset c*s_pad, m_s[t] = offset
// of support slot 0 in the s source, m_q[t] = q offset, m_x[t] = x_c -- for
// t < nt, and the s source is `s_src` (shared patch or global s_row); with
// `irow` non-null, the global generic layout maps support slots to rows.
// shared: kt [TC][ldk] (K, then O), yb [n08][ldy], yp [split][n08][TC].
// ---------------------------------------------------------------------------
// K-split pairs (P.cta_pair, patch mode): this CTA's half of the support
// rows [p_lo, p_hi) in GEMM 1 (partial Y), GEMM 2 and the epilogue; the two
// partial Y are swapped through global memory (double-buffered, a release /
// acquire counter per CTA) and summed in the same order in both CTAs.
struct KSplit {
  int partner = -1, half = 0;
  int* cnt = nullptr;   // this CTA's publications so far in the launch
};

__device__ __forceinline__ void ksplit_exchange_y(const DevProblem& P, const KSplit& ks, double* yb, int ldy,
                                                  int n08, int TCc) {
  const int tid = threadIdx.x;
  const int slot = *ks.cnt & 1;
  const size_t per = static_cast<size_t>(P.n08_max) * TCc;
  double* mine = P.ypair + (static_cast<size_t>(VBID) * 2 + slot) * per;
  const double* theirs = P.ypair + (static_cast<size_t>(ks.partner) * 2 + slot) * per;
  for (int idx = tid; idx < n08 * TCc; idx += kThreads) {
    const int a = idx / TCc, t = idx - a * TCc;
    mine[idx] = yb[a * ldy + t];
  }
  __syncthreads();
  *ks.cnt += 1;
  if (tid == 0) {
    __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" :: "l"(P.pair_flag + VBID) : "memory");
    while (static_cast<int>(ld_acquire_u32(P.pair_flag + ks.partner) - static_cast<unsigned>(*ks.cnt)) < 0) {}
  }
  __syncthreads();
  for (int idx = tid; idx < n08 * TCc; idx += kThreads) {
    const int a = idx / TCc, t = idx - a * TCc;
    const double o = __ldcg(theirs + idx), m = yb[a * ldy + t];
    yb[a * ldy + t] = ks.half == 0 ? m + o : o + m;   // Y = Y(half 0) + Y(half 1) in both CTAs
  }
  __syncthreads();
}

// L1LD (the partial-cache patch kernels, kVarPcache): ψ, λ of the chunk with
// plain loads, prefetched into L1 under the Φ stage (chunk_prefetch_l1):
// the epilogue's second read of them hits L1 (d=6, T=30: 190.7 -> 185.5
// us/iter; in the other patch kernels it measured up to 2% slower).
template <int TC, bool S_GLOBAL, bool OPS, bool KS = false, bool L1LD = false>
__device__ void fast_chunk(const DevProblem& P, int k, int nt, const double* psi, const double* lam,
                           double* psi_n, double* lam_n, const double* s_src, const int* irow_tab,
                           double* smem, double& pri_m, double& dual_m, const double* st,
                           const KSplit& ks = KSplit()) {
  constexpr int NTN = TC / 8;
  constexpr int WPC = kWarps / TC;   // warps per column in the element loops
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tig = lane & 3;
  double* kt = smem + P.off_k;
  double* yb = smem + P.off_y;
  double* yp = smem + P.off_yp;
  const long long* m_pos = reinterpret_cast<const long long*>(smem + P.off_meta);
  const long long* m_s = m_pos + TC;
  const long long* m_q = m_pos + 2 * TC;
  const double* m_x = smem + P.off_meta + 3 * TC;
  const int ldk = P.ldk, ldy = P.ldy;
  const ClassDims cd = class_dims(P, smem, k);
  const int S = cd.s, S8 = (S + 7) & ~7;
  const int n0 = cd.n0, n08 = (n0 + 7) & ~7;
  const int ldn = cd.ldn;
  // the class operator: staged at smem offset 0 (LDS) or read from global
  const double* nop = OPS ? smem : P.null_pool + cd.off;
  PT_DECL
  PT_START
  const int t_el = warp / WPC;                  // this warp's column in element loops
  constexpr int PSTEP = 32 * WPC;
  // support rows of this CTA: all, or its half of a K-split pair (multiple of 8)
  // (a separate instantiation, KS: the unpaired path keeps its registers)
  const int p_lo = !KS || ks.half == 0 ? 0 : ((S8 >> 1) + 7) & ~7;
  const int p_hi = !KS || ks.half == 1 ? S8 : ((S8 >> 1) + 7) & ~7;
  const int p_el0 = p_lo + (warp % WPC) * 32 + lane;   // first support slot
  // prologue: K[t][p] = φ + λ (admm.py:183), zero padded to TC x S8
  {
    const int t = t_el;
    const bool col_ok = t < nt;
    const long long pos0 = col_ok ? m_pos[t] : 0, s0 = col_ok ? m_s[t] : 0;
    const double xc = col_ok ? m_x[t] : 0.0;
    for (int pb = p_el0; pb < p_hi; pb += 4 * PSTEP) {
      double ps[4], lm[4], sr[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int p = pb + u * PSTEP;
        ps[u] = lm[u] = sr[u] = 0.0;
        if (col_ok && p < S) {
          if (st) {
            ps[u] = st[(2 * t) * ldk + p];
            lm[u] = st[(2 * t + 1) * ldk + p];
          } else if (L1LD) {   // partial-cache patch kernels: L1 hits after chunk_prefetch_l1
            ps[u] = psi[pos0 + p];
            lm[u] = lam[pos0 + p];
          } else {
            ps[u] = ld_cg(psi + pos0 + p);
            lm[u] = ld_cg(lam + pos0 + p);
          }
          sr[u] = !S_GLOBAL ? s_src[s0 + p] : ld_cg(s_src + (irow_tab ? irow_tab[s0 + p] : s0 + p));
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int p = pb + u * PSTEP;
        if (p < p_hi) {
          double kv = 0.0;
          if (col_ok && p < S) kv = __dadd_rn(make_phi<false>(__dsub_rn(ps[u], lm[u]), sr[u], xc), lm[u]);
          kt[t * ldk + p] = kv;
        }
      }
    }
  }
  __syncthreads();
  PT_LAP(P, 1)
  if (TC == 8 && nt <= 2 && P.small_gemv && n08 * 10 <= kThreads && !KS)
    gemv1_small<TC>(S, n08, ldn, nop, kt, ldk, yp, yb, ldy, nt);
  else
    gemm1<TC, NoHook, kWarps, CtaBar, 1>(P, p_hi - p_lo, n08, ldn, nop + static_cast<size_t>(p_lo) * ldn,
                                         kt + p_lo, ldk, yb, ldy, yp);
  if constexpr (KS) ksplit_exchange_y(P, ks, yb, ldy, n08, TC);
  PT_LAP(P, 2)
  // GEMM 2: O[t][p] = sum_a N[p][a] Y[a][t]  (M = S, N = TC, K = n0) -> kt
  StoreO epi{kt + p_lo, ldk};
  gemm2<TC>(p_hi - p_lo, n08, ldn, nop + static_cast<size_t>(p_lo) * ldn, yb, ldy, epi);
  __syncthreads();
  PT_LAP(P, 3)
  // epilogue: ψ' = q + O, λ' = λ + (φ - ψ'), residuals (admm.py:186, 207, 216-217)
  {
    const int t = t_el;
    if (t < nt) {
      const long long pos0 = m_pos[t], s0 = m_s[t], q0 = m_q[t];
      const double xc = m_x[t];
      const int p_end = min(S, p_hi);
      for (int pb = p_el0; pb < p_end; pb += 4 * PSTEP) {
        double ps[4], lm[4], sr[4], qv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int p = pb + u * PSTEP;
          ps[u] = lm[u] = sr[u] = qv[u] = 0.0;
          if (p < p_end) {
            if (st) {
              ps[u] = st[(2 * t) * ldk + p];
              lm[u] = st[(2 * t + 1) * ldk + p];
            } else if (L1LD) {
              ps[u] = psi[pos0 + p];
              lm[u] = lam[pos0 + p];
            } else {
              ps[u] = ld_cg(psi + pos0 + p);
              lm[u] = ld_cg(lam + pos0 + p);
            }
            sr[u] = !S_GLOBAL ? s_src[s0 + p] : ld_cg(s_src + (irow_tab ? irow_tab[s0 + p] : s0 + p));
            qv[u] = P.q_pool[q0 + p];
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int p = pb + u * PSTEP;
          if (p < p_end) {
            const double phi = make_phi<false>(__dsub_rn(ps[u], lm[u]), sr[u], xc);
            const double pn = qv[u] + kt[t * ldk + p];
            const double d = __dsub_rn(phi, pn);
            if (DCHK_CELL(P, pos0 + p, 1)) {
              psi_n[pos0 + p] = pn;
              lam_n[pos0 + p] = __dadd_rn(lm[u], d);
            }
            pri_m = rmax(pri_m, fabs(d));
            dual_m = rmax(dual_m, fabs(__dsub_rn(pn, ps[u])));
          }
        }
      }
    }
  }
  __syncthreads();
  PT_LAP(P, 4)
}

// Make class k's null-space operator resident at smem offset 0 if it fits
// (cooperative copy, once per class change -- with the class-aware CTA
// assignment, once per launch). Returns whether it is in shared memory.
__device__ __forceinline__ bool stage_operator(const DevProblem& P, int k, double* smem, int& cur) {
  const ClassDims cd = class_dims(P, smem, k);
  const long long n = static_cast<long long>((cd.s + 7) & ~7) * cd.ldn;
  if (n > P.opr_cap) return false;
  if (k != cur) {
    __syncthreads();
    const double2* src = reinterpret_cast<const double2*>(P.null_pool + cd.off);
    double2* dst = reinterpret_cast<double2*>(smem);
    for (long long q = threadIdx.x; q < n / 2; q += kThreads) dst[q] = __ldg(src + q);
    __syncthreads();
    cur = k;
  }
  return true;
}

// stage_operator with the class sizes already known (no global loads)
__device__ __forceinline__ void stage_operator_sized(const DevProblem& P, int k, int S8, int ldn, double* smem,
                                                     int& cur) {
  if (k == cur) return;
  __syncthreads();
  const long long n = static_cast<long long>(S8) * ldn;
  const double2* src = reinterpret_cast<const double2*>(P.null_pool + P.class_null_off[k]);
  double2* dst = reinterpret_cast<double2*>(smem);
  for (long long q = threadIdx.x; q < n / 2; q += kThreads) dst[q] = __ldg(src + q);
  __syncthreads();
  cur = k;
}

template <int TC, bool S_GLOBAL, bool L1LD = false>
__device__ __forceinline__ void run_chunk(const DevProblem& P, int k, int nt, const double* psi,
                                          const double* lam, double* psi_n, double* lam_n,
                                          const double* s_src, const int* irow_tab, double* smem,
                                          int& cur, double& pri_m, double& dual_m,
                                          const double* st = nullptr, const KSplit& ks = KSplit()) {
  const bool ops = stage_operator(P, k, smem, cur);
  if (!S_GLOBAL && ks.partner >= 0) {   // K-split pair (patch mode; bases that live in L2)
    if (ops) fast_chunk<TC, S_GLOBAL, true, true, L1LD>(P, k, nt, psi, lam, psi_n, lam_n, s_src, irow_tab, smem, pri_m, dual_m, st, ks);
    else fast_chunk<TC, S_GLOBAL, false, true, L1LD>(P, k, nt, psi, lam, psi_n, lam_n, s_src, irow_tab, smem, pri_m, dual_m, st, ks);
  } else if (ops) {
    fast_chunk<TC, S_GLOBAL, true, false, L1LD>(P, k, nt, psi, lam, psi_n, lam_n, s_src, irow_tab, smem, pri_m, dual_m, st);
  } else {
    fast_chunk<TC, S_GLOBAL, false, false, L1LD>(P, k, nt, psi, lam, psi_n, lam_n, s_src, irow_tab, smem, pri_m, dual_m, st);
  }
}

// Patch-kernel chunk of <= 2 columns on the register-blocked GEMV pair
// (P.rb_gemv): K = φ + λ is formed inside GEMV 1 from the staged ψ, λ and the
// patch's Φ scales (no prologue pass), and every thread runs the epilogue of
// the one (row, column) element GEMV 2 leaves it, with its operands fetched
// before the GEMVs. Same formulas as fast_chunk (admm.py:183-186, 207,
// 216-217); the operator is staged thread-major once per class.
constexpr int kRbTag = 1 << 24;   // `cur` = k + AL * kRbTag: a thread-major staged operator
template <int TC, int RB_AL>
__device__ void rb_chunk_al(const DevProblem& P, int k, int S, int nt, double* psi_n, double* lam_n,
                            const double* s_src, double* smem, int& cur, double& pri_m, double& dual_m,
                            const double* st) {
  if (cur != k + RB_AL * kRbTag) {
    __syncthreads();
    stage_operator_rb<RB_AL>(P, k, smem);
    __syncthreads();
    cur = k + RB_AL * kRbTag;
  }
  const long long* m_pos = reinterpret_cast<const long long*>(smem + P.off_meta);
  const long long* m_s = m_pos + TC;
  const long long* m_q = m_pos + 2 * TC;
  const double* m_x = smem + P.off_meta + 3 * TC;
  const int ldk = P.ldk;
  const int l = threadIdx.x & 31, w = threadIdx.x >> 5, h = l >> 4, j = l & 15;
  const int PB = (((S + 7) & ~7) + 15) >> 4;
  const int prow0 = w * PB + h * RB_PL;
  const int nrow = max(0, min(RB_PL, min(PB - h * RB_PL, S - prow0)));
  PT_DECL
  PT_START
  double op[RB_PL][RB_AL];
  load_operator_rb<RB_AL>(smem, op);
  // this thread's epilogue element (row prow0 + (j & 7), column j >> 3)
  const int et = j >> 3, ep = prow0 + (j & 7);
  const bool eok = (j & 7) < nrow && et < nt;
  double e_ps = 0.0, e_lm = 0.0, e_sr = 0.0, e_q = 0.0, e_x = 0.0;
  long long e_pos = 0;
  if (eok) {
    e_pos = m_pos[et]; e_x = m_x[et];
    e_ps = st[(2 * et) * ldk + ep]; e_lm = st[(2 * et + 1) * ldk + ep];
    e_sr = s_src[m_s[et] + ep];
    e_q = P.q_pool[m_q[et] + ep];
  }
  const long long s00 = m_s[0], s01 = m_s[1];
  const double x0 = m_x[0], x1 = m_x[1];
  auto kf = [&](int t, int p) {   // K = φ + λ, one rounding more than φ (the fast_chunk prologue)
    const double ps = st[(2 * t) * ldk + p], lm = st[(2 * t + 1) * ldk + p];
    const double sr = s_src[(t ? s01 : s00) + p];
    return __dadd_rn(make_phi<false>(__dsub_rn(ps, lm), sr, t ? x1 : x0), lm);
  };
  auto epi = [&](int, int, double o) {
    const double phi = make_phi<false>(__dsub_rn(e_ps, e_lm), e_sr, e_x);
    const double pn = e_q + o;
    const double d = __dsub_rn(phi, pn);
    if (DCHK_CELL(P, e_pos + ep, 2)) {
      psi_n[e_pos + ep] = pn;
      lam_n[e_pos + ep] = __dadd_rn(e_lm, d);
    }
    pri_m = rmax(pri_m, fabs(d));
    dual_m = rmax(dual_m, fabs(__dsub_rn(pn, e_ps)));
  };
  PT_LAP(P, 1)
  gemv_pair_rb<RB_AL>(S, op, kf, smem + P.off_yp, smem + P.off_y, nt, epi);
  PT_LAP(P, 2)
}

// One blocking (RB_AL = 4, n0 <= 64) for every class: a second, narrower
// instantiation for the d=3 interior class (n0 = 47) saves its idle FMAs but
// doubles the hot loop's code, and measured 10.6 vs 8.4 us/iteration on C2.
// S: the class's support length (the caller has it: no global table load
// after the iteration barrier, whose acquire invalidates L1).
template <int TC>
__device__ __forceinline__ void rb_chunk(const DevProblem& P, int k, int S, int nt, double* psi_n, double* lam_n,
                                         const double* s_src, double* smem, int& cur, double& pri_m,
                                         double& dual_m, const double* st) {
  rb_chunk_al<TC, RB_AL_MAX>(P, k, S, nt, psi_n, lam_n, s_src, smem, cur, pri_m, dual_m, st);
}

// Column stage of the two-phase fast kernel (class-sorted tiles, generic graphs).
template <int TC>
__device__ void column_stage_tiles(const DevProblem& P, int b, const double* x, int it, double* smem,
                                   int& cur) {
  long long* m_pos = reinterpret_cast<long long*>(smem + P.off_meta);
  double* m_x = smem + P.off_meta + 3 * TC;
  double pri_m = 0.0, dual_m = 0.0;
  for (int tile = VBID; tile < P.n_tiles; tile += VGRID) {
    const int k = P.tile_class[tile], first = P.tile_first[tile], nt = P.tile_count[tile];
    if (threadIdx.x < TC) {
      const int t = threadIdx.x;
      long long pos = 0, s0 = 0, q0 = 0;
      double xc = 0.0;
      if (t < nt) {
        const int c = P.tile_colv[first + t];
        pos = static_cast<long long>(c) * P.s_pad;
        s0 = P.contiguous ? P.col_rowbase[c] : static_cast<long long>(P.col_owner[c]) * P.s_pad;
        q0 = static_cast<long long>(P.col_vec[c]) * P.s_pad;
        xc = ld_cg(x + c);
      }
      m_pos[t] = pos; m_pos[TC + t] = s0; m_pos[2 * TC + t] = q0; m_x[t] = xc;
    }
    __syncthreads();
    run_chunk<TC, true>(P, k, nt, P.psi[b], P.lam[b], P.psi[b ^ 1], P.lam[b ^ 1], P.s_row,
                        P.contiguous ? nullptr : P.col_irow, smem, cur, pri_m, dual_m);
  }
  publish_residuals(P, it, pri_m, dual_m, smem + P.off_red);
}

// Per-step Φ metadata of a CTA's single unit, cached in shared memory (the
// support descriptors, x on the support, row costs/bounds and ||a||^2 are
// constant for a whole MPC step): each iteration's Φ then needs one L2 round
// trip (the ψ,λ reads) instead of three.
// layout at off_phimeta: base [np*d_pad] (int64), xk [np*d_pad], ada [np],
//                        inv_den/lo/hi [3*prows], len [np] (int32 in a double slot),
//                        then at off_ublk: ublk [16 ints], rinfo [np] (int2: local row offset, rows)
// inv_den = 1/(ρ + 2w·||a||²) and 1/||a||² (in the ada slot) turn the two
// per-row IEEE divisions of the fast path into multiplications. The unit
// block holds the unit's ranges and its first chunk; a unit of one chunk
// also gets that chunk's column metadata (off_meta) once per step, so an
// iteration's control path touches no global memory.
// ublk: has_unit, own_lo, own_hi, plo, phi, prows, prow0 (2 ints), ch_a, ch_b,
//       k, c0, nt, S of the first chunk, own-row offset in the patch, own rows
// `full` (first MPC step of a launch): also the step-invariant part (support
// positions and lengths, row bounds, unit block, row info, the single
// chunk's column positions); later steps refresh only what depends on x
// (x of the supports and of the chunk's columns, 1/||a||², 1/(ρ + 2w·||a||²)).
// The x-dependent scales of patch subsystem q's rows from its ||a||^2 (one
// warp): 1/||a||^2 and 1/(ρ + 2w·||a||^2) per row (shared by cache_phi_meta
// and fused_transition, so both produce the same bits).
__device__ __forceinline__ void phi_cache_scales(const DevProblem& P, double a, int2 ri, const double* w,
                                                 double* ada_q, double* rw) {
  const int lane = threadIdx.x & 31;
  if (lane == 0) *ada_q = a > 0.0 ? 1.0 / a : 0.0;
  for (int l = lane; l < ri.y; l += 32) rw[ri.x + l] = 1.0 / (P.rho + 2.0 * w[ri.x + l] * a);
}

template <int TC>
__device__ void cache_phi_meta(const DevProblem& P, const double* x, double* smem, bool full) {
  const int un0 = P.cta_unit_ptr[VBID];
  if (un0 == P.cta_unit_ptr[VBID + 1]) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int plo = P.unit_patch_lo[un0], phi_ = P.unit_patch_hi[un0];
  const int np = phi_ - plo;
  const long long prow0 = P.row_start[plo];
  const int prows = static_cast<int>(P.row_start[phi_] - prow0);
  double* base = smem + P.off_phimeta;
  long long* bk = reinterpret_cast<long long*>(base);
  double* xk = base + static_cast<size_t>(np) * P.d_pad;
  double* ada = xk + static_cast<size_t>(np) * P.d_pad;
  double* rw = ada + np;
  const bool part = P.cache_phi == 2;   // partial cache: no per-row scales and bounds, raw ||a||^2
  int* len = reinterpret_cast<int*>(rw + (part ? 0 : 3 * prows));
  int* ublk = reinterpret_cast<int*>(smem + P.off_ublk);
  int2* rinfo = reinterpret_cast<int2*>(smem + P.off_ublk + 8);
  const int ch_a = P.unit_chunk_ptr[un0], ch_b = P.unit_chunk_ptr[un0 + 1];
  const bool one_chunk = ch_b - ch_a == 1;
  long long* m_pos = reinterpret_cast<long long*>(smem + P.off_meta);
  double* m_x = smem + P.off_meta + 3 * TC;
  if (full) {
    for (int q = threadIdx.x; q < np * P.d_pad; q += kThreads) {
      const int i = plo + q / P.d_pad, k = q % P.d_pad;
      if (k < P.supp_len[i]) {
        const size_t e = static_cast<size_t>(i) * P.d_pad + k;
        bk[q] = static_cast<long long>(P.supp_col[e]) * P.s_pad + P.supp_off[e];
      }
    }
    for (int q = threadIdx.x; q < np; q += kThreads) {
      len[q] = P.supp_len[plo + q];
      rinfo[q] = make_int2(static_cast<int>(P.row_start[plo + q] - prow0),
                           static_cast<int>(P.row_start[plo + q + 1] - P.row_start[plo + q]));
    }
    for (int q = threadIdx.x; q < (part ? 0 : prows); q += kThreads) {
      rw[prows + q] = P.row_lo[prow0 + q]; rw[2 * prows + q] = P.row_hi[prow0 + q];
    }
    const int own_lo = P.unit_sub_lo[un0], own_hi = P.unit_sub_hi[un0];
    if (threadIdx.x == 0) {
      ublk[0] = 1; ublk[1] = own_lo; ublk[2] = own_hi; ublk[3] = plo; ublk[4] = phi_; ublk[5] = prows;
      ublk[6] = static_cast<int>(prow0 & 0xffffffffLL); ublk[7] = static_cast<int>(prow0 >> 32);
      ublk[8] = ch_a; ublk[9] = ch_b;
      const int k = P.chunk_class[ch_a];
      ublk[10] = k; ublk[11] = P.chunk_col0[ch_a]; ublk[12] = P.chunk_n[ch_a]; ublk[13] = P.class_s[k];
      ublk[14] = static_cast<int>(P.row_start[own_lo] - prow0);
      ublk[15] = static_cast<int>(P.row_start[own_hi] - P.row_start[own_lo]);
    }
    if (one_chunk && threadIdx.x < TC) {   // the single chunk's column metadata
      const int t = threadIdx.x, c0 = P.chunk_col0[ch_a], nt = P.chunk_n[ch_a];
      long long pos = 0, s0 = 0, q0 = 0;
      if (t < nt) {
        const int c = c0 + t;
        pos = static_cast<long long>(c) * P.s_pad;
        s0 = P.col_rowbase[c] - prow0;
        q0 = static_cast<long long>(P.col_vec[c]) * P.s_pad;
      }
      m_pos[t] = pos; m_pos[TC + t] = s0; m_pos[2 * TC + t] = q0;
    }
    __syncthreads();
  }
  // x-dependent part (every MPC step); a warp per patch subsystem
  for (int q = warp; q < np; q += kWarps) {
    const int i = plo + q;
    const int D = len[q];
    for (int k = lane; k < D; k += 32) xk[q * P.d_pad + k] = ld_cg(x + P.supp_col[static_cast<size_t>(i) * P.d_pad + k]);
    if (part) { if (lane == 0) ada[q] = ld_cg(P.ada + i); }
    else phi_cache_scales(P, ld_cg(P.ada + i), rinfo[q], P.row_w + prow0, ada + q, rw);
  }
  if (one_chunk && threadIdx.x < TC) {
    const int t = threadIdx.x;
    m_x[t] = t < P.chunk_n[ch_a] ? ld_cg(x + P.chunk_col0[ch_a] + t) : 0.0;
  }
  __syncthreads();
}

// Φ scale of the rows of patch subsystem q from the cached metadata (fast path).
// UNCOND: the support loads unconditional (slots past the support repeat
// the last one), so all 32 are in flight before the first use. Measured on
// the register-blocked GEMV kernel (C2 closed loops): +3.2%; on the DMMA
// patch kernels (N=1000 C4 cells) -1% to +1%, so those keep the guarded loads.
template <bool UNCOND, class Out>
__device__ __forceinline__ void phi_rows_cached(const DevProblem& P, int q, int np, int prows,
                                                int r_off, int nr, const double* psi, const double* lam,
                                                const double* smem, const Out& out) {
  const int lane = threadIdx.x & 31;
  const double* base = smem + P.off_phimeta;
  const long long* bk = reinterpret_cast<const long long*>(base) + static_cast<size_t>(q) * P.d_pad;
  const double* xk = base + static_cast<size_t>(np) * P.d_pad + static_cast<size_t>(q) * P.d_pad;
  const double* ada_p = base + 2 * static_cast<size_t>(np) * P.d_pad;
  const double* rw = ada_p + np;
  const int D = reinterpret_cast<const int*>(rw + 3 * prows)[q];
  const double inv_ada = ada_p[q];
  const double rho = P.rho;
  for (int l0 = 0; l0 < nr; l0 += 32) {
    const int l = l0 + lane;
    if (l >= nr) break;
    double acc = 0.0;
    for (int k0 = 0; k0 < D; k0 += 16) {
      double pv[16], lv[16];
#ifndef DLMPC_CHECKED
      if constexpr (UNCOND) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const long long b = bk[min(k0 + u, D - 1)] + l;
          pv[u] = ld_cg(psi + b);
          lv[u] = ld_cg(lam + b);
        }
      } else
#endif
      {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          pv[u] = lv[u] = 0.0;
          if (k0 + u < D) {
            const long long b = bk[k0 + u] + l;
            if (DCHK(P, b >= 0 && b < static_cast<long long>(P.n_cols) * P.s_pad, 10, b)) {
              pv[u] = ld_cg(psi + b);
              lv[u] = ld_cg(lam + b);
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 16; ++u)
        if (k0 + u < D) acc = fma(__dsub_rn(pv[u], lv[u]), xk[k0 + u], acc);
    }
    const int rr = r_off + l;
    const double y = fmin(fmax(rho * acc * rw[rr], rw[prows + rr]), rw[2 * prows + rr]);
    out(l, (y - acc) * inv_ada);
  }
}

// Φ scale of the rows of patch subsystem q from the partial cache
// (P.cache_phi == 2: the support descriptors, x on the support and the raw
// ||a||^2 in shared memory; a plan whose per-row scales and bounds do not fit
// shared memory). The row weight and bounds come from global memory with the
// row's ψ, λ (one round trip); the two reciprocals are formed as
// phi_cache_scales forms them.
template <class Out>
__device__ __forceinline__ void phi_rows_pcached(const DevProblem& P, int q, int np, long long prow0, int r_off,
                                                 int nr, const double* psi, const double* lam, const double* smem,
                                                 const Out& out) {
  const int lane = threadIdx.x & 31;
  const double* base = smem + P.off_phimeta;
  const long long* bk = reinterpret_cast<const long long*>(base) + static_cast<size_t>(q) * P.d_pad;
  const double* xk = base + static_cast<size_t>(np) * P.d_pad + static_cast<size_t>(q) * P.d_pad;
  const double* ada_p = base + 2 * static_cast<size_t>(np) * P.d_pad;
  const int D = reinterpret_cast<const int*>(ada_p + np)[q];
  const double a = ada_p[q];
  const double inv_ada = a > 0.0 ? 1.0 / a : 0.0;
  const double rho = P.rho;
  for (int l0 = 0; l0 < nr; l0 += 32) {
    const int l = l0 + lane;
    if (l >= nr) break;
    const long long gr = prow0 + r_off + l;
    const double w = P.row_w[gr], lo = P.row_lo[gr], hi = P.row_hi[gr];
    double acc = 0.0;
    for (int k0 = 0; k0 < D; k0 += 16) {
      double pv[16], lv[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        pv[u] = lv[u] = 0.0;
        if (k0 + u < D) {
          const long long b = bk[k0 + u] + l;
          if (DCHK(P, b >= 0 && b < static_cast<long long>(P.n_cols) * P.s_pad, 10, b)) {
            pv[u] = ld_cg(psi + b);
            lv[u] = ld_cg(lam + b);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 16; ++u)
        if (k0 + u < D) acc = fma(__dsub_rn(pv[u], lv[u]), xk[k0 + u], acc);
    }
    const double inv_den = 1.0 / (P.rho + 2.0 * w * a);
    const double y = fmin(fmax(rho * acc * inv_den, lo), hi);
    out(l, (y - acc) * inv_ada);
  }
}

// One ADMM iteration of the patch kernel for this CTA's units.
// The stop test of iteration it-1 (global residual maxima, published before
// the grid barrier) is overlapped with iteration it's first Φ stage: the two
// words are fetched first, the unit's Φ goes to shared memory only, then the
// test; on convergence the CTA returns `true` with the state of iteration
// it-1 untouched (ψ, λ and the global s_row of its own rows). Every CTA reads
// the same words, so the decision is grid-uniform.
__device__ __forceinline__ bool patch_stop_test(const DevProblem& P, const RunArgs& R, int it,
                                                unsigned long long rp, unsigned long long rd) {
  const double pri = __longlong_as_double(static_cast<long long>(rp));
  const double dual = P.rho * __longlong_as_double(static_cast<long long>(rd));
  if (VBID == 0 && threadIdx.x == 0) { R.hist[2 * (it - 1)] = pri; R.hist[2 * (it - 1) + 1] = dual; }
  return R.stop_on_conv && pri <= R.eps_pri && dual <= R.eps_dual;
}

// roff: this MPC step's residual region (word offset in P.resid). pre_target
// (fused step transitions, iteration 0 only; 0 = none): the split barrier of
// the previous step's transition -- every CTA has finished reading the final
// iterate (buffer b ^ 1, s_row) once the counter reaches it; waited for by
// the last warp under the Φ stage, before the first store into b ^ 1 or s_row.
// FUSE (kVarFuse kernels only; measured: the extra state compiled into the
// plain kernel made ptxas interleave the Φ loads with the dot product, +47%
// per C2 iteration, so the plain path keeps its original form):
template <int TC, bool RB, bool PAIRS, bool FUSE, bool PCACHE>
__device__ bool patch_iteration(const DevProblem& P, int b, const double* x, int it, double* smem,
                                int& cur, const RunArgs& R, unsigned bar_target, int& pair_cnt, int roff,
                                unsigned pre_target) {
  double* s_patch = smem + P.off_patch;
  long long* m_pos = reinterpret_cast<long long*>(smem + P.off_meta);
  double* m_x = smem + P.off_meta + 3 * TC;
  const int warp = threadIdx.x >> 5;
  const double* psi = P.psi[b];
  const double* lam = P.lam[b];
  double pri_m = 0.0, dual_m = 0.0;
  bool tested = it == 0;
  // FUSE, iteration 0: the own rows' s reach s_row after the Φ barrier (and the split-barrier wait)
  const bool defer0 = FUSE && pre_target != 0u;
  // the two residual words: one load per CTA (thread 0), broadcast through
  // shared memory at the Φ barrier -- every thread of every CTA loading the
  // same L2 line is a hot spot of ~5k requests per iteration
  unsigned long long rp = 0, rd = 0;
  unsigned long long* rbc = reinterpret_cast<unsigned long long*>(smem + P.off_red);
  if (!tested && threadIdx.x == 0) {
    rp = __ldcg(P.resid + roff + 2 * (it - 1)); rd = __ldcg(P.resid + roff + 2 * (it - 1) + 1);
  }
  if constexpr (FUSE) {
    if (pre_target != 0u && threadIdx.x == kThreads - 32)
      while (static_cast<int>(ld_acquire_u32(P.gbar) - pre_target) < 0) {}
  }
  PT_DECL
  // the CTA's unit range, staged in shared memory at launch: the iteration
  // barrier's acquire invalidates L1, so a table load here would be an L2
  // round trip at the start of every iteration
  const int* urange = reinterpret_cast<const int*>(smem + P.off_red + 32);
  const int un_a = urange[0], un_b = urange[1];
  if (un_a == un_b && !tested) {
    if (threadIdx.x == 0) { rbc[0] = rp; rbc[1] = rd; }
    __syncthreads();
    rp = rbc[0]; rd = rbc[1];
    __syncthreads();   // every warp has read the slots before the publish reuses them
    if (patch_stop_test(P, R, it, rp, rd)) return true;
  }
  for (int un = un_a; un < un_b; ++un) {
    PT_START
    int own_lo, own_hi, plo, phi_, prows, ch_a, ch_b, k0 = 0, c00 = 0, nt0 = 0, S0 = 0, o_off, o_n;
    long long prow0;
    const int* ublk = nullptr;
    const int2* rinfo = nullptr;
    if (P.cache_phi) {   // one unit per CTA: the control data cached at step start
      ublk = reinterpret_cast<const int*>(smem + P.off_ublk);
      rinfo = reinterpret_cast<const int2*>(smem + P.off_ublk + 8);
      own_lo = ublk[1]; own_hi = ublk[2]; plo = ublk[3]; phi_ = ublk[4]; prows = ublk[5];
      prow0 = static_cast<long long>(static_cast<unsigned>(ublk[6])) | (static_cast<long long>(ublk[7]) << 32);
      ch_a = ublk[8]; ch_b = ublk[9]; k0 = ublk[10]; c00 = ublk[11]; nt0 = ublk[12]; S0 = ublk[13];
      o_off = ublk[14]; o_n = ublk[15];
    } else {
      own_lo = P.unit_sub_lo[un]; own_hi = P.unit_sub_hi[un];
      plo = P.unit_patch_lo[un]; phi_ = P.unit_patch_hi[un];
      prow0 = P.row_start[plo];
      prows = static_cast<int>(P.row_start[phi_] - prow0);
      ch_a = P.unit_chunk_ptr[un]; ch_b = P.unit_chunk_ptr[un + 1];
      if (ch_a < ch_b) {
        k0 = P.chunk_class[ch_a]; c00 = P.chunk_col0[ch_a]; nt0 = P.chunk_n[ch_a]; S0 = P.class_s[k0];
      }
      o_off = static_cast<int>(P.row_start[own_lo] - prow0);
      o_n = static_cast<int>(P.row_start[own_hi] - P.row_start[own_lo]);
    }
    // first chunk's ψ,λ start streaming into shared memory under the Φ stage
    double* stash = smem + P.off_stash;
    const int stash_stride = 2 * P.stash_cols * P.ldk;
    if (P.stash_bufs > 0 && ch_a < ch_b) stash_issue(P, c00, nt0, S0, psi, lam, stash);
    else if (PCACHE && ch_a < ch_b) chunk_prefetch_l1(psi, lam, c00, nt0, P.s_pad);
    PT_LAP(P, 12)   // timing build, patch modes: thread 0's view of the Φ stage in slots 12-15
    // Φ scale of every row the unit's columns touch (own rows + d-hop halo);
    // before the stop test the own rows' s goes to shared memory only
    for (int i = plo + warp; i < phi_; i += kWarps) {
      int r_off, nrow;
      if (rinfo) { const int2 ri = rinfo[i - plo]; r_off = ri.x; nrow = ri.y; }
      else { r_off = static_cast<int>(P.row_start[i] - prow0); nrow = static_cast<int>(P.row_start[i + 1] - P.row_start[i]); }
      double* dst = s_patch + r_off;
      double* gdst = (tested && !defer0 && i >= own_lo && i < own_hi) ? P.s_row + prow0 + r_off : nullptr;
      auto out = [dst, gdst](int l, double s) {
        dst[l] = s;
        if (gdst) gdst[l] = s;
      };
      if constexpr (PCACHE)   // the partial cache (kVarPcache kernels: P.cache_phi == 2)
        phi_rows_pcached(P, i - plo, phi_ - plo, prow0, r_off, nrow, psi, lam, smem, out);
      else if (P.cache_phi)
        phi_rows_cached<RB>(P, i - plo, phi_ - plo, prows, r_off, nrow, psi, lam, smem, out);
      else
        phi_rows_of<false>(P, i, psi, lam, x, out);
    }
    PT_LAP(P, 13)
    if (!tested && threadIdx.x == 0) { rbc[0] = rp; rbc[1] = rd; }
    PT_LAP(P, 14)
    // a unit of one chunk with cached metadata: its staged ψ, λ (issued
    // before Φ) are waited for here, so this barrier also publishes them and
    // the chunk needs no barrier of its own
    const bool one_chunk = P.cache_phi && ch_b - ch_a == 1 && P.stash_bufs > 0;
    if (one_chunk) cp_async_wait<0>();
    PT_LAP(P, 15)
    __syncthreads();
    PT_LAP(P, 0)
    if (!tested) {
      tested = true;
      rp = rbc[0]; rd = rbc[1];
      if (patch_stop_test(P, R, it, rp, rd)) {
        cp_async_wait<0>();
        return true;
      }
      for (int r = threadIdx.x; r < o_n; r += kThreads)
        if (DCHK_ROW(P, prow0 + o_off + r, 5) && DCHK(P, o_off + r < P.patch_cap, 6, o_off + r))
          P.s_row[prow0 + o_off + r] = s_patch[o_off + r];
    } else if (defer0) {
      for (int r = threadIdx.x; r < o_n; r += kThreads)
        if (DCHK_ROW(P, prow0 + o_off + r, 5) && DCHK(P, o_off + r < P.patch_cap, 6, o_off + r))
          P.s_row[prow0 + o_off + r] = s_patch[o_off + r];
    }
    PT_LAP(P, 7)
    // chunk pipeline: ψ,λ of chunk i+1 stream into the other staging buffer
    // (cp.async) while chunk i runs its GEMMs
    const bool meta_cached = P.cache_phi && ch_b - ch_a == 1;
    for (int ch = ch_a; ch < ch_b; ++ch) {
      const int k = ch == ch_a ? k0 : P.chunk_class[ch];
      const int c0 = ch == ch_a ? c00 : P.chunk_col0[ch];
      const int nt = ch == ch_a ? nt0 : P.chunk_n[ch];
      const int sb = P.stash_bufs == 2 ? ((ch - ch_a) & 1) : 0;
      if (!one_chunk) {
        if (P.stash_bufs == 2 && ch + 1 < ch_b) {
          stash_issue(P, P.chunk_col0[ch + 1], P.chunk_n[ch + 1], P.class_s[P.chunk_class[ch + 1]], psi, lam,
                      stash + (sb ^ 1) * stash_stride);
          cp_async_wait<1>();
        } else if (P.stash_bufs > 0) {
          cp_async_wait<0>();
        }
        if (!meta_cached && threadIdx.x < TC) {
          const int t = threadIdx.x;
          long long pos = 0, s0 = 0, q0 = 0;
          double xc = 0.0;
          if (t < nt) {
            const int c = c0 + t;
            pos = static_cast<long long>(c) * P.s_pad;
            s0 = P.col_rowbase[c] - prow0;
            q0 = static_cast<long long>(P.col_vec[c]) * P.s_pad;
            xc = ld_cg(x + c);
          }
          m_pos[t] = pos; m_pos[TC + t] = s0; m_pos[2 * TC + t] = q0; m_x[t] = xc;
        }
        __syncthreads();
      }
      if constexpr (RB)
        rb_chunk<TC>(P, k, ch == ch_a ? S0 : P.class_s[k], nt, P.psi[b ^ 1], P.lam[b ^ 1], s_patch, smem, cur,
                     pri_m, dual_m, stash + sb * stash_stride);
      else
      {
        KSplit ks;
        if constexpr (PAIRS) {   // a separate kernel instantiation (kVarPairs)
          const int pv = P.cta_pair[VBID];
          if (pv >= 0) { ks.partner = pv >> 1; ks.half = pv & 1; ks.cnt = &pair_cnt; }
        }
        run_chunk<TC, false, PCACHE>(P, k, nt, psi, lam, P.psi[b ^ 1], P.lam[b ^ 1], s_patch, nullptr, smem, cur,
                             pri_m, dual_m, P.stash_bufs > 0 ? stash + sb * stash_stride : nullptr, ks);
      }
      if (P.stash_bufs == 1 && ch + 1 < ch_b)   // single buffer: refill after the chunk is done
        stash_issue(P, P.chunk_col0[ch + 1], P.chunk_n[ch + 1], P.class_s[P.chunk_class[ch + 1]], psi, lam, stash);
    }
  }
  PT_START
  publish_barrier(P, P.resid + roff + 2 * it, pri_m, dual_m, smem + P.off_red, bar_target);
  PT_LAP(P, 5)
  return false;
}


// ---------------------------------------------------------------------------
// Stream mode (fast path, wide contiguous units; chosen by the host when
// every d-hop ball meets at most two units). Per chunk of TC same-class
// columns:
//   ψ staged by cp.async one chunk ahead -> K = ψ + s·x in place (= φ + λ,
//   one rounding) -> GEMM 1 -> GEMM 2 whose accumulators go straight into
//   the epilogue (ψ, λ, q prefetched into registers before the GEMM-2 k
//   loop): ψ' = q + O, λ' = λ + (φ - ψ'), residual maxima, ψ', λ' stored,
//   and v' = ψ' - λ' left in the stage buffer -> a banded pass adds
//   Σ_t v'(r,t)·x_t to the unit's per-row partial of the NEXT iteration's Φ
//   dot (ascending column order). At the unit's end each partial goes to the
//   unit's own slot of the row; the next Φ sums a row's slots in unit order
//   (deterministic, no atomics). From the second iteration of a step on, Φ
//   reads a few partials per row instead of the row's whole (ψ, λ)
//   neighbourhood.
// ---------------------------------------------------------------------------
// Stage one array's columns [c0, c0+nt) (s_pad doubles each) into `st`
// ([t][ldk]) with TMA bulk copies on `bar` (thread 0 issues; the caller has
// synchronised the CTA after the buffer's last generic-proxy use).
__device__ __forceinline__ void stash_cols_bulk(const DevProblem& P, int c0, int nt, const double* src,
                                                double* st, unsigned long long* bar, int issuer = 0) {
  if (threadIdx.x == issuer) {
    const unsigned bytes = static_cast<unsigned>(P.s_pad) * 8u;
#ifdef DLMPC_CHECKED
    extern __shared__ double dyn_smem_chk[];
    if (!DCHK(P, c0 >= 0 && c0 + nt <= P.n_cols, 11, c0) ||
        !DCHK(P, (st - dyn_smem_chk) + static_cast<long long>(nt - 1) * P.ldk + P.s_pad <= P.smem_doubles, 12,
              st - dyn_smem_chk))
      nt = 0;
#endif
    fence_proxy_async();
    mbar_expect_tx(bar, bytes * nt);
    if (P.ldk == P.s_pad)   // consecutive columns are one contiguous range
      bulk_load(st, src + static_cast<size_t>(c0) * P.s_pad, bytes * nt, bar);
    else
      for (int t = 0; t < nt; ++t)
        bulk_load(st + t * P.ldk, src + static_cast<size_t>(c0 + t) * P.s_pad, bytes, bar);
  }
}

// λ staging at its own row stride `ldl` (the register epilogue's access
// pattern is conflict free when 2*ldl % 16 is 4 or 12): one bulk copy per
// column, issued in parallel by the lanes of the last warp.
__device__ __forceinline__ void stash_lam_bulk(const DevProblem& P, int c0, int nt, const double* src,
                                               double* st, int ldl, unsigned long long* bar) {
  if ((threadIdx.x >> 5) == kWarps - 1) {
    const int lane = threadIdx.x & 31;
    const unsigned bytes = static_cast<unsigned>(P.s_pad) * 8u;
#ifdef DLMPC_CHECKED
    extern __shared__ double dyn_smem_chk[];
    if (!DCHK(P, c0 >= 0 && c0 + nt <= P.n_cols, 13, c0) ||
        !DCHK(P, (st - dyn_smem_chk) + static_cast<long long>(nt - 1) * ldl + P.s_pad <= P.smem_doubles, 14,
              st - dyn_smem_chk))
      nt = 0;
#endif
    if (lane == 0) mbar_expect_tx(bar, bytes * nt);
    __syncwarp();
    if (lane < nt) {
      fence_proxy_async();
      bulk_load(st + lane * ldl, src + static_cast<size_t>(c0 + lane) * P.s_pad, bytes, bar);
    }
  }
}

// GEMM-2 epilogue of the stream kernel, all operands in shared memory:
// kt holds K = φ + λ, lt holds λ (then receives v' = ψ' - λ').
//   ψ' = q + O;  λ' = λ + (φ - ψ') = K - ψ';  pri: |λ' - λ| = |φ - ψ'|;
//   dual: |ψ' - ψ| with ψ = K - s·x.
template <int TC>
struct StreamEpi {
  static constexpr int NTN = TC / 8;
  double* psi_n; double* lam_n; const double* q_pool;
  const long long* m_pos; const long long* m_s; const long long* m_q; const double* m_x;
  const double* s_patch; const double* kt; double* lt; int ldk, ldl, S, nt;
  double pri_m, dual_m;
  unsigned long long* lam_bar; unsigned lam_phase;   // if set: λ lands before the first store
  bool paired;   // column pairs (2q, 2q+1) share support rows (host flag per chunk)
  double qv[kMG2][NTN][2];
#ifdef DLMPC_CHECKED
  CellChk chk;   // bounds checks of the epilogue stores
#endif
#ifdef DLMPC_PHASE_TIMING
  unsigned long long t_kloop = 0, t_lam = 0;   // profiling build: end of the k loop, λ landed (thread 0)
  __device__ __forceinline__ void before_store() {
    if (threadIdx.x == 0) t_kloop = gtimer();
    if (lam_bar) mbar_wait(lam_bar, lam_phase);
    if (threadIdx.x == 0) t_lam = gtimer();
  }
#else
  __device__ __forceinline__ void before_store() const {
    if (lam_bar) mbar_wait(lam_bar, lam_phase);
  }
#endif
  __device__ __forceinline__ void prefetch(int m, int mt) {
    const int lane = threadIdx.x & 31, g = lane >> 2, tig = lane & 3;
    const int p = mt * 8 + g;
#pragma unroll
    for (int nn = 0; nn < NTN; ++nn)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int t = nn * 8 + 2 * tig + e;
        qv[m][nn][e] = (p < S && t < nt) ? __ldg(q_pool + m_q[t] + p) : 0.0;
      }
  }
  __device__ __forceinline__ void store(int m, int mt, int nn, double c0, double c1) {
    const int lane = threadIdx.x & 31, g = lane >> 2, tig = lane & 3;
    const int p = mt * 8 + g;
    double contrib = 0.0;   // paired chunks: this pair's share of the row's next Φ dot
    double s_pair = 0.0;    // paired chunks: both columns share the support row's Φ scale
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int t = nn * 8 + 2 * tig + e;
      if (p < S && t < nt) {
        const double kv = kt[t * ldk + p], lm = lt[t * ldl + p];
        const double pn = qv[m][nn][e] + (e ? c1 : c0);
        const double ln = __dsub_rn(kv, pn);
        const double sv = (paired && e) ? s_pair : s_patch[m_s[t] + p];
        s_pair = sv;
        const double ps = fma(-sv, m_x[t], kv);
        const long long pos = m_pos[t] + p;
        if (DCHK_CELL(chk, pos, 3)) {
          psi_n[pos] = pn;
          lam_n[pos] = ln;
        }
        pri_m = rmax(pri_m, fabs(__dsub_rn(ln, lm)));
        dual_m = rmax(dual_m, fabs(__dsub_rn(pn, ps)));
        const double v = __dsub_rn(pn, ln);
        if (paired) contrib = e ? fma(v, m_x[t], contrib) : __dmul_rn(v, m_x[t]);
        else lt[t * ldl + p] = v;
      }
    }
    // the pair's two columns share support rows: one value in the even slot
    // (both of its λ reads above were this thread's own)
    if (paired && p < S && nn * 8 + 2 * tig < nt) lt[(nn * 8 + 2 * tig) * ldl + p] = contrib;
  }
};

// λ(ch) must have landed before GEMM 1's closing barrier (mbarrier phase).
struct LamWait {
  unsigned long long* bar; unsigned phase;
  __device__ __forceinline__ void operator()() const { mbar_wait(bar, phase); }
};

// OPS: class operators staged in shared memory (LDS fragments). CTAs holding
// a class whose basis does not fit the region (the host flags them; on chains
// only the few chain-end CTAs, which carry a chunk or two) run the OPS=false
// instantiation and read the basis from L2 -- a separate instantiation, so
// the common path keeps shared-memory fragment loads.
template <int TC, bool OPS>
// keep_tab: an earlier iteration of this launch left this CTA's control
// tables in shared memory (reused when the CTA has a single unit: the tables
// are invariant, and a reload would cost dependent L2 round trips after the
// grid barrier, whose acquire invalidates L1); keep_pada: the same for the
// 1/||a||^2 of the patch subsystems (constant within an MPC step).
__device__ void stream_iteration(const DevProblem& P, int b, const double* x, int it, int itg, double* smem,
                                 int& cur, unsigned& ph, bool keep_tab, bool keep_pada) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* s_patch = smem + P.off_patch;
  double* c_patch = smem + P.off_cpatch;
  double* yb = smem + P.off_y;
  double* yp = smem + P.off_yp;
  long long* meta0 = reinterpret_cast<long long*>(smem + P.off_meta);   // [2][4][TC]
  int* const chtab0 = reinterpret_cast<int*>(smem + P.off_chtab);       // [ch][8 + 2 TC], two copies
  double* const ptab0 = smem + P.off_ptab;                               // [q][6], two copies
  double* const pada0 = smem + P.off_pada;
  int* rowq = reinterpret_cast<int*>(smem + P.off_rowq);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + P.off_bar);   // ψ0, ψ1, λ
  const int ldk = P.ldk;
  double* psi_st = smem + P.off_k;                  // [2][TC][ldk]
  double* lam_st = psi_st + 2 * TC * ldk;           // [TC][ldl]
  const int ldl = P.ldl;
  const double* psi = P.psi[b];
  const double* lam = P.lam[b];
  // itg counts iterations on this state across launches (it + it_base)
  double* part_out = P.part_buf[itg & 1];
  const double* part_in = P.part_buf[(itg & 1) ^ 1];
  const double rho = P.rho;
  double pri_m = 0.0, dual_m = 0.0;
  PT_DECL
  constexpr int CHW = 8 + 2 * TC;   // ints per chunk descriptor
  // unit descriptors, double-buffered in shared memory: the next unit's is
  // fetched (cp.async) while the current unit runs
  int* udesc = reinterpret_cast<int*>(smem + P.off_udesc);   // [2][16]
  const int* urange = reinterpret_cast<const int*>(smem + P.off_red + 32);   // staged at launch
  const int un_a = urange[0], un_b = urange[1];
  const bool single = un_b - un_a == 1;
  keep_tab = keep_tab && single;
  keep_pada = keep_pada && single;
  if (un_a < un_b && tid < 4 && !keep_tab)
    reinterpret_cast<int4*>(udesc)[tid] = __ldg(reinterpret_cast<const int4*>(P.unit_desc) + 4 * un_a + tid);
  __syncthreads();
  for (int un = un_a; un < un_b; ++un) {
    PT_START
    const int ub = (un - un_a) & 1;
    const int4 ud0 = reinterpret_cast<const int4*>(udesc + 16 * ub)[0];
    const int4 ud1 = reinterpret_cast<const int4*>(udesc + 16 * ub)[1];
    const int4 ud2 = reinterpret_cast<const int4*>(udesc + 16 * ub)[2];
    const int4 ud3 = reinterpret_cast<const int4*>(udesc + 16 * ub)[3];
    if (un + 1 < un_b && tid < 4) {
      cp_async16(reinterpret_cast<double*>(udesc + 16 * (ub ^ 1) + 4 * tid),
                 reinterpret_cast<const double*>(P.unit_desc + 16 * static_cast<size_t>(un + 1) + 4 * tid));
    }
    cp_async_commit();
    // the first chunks' ψ/λ copies start before the tables arrive
    if (ud2.z > 0) {
      stash_cols_bulk(P, ud2.w, ud2.z, psi, psi_st, bars + 0);
      stash_lam_bulk(P, ud2.w, ud2.z, lam, lam_st, ldl, bars + 2);
      if (ud3.x > 0) stash_cols_bulk(P, ud2.w + ud2.z, ud3.x, psi, psi_st + TC * ldk, bars + 1);
    }
    const int own_lo = ud0.x, own_hi = ud0.y, plo = ud0.z, phi_ = ud0.w;
    const long long prow0 = static_cast<long long>(static_cast<unsigned>(ud1.x)) |
                            (static_cast<long long>(ud1.y) << 32);
    const int prows = ud1.z, ch_a = ud1.w, ch_b = ud2.x, pt_off = ud2.y;
    const int npq = phi_ - plo;
    const int nch = ch_b - ch_a;
    // the unit's control tables: copy (un - un_a) & 1 of [chunk table | patch
    // table | raw ‖a‖² (from the even index below plo)]; the first unit of
    // the iteration loads its own, every later one was prefetched (cp.async)
    // into its copy during the previous unit
    const int tb = (un - un_a) & 1;
    int* chtab = chtab0 + 2 * tb * P.tab_alt;
    double* ptab = ptab0 + tb * P.tab_alt;
    if (un == un_a) {
      if (!keep_tab) {
        const int4* src = reinterpret_cast<const int4*>(P.chunk_desc + static_cast<size_t>(ch_a) * CHW);
        int4* dst = reinterpret_cast<int4*>(chtab);
        for (int q = tid; q < nch * CHW / 4; q += kThreads) dst[q] = __ldg(src + q);
        const double2* ps = reinterpret_cast<const double2*>(P.unit_ptab + static_cast<size_t>(pt_off) * 6);
        double2* pd = reinterpret_cast<double2*>(ptab);
        for (int q = tid; q < npq * 3; q += kThreads) pd[q] = __ldg(ps + q);
      }
      if (!keep_pada) {
        for (int q = tid; q < npq; q += kThreads) {
          const double a = ld_cg(P.ada + plo + q);
          pada0[q] = a > 0.0 ? 1.0 / a : 0.0;   // only read in iterations >= 1 (reciprocal form)
        }
      }
    } else {
      const double* raw = pada0 + P.np_cap + tb * P.tab_alt + (plo & 1);
      for (int q = tid; q < npq; q += kThreads) {
        const double a = raw[q];
        pada0[q] = a > 0.0 ? 1.0 / a : 0.0;
      }
    }
    double* const pada = pada0;
    __syncthreads();
    PT_LAP(P, 2)
    for (int q = warp; q < npq; q += kWarps) {
      const int* ei = reinterpret_cast<const int*>(ptab + 6 * q);
      for (int l = lane; l < ei[1]; l += 32) rowq[ei[0] + l] = q;
    }
    for (int r = tid; r < prows; r += kThreads) c_patch[r] = 0.0;
    // staging: ψ(a) -> ψ buffer 0, λ(a) -> λ buffer, ψ(a+1) -> ψ buffer 1
    // (TMA bulk copies, one per chunk and array; mbarriers ψ0, ψ1, λ)
    double x_first = 0.0;
    if (nch > 0 && tid < chtab[2]) x_first = ld_cg(x + chtab[1] + tid);   // consumed after the Φ loop
    PT_LAP(P, 3)
    // Φ scales of the patch rows
    if (itg == 0) {
      for (int i = plo + warp; i < phi_; i += kWarps) {
        const int r_off = static_cast<int>(P.row_start[i] - prow0);
        double* dst = s_patch + r_off;
        double* gdst = (i >= own_lo && i < own_hi) ? P.s_row + P.row_start[i] : nullptr;
        auto out = [dst, gdst](int l, double s) {
          dst[l] = s;
          if (gdst) gdst[l] = s;
        };
        phi_rows_of<false>(P, i, psi, lam, x, out,
                           (i >= own_lo && i < own_hi) ? P.row_invden + P.row_start[i] : nullptr);
      }
    } else {
      // partitioned sub-problem: patch subsystems whose ball holds another
      // rank's columns (flag ei[11]) get the full Φ from the exchanged ψ, λ
      if (P.own_sub_lo > 0 || P.own_sub_hi < P.n_sub) {
        for (int q = warp; q < npq; q += kWarps) {
          const int* ei = reinterpret_cast<const int*>(ptab + 6 * q);
          if (!ei[11]) continue;
          const int i = plo + q;
          double* dst = s_patch + ei[0];
          double* gdst = ei[10] ? P.s_row + P.row_start[i] : nullptr;
          auto out = [dst, gdst](int l, double s) {
            dst[l] = s;
            if (gdst) gdst[l] = s;
          };
          phi_rows_of<false>(P, i, psi, lam, x, out);
        }
      }
      // from the per-unit dot partials of the last iteration (slot order);
      // every thread issues the loads of up to kRB rows before using any
      constexpr int kRB = DLMPC_STREAM_KRB;
      for (int r0 = tid; r0 < prows; r0 += kRB * kThreads) {
        double w[kRB], lo[kRB], hi[kRB], c[kRB], ada[kRB];
        long long grow[kRB];
        bool own[kRB], ok[kRB];
#pragma unroll
        for (int u = 0; u < kRB; ++u) {
          const int r = r0 + u * kThreads;
          ok[u] = r < prows && !reinterpret_cast<const int*>(ptab + 6 * rowq[r < prows ? r : 0])[11];
          w[u] = lo[u] = hi[u] = c[u] = ada[u] = 0.0;
          grow[u] = 0; own[u] = false;
          if (ok[u]) {
            const int q = rowq[r];
            const double* e = ptab + 6 * q;
            const int* ei = reinterpret_cast<const int*>(e);
            const int l = r - ei[0], nr = ei[1], np = ei[2];
            grow[u] = reinterpret_cast<const long long*>(e)[4] + l;
            own[u] = ei[10] != 0;
            ada[u] = pada[q];
            const double* pb = part_in + reinterpret_cast<const long long*>(e)[2] + l;
            w[u] = __ldcg(P.row_invden + grow[u]); lo[u] = __ldg(P.row_lo + grow[u]); hi[u] = __ldg(P.row_hi + grow[u]);
            c[u] = __ldcg(pb);
            for (int sl = 1; sl < np; ++sl) c[u] += __ldcg(pb + sl * nr);
          }
        }
#pragma unroll
        for (int u = 0; u < kRB; ++u) {
          if (!ok[u]) continue;
          // w[] holds 1/(ρ + 2w·ada) (first iteration of the step), ada[] 1/ada
          const double y = fmin(fmax(rho * c[u] * w[u], lo[u]), hi[u]);
          const double sv = (y - c[u]) * ada[u];
          s_patch[r0 + u * kThreads] = sv;
          if (own[u] && DCHK_ROW(P, grow[u], 7)) P.s_row[grow[u]] = sv;
        }
      }
    }
    if (nch > 0 && tid < TC) {
      long long* mm = meta0;
      const bool ok = tid < chtab[2];
      mm[tid] = ok ? static_cast<long long>(chtab[1] + tid) * P.s_pad : 0;
      mm[TC + tid] = ok ? chtab[8 + tid] : 0;
      mm[2 * TC + tid] = ok ? static_cast<long long>(chtab[8 + TC + tid]) * P.s_pad : 0;
      reinterpret_cast<double*>(mm)[3 * TC + tid] = x_first;
    }
    if (tid < 4) cp_async_wait<0>();   // the next unit's descriptor (read after the barrier)
    __syncthreads();
    if (un + 1 < un_b) {
      // the next unit's tables -> the other copy, under this unit's chunks
      // (cp.async, waited at this unit's end)
      const int* nd = udesc + 16 * (ub ^ 1);
      const int n_plo = nd[2], n_np = nd[3] - nd[2], n_cha = nd[7], n_nch = nd[8] - nd[7], n_pt = nd[9];
      int* cdst = chtab0 + 2 * (tb ^ 1) * P.tab_alt;
      const int* csrc = P.chunk_desc + static_cast<size_t>(n_cha) * CHW;
      for (int q = tid; q < n_nch * CHW / 4; q += kThreads)
        cp_async16(reinterpret_cast<double*>(cdst + 4 * q), reinterpret_cast<const double*>(csrc + 4 * q));
      double* pdst = ptab0 + (tb ^ 1) * P.tab_alt;
      const double* psrc = P.unit_ptab + static_cast<size_t>(n_pt) * 6;
      for (int q = tid; q < n_np * 3; q += kThreads) cp_async16(pdst + 2 * q, psrc + 2 * q);
      double* adst = pada0 + P.np_cap + (tb ^ 1) * P.tab_alt;
      const int a0 = n_plo & ~1;
      for (int q = tid; 2 * q < n_plo + n_np - a0; q += kThreads) cp_async16(adst + 2 * q, P.ada + a0 + 2 * q);
    }
    cp_async_commit();
    PT_LAP(P, 0)
    // K = ψ + s·x (= φ + λ) in place, zero padded to TC x S4 (GEMM 1 k-steps
    // of 4); one warp per column
    auto k_pass = [&](double* kt, const long long* m_s, const double* m_x, int S, int nt_,
                      int w0 = 0, int nw = kWarps) {
      const int S4 = (S + 3) & ~3;
      for (int t = warp - w0; t < TC; t += nw) {
        double* kp = kt + t * ldk;
        const long long s0 = m_s[t];
        const double xc = m_x[t];
        for (int p = lane; p < S4; p += 32)
          kp[p] = (t < nt_ && p < S) ? fma(s_patch[s0 + p], xc, kp[p]) : 0.0;
      }
    };
    if (nch > 0) {   // first chunk: operator, ψ landed, K
      if (OPS) stage_operator_sized(P, chtab[0], (chtab[3] + 7) & ~7, chtab[5], smem, cur);
      mbar_wait(bars + 0, ph & 1u);
      ph ^= 1u;
      k_pass(psi_st, meta0 + TC, reinterpret_cast<const double*>(meta0 + 3 * TC), chtab[3], chtab[2]);
      __syncthreads();
    }
    PT_LAP(P, 4)
    auto row_pass = [&](const long long* m_s, const double* m_x, int S, int nt_, int t0, int nthr, bool paired) {
      const int rlo = static_cast<int>(m_s[0]);
      const int rhi = static_cast<int>(m_s[nt_ - 1]) + S;
      for (int r = rlo + t0; r < rhi; r += nthr) {
        double acc = c_patch[r];
        if (paired) {
          for (int t = 0; t < nt_; t += 2) {
            const int p = r - static_cast<int>(m_s[t]);
            if (p >= 0 && p < S) acc += lam_st[t * ldl + p];
          }
        } else {
          for (int t = 0; t < nt_; ++t) {
            const int p = r - static_cast<int>(m_s[t]);
            if (p >= 0 && p < S) acc = fma(lam_st[t * ldl + p], m_x[t], acc);
          }
        }
        c_patch[r] = acc;
      }
    };
    if (P.warp_spec) {
      // Hybrid pipeline: while warps 0..kCons-1 run GEMM 1 and GEMM 2 +
      // epilogue of chunk ch (13 warps split GEMM 2's 26 m-tiles evenly), the
      // other warps -- idle in the GEMMs -- build K(ch+1). The row pass of ch
      // stays a whole-CTA phase (latency-bound, it needs every thread).
#ifndef DLMPC_STREAM_CONS
#define DLMPC_STREAM_CONS 13
#endif
      constexpr int kCons = DLMPC_STREAM_CONS, kProd = kWarps - kCons;
      const bool prod = warp >= kCons;
      const int ptid = tid - kCons * 32;
      for (int ch = ch_a; ch < ch_b; ++ch) {
        const int cq = ch - ch_a;
        const int mb = cq & 1;
        const bool has_next = ch + 1 < ch_b, has_next2 = ch + 2 < ch_b;
        const int* ce = chtab + CHW * cq;
        const int nt = ce[2], S = ce[3], S8 = (S + 7) & ~7, S4 = (S + 3) & ~3, n08 = ce[4], ldn = ce[5];
        const long long* m_pos = meta0 + mb * 4 * TC;
        const long long* m_s = m_pos + TC;
        const long long* m_q = m_pos + 2 * TC;
        const double* m_x = reinterpret_cast<const double*>(m_pos + 3 * TC);
        double* kt = psi_st + mb * TC * ldk;
        if (prod) {
          if (has_next) {
            if (ptid < TC) {
              long long* mm = meta0 + (mb ^ 1) * 4 * TC;
              const bool ok = ptid < ce[CHW + 2];
              mm[ptid] = ok ? static_cast<long long>(ce[CHW + 1] + ptid) * P.s_pad : 0;
              mm[TC + ptid] = ok ? ce[CHW + 8 + ptid] : 0;
              mm[2 * TC + ptid] = ok ? static_cast<long long>(ce[CHW + 8 + TC + ptid]) * P.s_pad : 0;
              reinterpret_cast<double*>(mm)[3 * TC + ptid] = ok ? ld_cg(x + ce[CHW + 1] + ptid) : 0.0;
            }
            nbar_sync(6, kProd * 32);
            mbar_wait(bars + (mb ^ 1), (ph >> (mb ^ 1)) & 1u);
            const long long* mn = meta0 + (mb ^ 1) * 4 * TC;
            k_pass(psi_st + (mb ^ 1) * TC * ldk, mn + TC, reinterpret_cast<const double*>(mn + 3 * TC),
                   ce[CHW + 3], ce[CHW + 2], kCons, kProd);
          }
        } else {
          const double* nop = OPS ? smem : P.null_pool + P.class_null_off[ce[0]];
          PT_LAP(P, 1)
          gemm1<TC, NoHook, kCons, GroupBar<kCons>>(P, S4, n08, ldn, nop, kt, ldk, yb, P.ldy, yp);
          PT_LAP(P, 12)
          StreamEpi<TC> epi{P.psi[b ^ 1], P.lam[b ^ 1], P.q_pool, m_pos, m_s, m_q, m_x,
                            s_patch, kt, lam_st, ldk, ldl, S, nt, pri_m, dual_m, bars + 2, (ph >> 2) & 1u, ce[6] != 0};
#ifdef DLMPC_CHECKED
          epi.chk = CellChk{P.dbg, P.own_col_lo, P.own_col_hi, P.s_pad, P.col_len};
#endif
          if (DLMPC_STREAM_G2M16) gemm2_m16<TC, StreamEpi<TC>, kCons>(S8, n08, ldn, nop, yb, P.ldy, epi);
          else gemm2<TC, StreamEpi<TC>, kCons>(S8, n08, ldn, nop, yb, P.ldy, epi);
          pri_m = epi.pri_m; dual_m = epi.dual_m;
#ifdef DLMPC_PHASE_TIMING
          if (tid == 0) {
            pt_sh[9] += epi.t_kloop - pt_t0;
            pt_sh[10] += epi.t_lam - epi.t_kloop;
            pt_t0 = epi.t_lam;
          }
#endif
          PT_LAP(P, 13)
        }
        ph ^= 4u;
        if (has_next) ph ^= 1u << (mb ^ 1);
        __syncthreads();
        PT_LAP(P, 14)
        row_pass(m_s, m_x, S, nt, tid, kThreads, ce[6] != 0);
        __syncthreads();
        PT_LAP(P, 15)
        if (has_next) stash_lam_bulk(P, ce[CHW + 1], ce[CHW + 2], lam, lam_st, ldl, bars + 2);
        if (has_next2) stash_cols_bulk(P, ce[2 * CHW + 1], ce[2 * CHW + 2], psi, kt, bars + mb);
      }
    } else
    // chunk pipeline: GEMM 1 -> GEMM 2 + epilogue -> (row pass of this chunk
    // | K pass of the next) -> stage λ(next) and ψ(next+1)
    for (int ch = ch_a; ch < ch_b; ++ch) {
      const int cq = ch - ch_a;
      const int mb = cq & 1;
      const bool has_next = ch + 1 < ch_b, has_next2 = ch + 2 < ch_b;
      double* kt = psi_st + mb * TC * ldk;
      const long long* m_pos = meta0 + mb * 4 * TC;
      const long long* m_s = m_pos + TC;
      const long long* m_q = m_pos + 2 * TC;
      const double* m_x = reinterpret_cast<const double*>(m_pos + 3 * TC);
      const int* ce = chtab + CHW * cq;
      const int nt = ce[2], S = ce[3], S8 = (S + 7) & ~7, S4 = (S + 3) & ~3, n08 = ce[4], ldn = ce[5];
      double xn = 0.0;   // x of the next chunk's columns (meta written after GEMM 1)
      if (has_next && tid < ce[CHW + 2]) xn = ld_cg(x + ce[CHW + 1] + tid);
      const double* nop = OPS ? smem : P.null_pool + P.class_null_off[ce[0]];
      gemm1<TC, LamWait, kWarps, CtaBar, DLMPC_STREAM_MROW>(P, S4, n08, ldn, nop, kt, ldk, yb, P.ldy, yp,
                                                            LamWait{bars + 2, (ph >> 2) & 1u});
      ph ^= 4u;
      if (has_next && tid < TC) {
        long long* mm = meta0 + (mb ^ 1) * 4 * TC;
        const bool ok = tid < ce[CHW + 2];
        mm[tid] = ok ? static_cast<long long>(ce[CHW + 1] + tid) * P.s_pad : 0;
        mm[TC + tid] = ok ? ce[CHW + 8 + tid] : 0;
        mm[2 * TC + tid] = ok ? static_cast<long long>(ce[CHW + 8 + TC + tid]) * P.s_pad : 0;
        reinterpret_cast<double*>(mm)[3 * TC + tid] = xn;
      }
      PT_LAP(P, 2)
      StreamEpi<TC> epi{P.psi[b ^ 1], P.lam[b ^ 1], P.q_pool, m_pos, m_s, m_q, m_x,
                        s_patch, kt, lam_st, ldk, ldl, S, nt, pri_m, dual_m, nullptr, 0u, ce[6] != 0};
#ifdef DLMPC_CHECKED
      epi.chk = CellChk{P.dbg, P.own_col_lo, P.own_col_hi, P.s_pad, P.col_len};
#endif
      if (DLMPC_STREAM_G2M16) gemm2_m16<TC>(S8, n08, ldn, nop, yb, P.ldy, epi);
      else gemm2<TC>(S8, n08, ldn, nop, yb, P.ldy, epi);
      pri_m = epi.pri_m; dual_m = epi.dual_m;
      __syncthreads();
      PT_LAP(P, 3)
      // banded pass: row r of the patch gets v'(r - s0_t, t)·x_t from every
      // chunk column t whose support holds it, in ascending column order
      row_pass(m_s, m_x, S, nt, tid, kThreads, ce[6] != 0);
      if (has_next) {   // next chunk: operator, ψ landed, K
        const long long* mn = meta0 + (mb ^ 1) * 4 * TC;
        if (OPS) stage_operator_sized(P, ce[CHW], (ce[CHW + 3] + 7) & ~7, ce[CHW + 5], smem, cur);
        mbar_wait(bars + (mb ^ 1), (ph >> (mb ^ 1)) & 1u);
        ph ^= 1u << (mb ^ 1);
        k_pass(psi_st + (mb ^ 1) * TC * ldk, mn + TC, reinterpret_cast<const double*>(mn + 3 * TC),
               ce[CHW + 3], ce[CHW + 2]);
      }
      __syncthreads();
      if (has_next) stash_lam_bulk(P, ce[CHW + 1], ce[CHW + 2], lam, lam_st, ldl, bars + 2);
      if (has_next2) stash_cols_bulk(P, ce[2 * CHW + 1], ce[2 * CHW + 2], psi, kt, bars + mb);
      PT_LAP(P, 4)
    }
    PT_LAP(P, 1)
    cp_async_wait<0>();   // next unit's descriptor
    // this unit's Φ-dot partials -> its slot of every patch row
    for (int r = tid; r < prows; r += kThreads) {
      const int q = rowq[r];
      const double* e = ptab + 6 * q;
      const int* ei = reinterpret_cast<const int*>(e);
      const long long pidx = reinterpret_cast<const long long*>(e)[2] + static_cast<long long>(ei[3]) * ei[1] + (r - ei[0]);
      if (DCHK(P, pidx >= 0 && pidx < P.part_cap, 8, pidx)) part_out[pidx] =
          c_patch[r];
    }
    __syncthreads();
    PT_LAP(P, 7)
  }
  PT_START
  publish_residuals(P, it, pri_m, dual_m, smem + P.off_red);
  PT_LAP(P, 5)
}

// Exact column stage: one column per CTA at a time, the reference's dense
// projector with numpy's pairwise order (admm.py:183-186).
static __device__ void column_stage_exact(const DevProblem& P, int b, const double* x, int it, double* smem) {
  const int tid = threadIdx.x;
  const int sp = P.s_pad;
  double* phi_s = smem + P.off_ex;   // internal order
  double* lam_s = phi_s + sp;
  double* psi_s = lam_s + sp;
  double* kref = psi_s + sp;          // reference order
  double* pnew = kref + sp;           // internal order
  double* res_s = pnew + sp;          // [m_pad]
  const double* psi = P.psi[b];
  const double* lam = P.lam[b];
  double* psi_n = P.psi[b ^ 1];
  double* lam_n = P.lam[b ^ 1];
  double pri_m = 0.0, dual_m = 0.0;
  for (int c = P.own_col_lo + VBID; c < P.own_col_hi; c += VGRID) {
    const int owner = P.col_owner[c];
    const int k = P.col_class[c];
    const int S = P.class_s[k], m = P.class_m[k];
    const double* gk = P.g_pool + P.class_g_off[k];
    const double* pk = P.p_pool + P.class_p_off[k];
    const double* rhs = P.rhs_pool + static_cast<size_t>(P.col_vec[c]) * P.m_pad;
    const int* rp = P.ref_pos + static_cast<size_t>(owner) * sp;
    const double xc = ld_cg(x + c);
    if (!DCHK(P, S <= sp && m <= P.m_pad && k >= 0 && k < P.n_classes, 20, c)) continue;
    for (int p = tid; p < S; p += kThreads) {
      const size_t pos = static_cast<size_t>(c) * sp + p;
      const double ps = ld_cg(psi + pos), lm = ld_cg(lam + pos);
      const long long ir = P.contiguous ? P.col_rowbase[c] + p : P.col_irow[static_cast<size_t>(owner) * sp + p];
      if (!DCHK_ROW(P, ir, 21) || !DCHK(P, rp[p] >= 0 && rp[p] < S, 22, p)) continue;
      phi_s[p] = make_phi<true>(__dsub_rn(ps, lm), ld_cg(P.s_row + ir), xc);
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
      pnew[rp[q]] = __dadd_rn(kref[q], pairwise_sum(ProdRow{pk + static_cast<size_t>(q) * m, res_s}, 0, m));
    __syncthreads();
    for (int p = tid; p < S; p += kThreads) {
      const size_t pos = static_cast<size_t>(c) * sp + p;
      const double pn = pnew[p];
      const double d = __dsub_rn(phi_s[p], pn);
      if (DCHK_CELL(P, static_cast<long long>(pos), 4)) {
        psi_n[pos] = pn;
        lam_n[pos] = __dadd_rn(lam_s[p], d);
      }
      pri_m = rmax(pri_m, fabs(d));
      dual_m = rmax(dual_m, fabs(__dsub_rn(pn, psi_s[p])));
    }
    __syncthreads();
  }
  publish_residuals(P, it, pri_m, dual_m, smem + P.off_red);
}

// u_k = ascending dot of φ_r[input row k, t=0] with x (admm.py:350-360);
// φ is rebuilt from the iterate the last Φ stage read (buffer pb). One warp;
// the result in every lane.
template <bool EXACT>
__device__ __forceinline__ double control_value(const DevProblem& P, int pb, const double* x, int k) {
  const int lane = threadIdx.x & 31;
  const int i = P.input_owner[k], l = P.input_local[k];
  const double s = ld_cg(P.s_row + P.row_start[i] + l);
  const int D = P.supp_len[i];
  const int* sc = P.supp_col + static_cast<size_t>(i) * P.d_pad;
  const int* so = P.supp_off + static_cast<size_t>(i) * P.d_pad;
  double acc = 0.0;
  bool first = true;
  for (int q0 = 0; q0 < D; q0 += 32) {
    const int kn = min(32, D - q0);
    double pr = 0.0;
    if (lane < kn) {
      const int c = sc[q0 + lane];
      const size_t pos = static_cast<size_t>(c) * P.s_pad + so[q0 + lane] + l;
      const double xc = ld_cg(x + c);
      const double phi = make_phi<EXACT>(__dsub_rn(ld_cg(P.psi[pb] + pos), ld_cg(P.lam[pb] + pos)), s, xc);
      pr = __dmul_rn(phi, xc);
    }
    acc = warp_ordered_sum(acc, first, pr, kn);
  }
  return acc;
}

template <bool EXACT>
__device__ void control_stage(const DevProblem& P, int pb, const double* x) {
  for (long long k = wspread_first(P); k < P.n_inputs; k += wspread_step(P)) {
    const double u = control_value<EXACT>(P, pb, x, static_cast<int>(k));
    if ((threadIdx.x & 31) == 0) P.u[k] = u;
  }
}

// x+ = A x + B u on the plant's CSR rows (admm.py:363-369: scipy csr_matvec
// accumulates from 0 in stored order without FMA, then the two vectors add).
// U(k) supplies input k (warp-uniform): P.u after a control stage, or
// computed in place. One warp; the result in every lane.
template <class U>
__device__ __forceinline__ double plant_row(const DevProblem& P, const double* x, int r, const U& uval) {
  const int lane = threadIdx.x & 31;
  double ax = 0.0, bu = 0.0;
  bool first = false;   // csr_matvec starts from 0
  const long long a0 = P.a_ptr[r], a1 = P.a_ptr[r + 1];
  for (long long q0 = a0; q0 < a1; q0 += 32) {
    const int kn = static_cast<int>(min(32LL, a1 - q0));
    const double pr = lane < kn ? __dmul_rn(P.a_val[q0 + lane], ld_cg(x + P.a_idx[q0 + lane])) : 0.0;
    ax = warp_ordered_sum(ax, first, pr, kn);
  }
  for (long long q = P.b_ptr[r]; q < P.b_ptr[r + 1]; ++q) bu = __dadd_rn(bu, __dmul_rn(P.b_val[q], uval(P.b_idx[q])));
  return __dadd_rn(ax, bu);
}

static __device__ void plant_stage(const DevProblem& P, const double* x, double* xn) {
  for (long long r = wspread_first(P); r < P.n_cols; r += wspread_step(P)) {
    const double v = plant_row(P, x, static_cast<int>(r), [&](int k) { return ld_cg(P.u + k); });
    if ((threadIdx.x & 31) == 0) xn[r] = v;
  }
}

// Closed loop, end of an MPC step: control extraction and the plant step in
// one stage (no grid barrier between them). A state row computes the inputs
// its B row references itself -- the same arithmetic as control_value, so
// bitwise the u the input's own warp stores to P.u and the trajectory.
template <bool EXACT>
__device__ void control_plant_stage(const DevProblem& P, int pb, const double* x, double* xn, double* inputs_out,
                                    double* states_out) {
  const long long n_items = static_cast<long long>(P.n_inputs) + P.n_cols;
  const bool lane0 = (threadIdx.x & 31) == 0;
  for (long long w = wspread_first(P); w < n_items; w += wspread_step(P)) {
    if (w < P.n_inputs) {
      const double u = control_value<EXACT>(P, pb, x, static_cast<int>(w));
      if (lane0) { P.u[w] = u; inputs_out[w] = u; }
    } else {
      const long long r = w - P.n_inputs;
      const double v = plant_row(P, x, static_cast<int>(r), [&](int k) { return control_value<EXACT>(P, pb, x, k); });
      if (lane0) { xn[r] = v; states_out[r] = v; }
    }
  }
}

// Closed loop, patch mode with the Φ cache of one unit per CTA
// (P.fuse_steps): the end of an MPC step inside each CTA, with no grid
// barrier. Replaces control_plant_stage + grid barrier + row_data_stage +
// grid barrier + cache_phi_meta. Every CTA can read the final iterate
// (buffer pb, s_row) and x once the last iteration barrier has passed, so
// the CTA computes what its unit needs itself, over its window (FuseTab,
// staged in shared memory by fused_tables_load):
//  1. u of the window inputs (as control_value: the same bits as the input's
//     owner computes; the owners store P.u and the trajectory's inputs) --
//     the one global round trip of the transition: ψ, λ, x, s of the inputs'
//     rows, with x of W2 for the plant rows loaded under it; then the CTA
//     arrives on the split barrier (P.gbar), which the next step's first
//     iteration waits for before its first store into pb / s_row;
//  2. x+ of the window states (as plant_row, from shared memory); the owners
//     store x+ and the trajectory's states;
//  3. (refresh: a next step follows) the x-dependent Φ cache from the
//     window: x on the supports, ||a||^2 in ascending order as
//     row_data_stage (the owners store P.ada), 1/||a||^2, 1/(ρ + 2w·||a||^2),
//     x of the single chunk's columns. RowInfeasible (sls_core.py:346-348)
//     goes into next_bad; the next step tests it after its first iteration
//     barrier.
struct FuseSmem {
  double* fd; double* xo; double* xw; double* uw; double* wrow; int* fi;
  __device__ FuseSmem(const DevProblem& P, double* smem) {
    fd = smem + P.off_fw;
    xo = fd + P.ft_dcap;
    xw = xo + P.ft_w2cap;
    uw = xw + P.ft_wcap;
    wrow = uw + P.ft_ucap;
    fi = reinterpret_cast<int*>(wrow + P.patch_cap);
  }
};

// The unit's FuseTab and its patch rows' Φ weights into shared memory (once
// per launch; read after the next block barrier).
static __device__ void fused_tables_load(const DevProblem& P, double* smem) {
  const int un = P.cta_unit_ptr[VBID];
  if (un == P.cta_unit_ptr[VBID + 1]) return;
  FuseSmem f(P, smem);
  const int i0 = P.ft_iptr[un], ni = P.ft_iptr[un + 1] - i0;
  const int d0 = P.ft_dptr[un], nd = P.ft_dptr[un + 1] - d0;
  for (int q = threadIdx.x; q < ni; q += kThreads) f.fi[q] = P.ft_int[i0 + q];
  for (int q = threadIdx.x; q < nd; q += kThreads) f.fd[q] = P.ft_dbl[d0 + q];
  const long long prow0 = P.row_start[P.unit_patch_lo[un]];
  const int prows = static_cast<int>(P.row_start[P.unit_patch_hi[un]] - prow0);
  for (int q = threadIdx.x; q < prows; q += kThreads) f.wrow[q] = P.row_w[prow0 + q];
}

template <int TC>
__device__ void fused_transition(const DevProblem& P, int pb, const double* x, double* xn, double* inputs_out,
                                 double* states_out, double* smem, bool refresh, int* next_bad) {
  const int* urange = reinterpret_cast<const int*>(smem + P.off_red + 32);   // staged at launch
  const int un = urange[0];
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  if (un == urange[1]) {   // no unit: only the split-barrier arrival
    if (refresh && t == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" :: "l"(P.gbar) : "memory");
    return;
  }
  const FuseSmem f(P, smem);
  const int* fi = f.fi;
  const int nw = fi[FuseTab::kNw], nu = fi[FuseTab::kNu], nw2 = fi[FuseTab::kNw2], na = fi[FuseTab::kNa];
  const int* w2 = fi + fi[FuseTab::kW2];
  const double xr = t < nw2 ? ld_cg(x + w2[t]) : 0.0;   // stored after stage 1
  // 1. inputs
  const double* psi = P.psi[pb];
  const double* lam = P.lam[pb];
  for (int j = warp; j < nu; j += kWarps) {
    const int* hd = fi + fi[FuseTab::kUhead] + 4 * j;
    const int kf = hd[0], D = hd[2];
    const int* ue = fi + fi[FuseTab::kUent] + hd[3];
    const double s = ld_cg(P.s_row + hd[1]);
    double acc = 0.0;
    bool first = true;
    for (int q0 = 0; q0 < D; q0 += 32) {
      const int kn = min(32, D - q0);
      double pr = 0.0;
      if (lane < kn) {
        const int pos = ue[2 * (q0 + lane)], c = ue[2 * (q0 + lane) + 1];
        const double xc = ld_cg(x + c);
        const double phi = make_phi<false>(__dsub_rn(ld_cg(psi + pos), ld_cg(lam + pos)), s, xc);
        pr = __dmul_rn(phi, xc);
      }
      acc = warp_ordered_sum(acc, first, pr, kn);
    }
    if (lane == 0) {
      f.uw[j] = acc;
      if (kf & 1) { P.u[kf >> 1] = acc; inputs_out[kf >> 1] = acc; }
    }
  }
  if (t < nw2) f.xo[t] = xr;
  for (int q = t + kThreads; q < nw2; q += kThreads) f.xo[q] = ld_cg(x + w2[q]);
  __syncthreads();
  if (refresh && t == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" :: "l"(P.gbar) : "memory");
  // 2. states (csr_matvec order: from 0, no FMA; then + Bu)
  const int* aoff = fi + fi[FuseTab::kAoff];
  const int* boff = aoff + nw + 1;
  const int* aent = fi + fi[FuseTab::kAent];
  const int* bent = fi + fi[FuseTab::kBent];
  const int* wcol = fi + fi[FuseTab::kWcol];
  for (int j = warp; j < nw; j += kWarps) {
    double ax = 0.0, bu = 0.0;
    bool first = false;
    const int a0 = aoff[j], a1 = aoff[j + 1];
    for (int q0 = a0; q0 < a1; q0 += 32) {
      const int kn = min(32, a1 - q0);
      const double pr = lane < kn ? __dmul_rn(f.fd[q0 + lane], f.xo[aent[q0 + lane]]) : 0.0;
      ax = warp_ordered_sum(ax, first, pr, kn);
    }
    for (int q = boff[j]; q < boff[j + 1]; ++q) bu = __dadd_rn(bu, __dmul_rn(f.fd[na + q], f.uw[bent[q]]));
    const double v = __dadd_rn(ax, bu);
    if (lane == 0) {
      f.xw[j] = v;
      const int wf = wcol[j];
      if (wf & 1) { xn[wf >> 1] = v; states_out[wf >> 1] = v; }
    }
  }
  __syncthreads();
  if (!refresh) return;
  // 3. the next step's Φ cache (layout: cache_phi_meta)
  const int* ublk = reinterpret_cast<const int*>(smem + P.off_ublk);
  const int2* rinfo = reinterpret_cast<const int2*>(smem + P.off_ublk + 8);
  const int own_lo = ublk[1], own_hi = ublk[2], plo = ublk[3], np = ublk[4] - plo, prows = ublk[5];
  double* base = smem + P.off_phimeta;
  double* xk = base + static_cast<size_t>(np) * P.d_pad;
  double* ada = xk + static_cast<size_t>(np) * P.d_pad;
  double* rw = ada + np;
  const int* len = reinterpret_cast<const int*>(rw + 3 * prows);
  const int* fsup = fi + fi[FuseTab::kSupp];
  for (int q = warp; q < np; q += kWarps) {
    const int i = plo + q;
    const int D = len[q];
    double acc = 0.0;
    bool firstp = true;
    for (int k0 = 0; k0 < D; k0 += 32) {
      const int kn = min(32, D - k0);
      double xc = 0.0;
      if (lane < kn) {
        xc = f.xw[fsup[q * P.d_pad + k0 + lane]];
        xk[q * P.d_pad + k0 + lane] = xc;
      }
      acc = warp_ordered_sum(acc, firstp, __dmul_rn(xc, xc), kn);
    }
    if (D < P.d_row) acc = __dadd_rn(acc, 0.0);   // as row_data_stage
    if (lane == 0 && i >= own_lo && i < own_hi) {
      P.ada[i] = acc;
      if (acc == 0.0 && P.sub_first_bad[i] >= 0 && i >= P.own_sub_lo && i < P.own_sub_hi)
        atomicMin(next_bad, P.sub_first_bad[i]);
    }
    phi_cache_scales(P, acc, rinfo[q], f.wrow, ada + q, rw);
  }
  const int ch_a = ublk[8], ch_b = ublk[9];
  if (ch_b - ch_a == 1 && t < TC) {   // the single chunk's columns (own states: in the window)
    const int* mx = fi + fi[FuseTab::kMx];
    (smem + P.off_meta + 3 * TC)[t] = t < ublk[12] ? f.xw[mx[t]] : 0.0;
  }
  __syncthreads();
}

static __device__ void zero_iterate(const DevProblem& P, int b) {
  const size_t n = static_cast<size_t>(P.n_cols) * P.s_pad;
  const size_t gt = VBID * blockDim.x + threadIdx.x, GT = VGRID * blockDim.x;
  for (size_t q = gt; q < n; q += GT) { P.psi[b][q] = 0.0; P.lam[b][q] = 0.0; }
}


// ---------------------------------------------------------------------------
// Device-side exchange of the graph-partitioned solve (P.dist).
// Called by every CTA after the rank's grid barrier of iteration `it`, with
// ψ', λ' of the owned columns in buffer b and the rank's residual maxima in
// P.resid[2 it]:
//  1. every CTA stores its share of the halo cells the neighbour ranks read
//     straight into THEIR buffer b (peer memory), fences at system scope and
//     bumps each neighbour's arrival counter;
//  2. CTA 0 posts the rank's two maxima into every rank's slot table
//     (parity (epoch + it) & 1) and bumps every rank's residual counter;
//  3. thread 0 of every CTA waits (acquire, system scope) for all CTAs of
//     all sending neighbours and for all ranks' maxima of this iteration;
//     a ~4 s bound turns a protocol failure into an error instead of a hang;
//  4. a grid barrier makes the outcome uniform; every CTA forms the global
//     maxima from the slots -- the same bits on every rank, so every rank
//     takes the same stop decision.
// Buffer b of a rank is written by its neighbours only in halo cells it
// never writes itself, and only after the rank has finished reading b
// (ping-pong: iteration it+1 reads b, writes b^1; a neighbour's next push
// into b follows this rank's next arrival). Replaces the host-driven pack /
// NCCL send-recv / unpack / all-reduce per iteration (partition.py).
// Returns false on an exchange failure (P.d_abort set).
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned ld_acquire_sys_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <class Grid>
__device__ bool dist_exchange(const DevProblem& P, const RunArgs& R, int it, int b, Grid& grid,
                              unsigned long long* out2) {
  const int tid = threadIdx.x;
  const size_t gt = static_cast<size_t>(VBID) * blockDim.x + tid, GT = static_cast<size_t>(VGRID) * blockDim.x;
  const unsigned k = R.dist_epoch + static_cast<unsigned>(it);   // global iteration index
  const int par = k & 1;
  const double* psi = P.psi[b];
  const double* lam = P.lam[b];
  for (size_t i = gt; i < static_cast<size_t>(P.d_nsend); i += GT) {
    const int q = P.d_send_peer[i];
    const long long src = P.d_send_src[i], dst = P.d_send_dst[i];
    P.d_peer_psi[2 * q + b][dst] = psi[src];
    P.d_peer_lam[2 * q + b][dst] = lam[src];
  }
  __threadfence_system();
  __syncthreads();
  if (tid == 0)
    for (int q = 0; q < P.d_npeer; ++q) atomicAdd_system(P.d_peer_flag[q], 1u);
  if (VBID == 0 && tid == 0) {
    const unsigned long long rp = __ldcg(P.resid + 2 * it), rd = __ldcg(P.resid + 2 * it + 1);
    for (int r = 0; r < P.d_world; ++r) {
      volatile unsigned long long* slot = P.d_all_slots[r] + (static_cast<size_t>(par) * P.d_world + P.d_rank) * 2;
      slot[0] = rp;
      slot[1] = rd;
    }
    __threadfence_system();
    for (int r = 0; r < P.d_world; ++r) atomicAdd_system(P.d_all_rflag[r], 1u);
  }
  if (tid == 0) {
    const unsigned want_h = (k + 1) * P.d_halo_per_iter, want_r = (k + 1) * static_cast<unsigned>(P.d_world);
    const long long t0 = clock64();
    while (static_cast<int>(ld_acquire_sys_u32(P.d_flag) - want_h) < 0 ||
           static_cast<int>(ld_acquire_sys_u32(P.d_rflag) - want_r) < 0) {
      if (*reinterpret_cast<volatile int*>(P.d_abort)) break;
      if (clock64() - t0 > (8LL << 30)) { atomicExch(P.d_abort, 1); break; }
    }
  }
  __syncthreads();
  fence_proxy_async_global();   // the neighbours' stores are read by TMA bulk copies next
  grid.sync();
  if (*reinterpret_cast<volatile int*>(P.d_abort)) return false;
  unsigned long long mp = 0ull, md = 0ull;
  const volatile unsigned long long* own = P.d_slots + static_cast<size_t>(par) * P.d_world * 2;
  for (int r = 0; r < P.d_world; ++r) {   // ordered bits of non-negative maxima: NaN wins
    const unsigned long long a = own[2 * r] & 0x7fffffffffffffffull, c = own[2 * r + 1] & 0x7fffffffffffffffull;
    mp = a > mp ? a : mp;
    md = c > md ? c : md;
  }
  out2[0] = mp;
  out2[1] = md;
  return true;
}

// Kernel variants beyond (TC, MODE), each its own instantiation so the common
// path keeps its register allocation (measured: the dist branch compiled
// into the stream kernel cost 3% at N=1e4, the pair branch 1.6% on small
// patch cells):
constexpr int kVarDist = 1;    // graph-partitioned solve, exchange on the device (non-patch modes)
constexpr int kVarPairs = 2;   // patch mode with K-split CTA pairs
constexpr int kVarFuse = 4;    // patch mode closed loops, warm-started: fused MPC-step transitions (P.fuse_steps)
constexpr int kVarPcache = 8;  // patch mode with the partial Φ cache (P.cache_phi == 2; compiled into the
                               // common kernel it spilled and cost the other C4 cells 4%)

template <int TC, int MODE, int VAR>
__device__ __forceinline__ void persistent_body(const DevProblem& P, const RunArgs& R);

template <int TC, int MODE, int VAR = 0>
__global__ void __launch_bounds__(kThreads, 1) dlmpc_persistent(DevProblem P, RunArgs R) {
  persistent_body<TC, MODE, VAR>(P, R);
}

#ifdef DLMPC_VB_SHIFT
// The ranks of a graph-partitioned solve as contiguous CTA slices of ONE
// cooperative grid on one GPU (cta_base[r] .. cta_base[r+1]), each running
// its own sub-problem: the one-GPU test of the device-side exchange
// (dlmpc_multi.cu).
template <int TC, int MODE>
__global__ void __launch_bounds__(kThreads, 1) dlmpc_multi_kernel(const DevProblem* probs, const RunArgs* runs,
                                                                  const int* cta_base, int n_ranks) {
  int r = 0;
  while (r + 1 < n_ranks && static_cast<int>(blockIdx.x) >= cta_base[r + 1]) ++r;
  persistent_body<TC, MODE, kVarDist>(probs[r], runs[r]);   // probs[r].vbase / vgrid: the rank's slice
}
#endif

template <int TC, int MODE, int VAR>
__device__ __forceinline__ void persistent_body(const DevProblem& P, const RunArgs& R) {
  constexpr bool EXACT = MODE == kExact;
  constexpr bool PATCH = MODE == kPatch || MODE == kPatchRb;
  extern __shared__ __align__(16) double smem[];
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x;
  const bool leader = VBID == 0 && tid == 0;
  int cur = -1;   // class whose operator is staged at smem offset 0
  int b = P.ctl[4];
  unsigned ph = 0u;   // stream mode: mbarrier phase bits (ψ0, ψ1, λ) -- a register, not an indexed array
  if (MODE == kStream) {
    if (tid < 3) mbar_init(reinterpret_cast<unsigned long long*>(smem + P.off_bar) + tid, 1);
    __syncthreads();
  }
  const size_t gt = VBID * blockDim.x + tid, GT = VGRID * blockDim.x;
  PT_INIT
  if (MODE == kPatch) class_table_load(P, smem);   // DMMA patch chunks; read after step 0's grid barrier
  int lit = 0;   // stream mode: iterations run in this launch (table reuse, stream_iteration)
  if ((PATCH || MODE == kStream) && tid == 0) {   // the unit range (read after step 0's grid barrier)
    int* ur = reinterpret_cast<int*>(smem + P.off_red + 32);
    ur[0] = P.cta_unit_ptr[VBID];
    ur[1] = P.cta_unit_ptr[VBID + 1];
  }
  // fused MPC-step transitions (fused_transition; the host launches this
  // variant only for warm-started closed loops of more than one step with
  // P.fuse_steps): from step 1 on, no grid barrier between steps. A step's
  // residual words then rotate over three regions and its RowInfeasible slot
  // over three (ctl 2, 3, 6): a region is zeroed one step ahead, when every
  // CTA has passed the first iteration barrier of the step after its last
  // reader's.
  constexpr bool fuse = PATCH && (VAR & kVarFuse) != 0;
  // patch modes: the iteration barrier's counter value at launch (stable: the
  // previous launch has ended, and no CTA arrives before the first grid.sync);
  // fused: also read by the last warp, which waits on the split barriers
  const unsigned bar_base = (PATCH && (tid == 0 || (fuse && tid == kThreads - 32))) ? ld_acquire_u32(P.gbar) : 0u;
  unsigned bar_epoch = 0;
  int pair_cnt = 0;   // K-split pairs: partial-Y publications of this CTA in this launch
  unsigned pre_target = 0u;   // fused: the split barrier the next step's first iteration waits for
  if constexpr (fuse) fused_tables_load(P, smem);   // read after step 0's grid barrier
  for (int step = 0; step < R.t_sim; ++step) {
    PT_DECL
    PT_START
    const double* x = P.x[R.closed_loop ? (step & 1) : 0];
    const int roff = fuse ? (step % 3) * 2 * R.max_iters : 0;
    if (!fuse || step == 0) {
      int* bad_slot = P.ctl + 2 + (step & 1);
      for (size_t q = gt; q < static_cast<size_t>((fuse ? 4 : 2) * R.max_iters); q += GT) P.resid[q] = 0ull;
      if (R.closed_loop) {
        row_data_stage(P, x, bad_slot);
        if ((R.cold_start && step == 0) || !R.warm_start) zero_iterate(P, b);
      }
      if (MODE == kStream) fence_proxy_async_global();   // zeroed ψ, λ are read by TMA
      grid.sync();
      if (R.closed_loop) {
        const int bad = *reinterpret_cast<volatile int*>(bad_slot);
        if (bad != kBadNone) {
          if (leader) { P.ctl[0] = 2; P.ctl[1] = step; P.ctl[5] = 0; P.ctl[4] = b; }
          return;
        }
        if (leader) {
          P.ctl[2 + ((step + 1) & 1)] = kBadNone;
          if (fuse) P.ctl[6] = kBadNone;
        }
      }
      PT_LAP(P, 8)
      if (PATCH && P.cache_phi) cache_phi_meta<TC>(P, x, smem, step == 0);
      PT_LAP(P, 9)
    } else {   // the Φ cache came from the previous step's transition
      const size_t z = static_cast<size_t>(((step + 1) % 3) * 2 * R.max_iters);
      for (size_t q = gt; q < static_cast<size_t>(2 * R.max_iters); q += GT) P.resid[z + q] = 0ull;
    }
    int it = 0;
    bool conv = false;
    if (PATCH) {
      // stop test of iteration it-1 overlapped with iteration it's first Φ
      while (true) {
        PT_DECL
        if (it == R.max_iters) {
          if (it > 0) {
            const unsigned long long rp = __ldcg(P.resid + roff + 2 * (it - 1));
            const unsigned long long rd = __ldcg(P.resid + roff + 2 * (it - 1) + 1);
            conv = patch_stop_test(P, R, it, rp, rd);
          }
          break;
        }
        bar_epoch += VGRID;
        if (patch_iteration<TC, MODE == kPatchRb, (VAR & kVarPairs) != 0, fuse, PATCH && (VAR & kVarPcache) != 0>(
                P, b, x, it, smem, cur, R, bar_base + bar_epoch, pair_cnt, roff, it == 0 ? pre_target : 0u)) {
          bar_epoch -= VGRID;   // returned before arriving
          conv = true;
          break;
        }
        b ^= 1;
        ++it;
        if (fuse && step > 0 && it == 1) {   // the RowInfeasible test of this step's transition
          int* slot = (step % 3) == 2 ? P.ctl + 6 : P.ctl + 2 + step % 3;
          const int bad = *reinterpret_cast<volatile int*>(slot);
          if (bad != kBadNone) {   // the step's iterate in b ^ 1 is untouched
            if (leader) { P.ctl[2 + (step & 1)] = bad; P.ctl[0] = 2; P.ctl[1] = step; P.ctl[5] = 0; P.ctl[4] = b ^ 1; }
            return;
          }
          if (leader) {   // the slot of step + 2; its last reader has passed this barrier
            const int j = (step + 2) % 3;
            *(j == 2 ? P.ctl + 6 : P.ctl + 2 + j) = kBadNone;
          }
        }
      }
    }
    while (!PATCH && it < R.max_iters) {
      PT_DECL
      if (MODE == kStream) {
        const int itg = it + (R.closed_loop ? 0 : R.it_base);
        if (P.cta_gop && P.cta_gop[VBID]) stream_iteration<TC, false>(P, b, x, it, itg, smem, cur, ph, lit > 0, lit > 0 && it > 0);
        else stream_iteration<TC, true>(P, b, x, it, itg, smem, cur, ph, lit > 0, lit > 0 && it > 0);
        ++lit;
        fence_proxy_async_global();
        PT_START
      } else {
        PT_START
        phi_stage_global<EXACT>(P, b, x);
        PT_LAP(P, 0)
        grid.sync();
        PT_LAP(P, 6)
        if (EXACT) column_stage_exact(P, b, x, it, smem);
        else column_stage_tiles<TC>(P, b, x, it, smem, cur);
        PT_START
      }
      grid.sync();
      PT_LAP(P, 6)
      b ^= 1;
      // one load of the residual words per CTA, broadcast through shared memory
      unsigned long long* rbc = reinterpret_cast<unsigned long long*>(smem + P.off_red);
      if constexpr ((VAR & kVarDist) != 0) {   // the halo to the neighbour ranks, the global maxima from all ranks
        unsigned long long g2[2];
        if (!dist_exchange(P, R, it, b, grid, g2)) {
          if (leader) { P.ctl[0] = 4; P.ctl[1] = step; P.ctl[5] = it; P.ctl[4] = b; }
          return;
        }
        if (tid == 0) { rbc[0] = g2[0]; rbc[1] = g2[1]; }
      } else if (tid == 0) {
        rbc[0] = __ldcg(P.resid + 2 * it); rbc[1] = __ldcg(P.resid + 2 * it + 1);
      }
      __syncthreads();
      const double pri = __longlong_as_double(static_cast<long long>(rbc[0]));
      const double dual = P.rho * __longlong_as_double(static_cast<long long>(rbc[1]));
      __syncthreads();   // the slots are reused by the next iteration's residual publish
      if (leader) { R.hist[2 * it] = pri; R.hist[2 * it + 1] = dual; }
      ++it;
      if (R.stop_on_conv && pri <= R.eps_pri && dual <= R.eps_dual) { conv = true; break; }
    }
    PT_START
    if (leader) R.step_iters[step] = it;
    if (R.stop_on_conv && !conv) {
      PT_FLUSH(P)
      if (leader) { P.ctl[0] = 1; P.ctl[1] = step; P.ctl[5] = it; P.ctl[4] = b; }
      return;
    }
    if (R.closed_loop) {
      if (step == 0) {
        for (size_t q = gt; q < static_cast<size_t>(P.n_cols); q += GT) R.states[q] = x[q];
      }
      double* xn = P.x[(step + 1) & 1];
      if (fuse) {
        const bool refresh = step + 1 < R.t_sim;
        const int j = (step + 1) % 3;
        fused_transition<TC>(P, b ^ 1, x, xn, R.inputs + static_cast<size_t>(step) * P.n_inputs,
                             R.states + static_cast<size_t>(step + 1) * P.n_cols, smem, refresh,
                             j == 2 ? P.ctl + 6 : P.ctl + 2 + j);
        if (refresh) { bar_epoch += VGRID; pre_target = bar_base + bar_epoch; }
        PT_LAP(P, 10)
      } else {
        control_plant_stage<EXACT>(P, b ^ 1, x, xn, R.inputs + static_cast<size_t>(step) * P.n_inputs,
                                   R.states + static_cast<size_t>(step + 1) * P.n_cols);
        PT_LAP(P, 10)
        grid.sync();
        PT_LAP(P, 11)
      }
    }
  }
  PT_FLUSH(P)
  if (leader) { P.ctl[0] = 0; P.ctl[4] = b; }
}

#ifndef DLMPC_MULTI_TU   // the plain kernels live in the production translation unit only
// Row data for the solve API (dlmpc_set_x): a plain launch.
__global__ void set_x_kernel(DevProblem P) { row_data_stage(P, P.x[0], P.ctl + 2); }

// φ of the last iteration, internal column layout (for dlmpc_get(DLMPC_PHI)).
template <bool EXACT>
__global__ void phi_materialize_kernel(DevProblem P, int pb, double* out) {
  const size_t n = static_cast<size_t>(P.n_cols) * P.s_pad;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n; q += (size_t)gridDim.x * blockDim.x) {
    const int c = static_cast<int>(q / P.s_pad), p = static_cast<int>(q % P.s_pad);
    double v = 0.0;
    if (p < P.col_len[c]) {
      const long long ir = P.contiguous ? P.col_rowbase[c] + p
                                        : P.col_irow[static_cast<size_t>(P.col_owner[c]) * P.s_pad + p];
      v = make_phi<EXACT>(__dsub_rn(P.psi[pb][q], P.lam[pb][q]), P.s_row[ir], P.x[0][c]);
    }
    out[q] = v;
  }
}

// ---------------------------------------------------------------------------
// Fixed-point audit (reference verify_fixed_point, admm.py:417-434), run on
// the current iterate after a solve. Plain (non-cooperative) launches.
// ---------------------------------------------------------------------------

__device__ __forceinline__ void atomic_max_nonneg(double* dst, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(dst), static_cast<unsigned long long>(__double_as_longlong(v)));
}

// Φ scale at the current dual point (buffer b) for every row -> s_fresh.
template <bool EXACT>
__global__ void audit_phi_kernel(DevProblem P, int b, const double* x, double* s_fresh) {
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= P.n_sub) return;   // warp-uniform
  double* dst = s_fresh + P.row_start[i];
  phi_rows_of<EXACT>(P, i, P.psi[b], P.lam[b], x, [dst](int l, double s) { dst[l] = s; });
}

// re-solve residual max|φ_fresh - φ| and consensus gap max|φ - ψ| over every
// support entry (the reference's row_valid cells, admm.py:430-433).
template <bool EXACT>
__global__ void audit_entries_kernel(DevProblem P, int b, const double* x, const double* s_fresh,
                                     const double* phi_given, double* out) {
  __shared__ double red[64];
  double res = 0.0, gap = 0.0;
  const size_t n = static_cast<size_t>(P.n_cols) * P.s_pad;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n; q += (size_t)gridDim.x * blockDim.x) {
    const int c = static_cast<int>(q / P.s_pad), p = static_cast<int>(q % P.s_pad);
    if (p >= P.col_len[c]) continue;
    const long long ir = P.contiguous ? P.col_rowbase[c] + p
                                      : P.col_irow[static_cast<size_t>(P.col_owner[c]) * P.s_pad + p];
    const double xc = x[c];
    const double phi = phi_given ? phi_given[q]
                                 : make_phi<EXACT>(__dsub_rn(P.psi[b ^ 1][q], P.lam[b ^ 1][q]), P.s_row[ir], xc);
    const double fresh = make_phi<EXACT>(__dsub_rn(P.psi[b][q], P.lam[b][q]), s_fresh[ir], xc);
    res = rmax(res, fabs(__dsub_rn(fresh, phi)));
    gap = rmax(gap, fabs(__dsub_rn(phi, P.psi[b][q])));
  }
  for (int o = 16; o > 0; o >>= 1) {
    res = rmax(res, __shfl_xor_sync(0xffffffffu, res, o));
    gap = rmax(gap, __shfl_xor_sync(0xffffffffu, gap, o));
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { red[2 * warp] = res; red[2 * warp + 1] = gap; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (blockDim.x >> 5); ++w) { res = rmax(res, red[2 * w]); gap = rmax(gap, red[2 * w + 1]); }
    atomic_max_nonneg(out + 1, res);
    atomic_max_nonneg(out + 2, gap);
  }
}

// dynamics residual max|z ψ - rhs| restricted to each column's touched rows
// (the reference multiplies the sparse operator by the dense response:
// CSR order, products rounded then summed from zero, admm.py:427).
__global__ void audit_dynamics_kernel(DevProblem P, int b, double* out) {
  __shared__ double red[32];
  double worst = 0.0;
  for (int c = blockIdx.x; c < P.n_cols; c += gridDim.x) {
    const int k = P.col_class[c];
    const int S = P.class_s[k], nt = P.class_ntouch[k];
    const double* g0 = P.g0_pool + P.class_g0_off[k];
    const int* perm = P.perm_pool + P.class_perm_off[k];
    const double* psi = P.psi[b] + static_cast<size_t>(c) * P.s_pad;
    for (int i = threadIdx.x; i < nt; i += blockDim.x) {
      double acc = 0.0;
      for (int j = 0; j < S; ++j) {
        const double v = g0[static_cast<size_t>(i) * S + j];
        if (v != 0.0) acc = __dadd_rn(acc, __dmul_rn(v, psi[perm[j]]));
      }
      if (i == P.col_pin[c]) acc = __dsub_rn(acc, 1.0);
      worst = rmax(worst, fabs(acc));
    }
  }
  for (int o = 16; o > 0; o >>= 1) worst = rmax(worst, __shfl_xor_sync(0xffffffffu, worst, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = worst;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (blockDim.x >> 5); ++w) worst = rmax(worst, red[w]);
    atomic_max_nonneg(out, worst);
  }
}

// Control extraction and plant step for the loaded x after a host-driven
// solve (graph-partitioned multi-GPU path): plain launches, grid-stride.
template <bool EXACT>
__global__ void control_kernel(DevProblem P, int pb) { control_stage<EXACT>(P, pb, P.x[0]); }
__global__ void plant_kernel(DevProblem P) { plant_stage(P, P.x[0], P.x[1]); }

// Halo exchange of the partitioned path (partition.py halo_cells): gather
// the (ψ, λ) entries a neighbour reads into one interleaved message, and
// scatter a received message into the halo cells. Grid-stride, coalesced on
// the message side.
__global__ void halo_pack_kernel(const double* __restrict__ psi, const double* __restrict__ lam,
                                 const int64_t* __restrict__ cells, int64_t n, double2* __restrict__ out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = cells[k];
    out[k] = make_double2(psi[c], lam[c]);
  }
}

__global__ void halo_unpack_kernel(double* __restrict__ psi, double* __restrict__ lam,
                                   const int64_t* __restrict__ cells, int64_t n, const double2* __restrict__ in) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = cells[k];
    const double2 v = in[k];
    psi[c] = v.x;
    lam[c] = v.y;
  }
}
#endif  // DLMPC_MULTI_TU

}  // namespace dlmpc
