// dlmpc.cu -- host side (C ABI, include/dlmpc.h) of the B200 DLMPC ADMM hot
// path. Device code: dlmpc_device.cuh. The library owns all device memory of
// a problem (one handle), builds the CTA work decomposition for the SM count
// it finds, sizes the shared-memory plan, and launches exactly one persistent
// cooperative kernel per solve / iterate / closed loop.
#include "../../include/dlmpc.h"
#include "dlmpc_device.cuh"

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

using namespace dlmpc;

namespace {
thread_local std::string g_global_error;
}  // namespace

namespace dlmpc {   // dlmpc_multi.cu
cudaError_t launch_multi_kernel(int mode, int tc, const DevProblem* probs, const RunArgs* runs,
                                const int* cta_base, int n_ranks, int grid, int smem, cudaStream_t stream);
}

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
  double* d_scratch2 = nullptr;
  double* d_audit = nullptr;
  int mode = kPatch, n_units = 0;
  int it_cont = 0;   // iterations run on the current state (reset by any state change)
  int64_t* d_send_cells = nullptr; int64_t n_send = 0;
  int64_t* d_recv_cells = nullptr; int64_t n_recv = 0;
  double* d_halo = nullptr;
  char* h_stage = nullptr; size_t stage_cap = 0;   // pinned staging of dlmpc_simulate's host copies
  char* d_stage = nullptr;                          // its device mirror: one D2H copy per closed loop
  cudaStream_t own_stream = nullptr;   // the handle's stream; `stream` may be an external one (dlmpc_set_stream)
  int cur_b = 0, b_valid = 1;          // current ψ/λ buffer as known on the host (ctl[4])
  int dist_world = 0;                  // > 0 once dlmpc_dist_alloc ran
  unsigned dist_epoch = 0;             // iterations of the earlier dist launches (counter base)
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

KernelFn pick_kernel(int mode, int tc, int rb = 0) {
  if (mode == kExact) return dlmpc_persistent<8, kExact>;
  if (mode == kPatch && rb) return dlmpc_persistent<8, kPatchRb>;   // TC 8 only
  if (mode == kPatch) return tc == 16 ? dlmpc_persistent<16, kPatch> : dlmpc_persistent<8, kPatch>;
  if (mode == kStream) return tc == 16 ? dlmpc_persistent<16, kStream> : dlmpc_persistent<8, kStream>;
  return tc == 16 ? dlmpc_persistent<16, kTwoPhase> : dlmpc_persistent<8, kTwoPhase>;
}

// the instantiation with the K-split pairs (patch mode) or the device-side
// exchange (dlmpc_dist_solve; non-patch modes)
KernelFn pick_kernel_var(int mode, int tc, int var) {
  if (var == kVarPairs && mode == kPatch)
    return tc == 16 ? dlmpc_persistent<16, kPatch, kVarPairs> : dlmpc_persistent<8, kPatch, kVarPairs>;
  if (var == kVarPcache && mode == kPatch)
    return tc == 16 ? dlmpc_persistent<16, kPatch, kVarPcache> : dlmpc_persistent<8, kPatch, kVarPcache>;
  if (var == (kVarPairs | kVarPcache) && mode == kPatch)
    return tc == 16 ? dlmpc_persistent<16, kPatch, kVarPairs | kVarPcache>
                    : dlmpc_persistent<8, kPatch, kVarPairs | kVarPcache>;
  if (var == kVarFuse && mode == kPatch) return tc == 16 ? dlmpc_persistent<16, kPatch, kVarFuse> : dlmpc_persistent<8, kPatch, kVarFuse>;
  if (var == kVarFuse && mode == kPatchRb) return dlmpc_persistent<8, kPatchRb, kVarFuse>;
  if (var == kVarDist) {
    if (mode == kExact) return dlmpc_persistent<8, kExact, kVarDist>;
    if (mode == kStream) return tc == 16 ? dlmpc_persistent<16, kStream, kVarDist> : dlmpc_persistent<8, kStream, kVarDist>;
    if (mode == kTwoPhase) return tc == 16 ? dlmpc_persistent<16, kTwoPhase, kVarDist> : dlmpc_persistent<8, kTwoPhase, kVarDist>;
  }
  return nullptr;
}

int ld_frag(int n) {   // smallest ld >= n with ld % 16 in {4, 12}: conflict-free FP64 fragments
  int ld = std::max(n, 1);
  while (ld % 16 != 4 && ld % 16 != 12) ++ld;
  return ld;
}

// Grow-only run buffers. The replacements are allocated first and swapped in
// only when every allocation succeeded: a failed grow leaves the handle with
// its old (valid) buffers and capacities, never with freed pointers.
template <class T>
void swap_in(T** field, T* fresh) {
  if (*field) cudaFree(*field);
  *field = fresh;
}

int ensure_run_buffers(dlmpc_handle* h, int max_iters, int t_sim) {
  if (max_iters > h->max_iters_cap) {
    double* hist = nullptr; unsigned long long* resid = nullptr;
    cudaError_t e = cudaMalloc(&hist, sizeof(double) * 2 * max_iters);
    // three regions of 2 * max_iters words (fused MPC-step transitions rotate over them)
    if (e == cudaSuccess) e = cudaMalloc(&resid, sizeof(unsigned long long) * 6 * max_iters);
    if (e != cudaSuccess) {
      if (hist) cudaFree(hist);
      return fail(h, DLMPC_CUDA_ERROR, std::string("run buffers: ") + cudaGetErrorString(e));
    }
    swap_in(&h->d_hist, hist);
    swap_in(&h->P.resid, resid);
    h->max_iters_cap = max_iters;
  }
  if (t_sim > h->states_cap) {
    int* it = nullptr; double* st = nullptr; double* in = nullptr;
    cudaError_t e = cudaMalloc(&it, sizeof(int) * t_sim);
    if (e == cudaSuccess) e = cudaMalloc(&st, sizeof(double) * (size_t)(t_sim + 1) * h->P.n_cols);
    if (e == cudaSuccess) e = cudaMalloc(&in, sizeof(double) * (size_t)t_sim * (h->P.n_inputs ? h->P.n_inputs : 1));
    if (e != cudaSuccess) {
      if (it) cudaFree(it);
      if (st) cudaFree(st);
      return fail(h, DLMPC_CUDA_ERROR, std::string("closed-loop buffers: ") + cudaGetErrorString(e));
    }
    swap_in(&h->d_step_iters, it);
    swap_in(&h->d_states, st);
    swap_in(&h->d_inputs, in);
    h->states_cap = t_sim;
  }
  return DLMPC_OK;
}

int launch(dlmpc_handle* h, const RunArgs& R, int var = 0) {
  KernelFn fn = pick_kernel(h->mode, h->P.tile_cols, h->P.rb_gemv);
  if (h->P.cta_pair && h->mode == kPatch) var |= kVarPairs;
  if (h->P.cache_phi == 2 && h->mode == kPatch) var |= kVarPcache;
  if (h->P.fuse_steps && R.closed_loop && R.warm_start && R.t_sim > 1) var |= kVarFuse;
  if (var) fn = pick_kernel_var(var == kVarFuse && h->P.rb_gemv ? kPatchRb : h->mode, h->P.tile_cols, var);
  if (!fn) return fail(h, DLMPC_BAD_ARGUMENT, "no kernel variant for this mode");
  // the shared-memory limit is a per-function attribute: sessions of one
  // instantiation with different plans (the ranks of a partitioned solve in
  // one process) each set their own before launching
  CUDA_OR_FAIL(h, cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, h->smem_bytes));
  DevProblem P = h->P;
  RunArgs Rc = R;
  void* args[] = {&P, &Rc};
  if (h->P.pair_flag)   // K-split pair counters restart with every launch
    CUDA_OR_FAIL(h, cudaMemsetAsync(h->P.pair_flag, 0, sizeof(unsigned) * h->grid, h->stream));
  CUDA_OR_FAIL(h, cudaEventRecord(h->ev0, h->stream));
  CUDA_OR_FAIL(h, cudaLaunchCooperativeKernel(reinterpret_cast<void*>(fn), dim3(h->grid), dim3(kThreads),
                                              args, static_cast<size_t>(h->smem_bytes), h->stream));
  CUDA_OR_FAIL(h, cudaEventRecord(h->ev1, h->stream));
  h->last_launches = 1;
  h->b_valid = 0;   // a stop test may end the launch on either buffer
  return DLMPC_OK;
}

int finish_timing(dlmpc_handle* h) {
  CUDA_OR_FAIL(h, cudaEventSynchronize(h->ev1));
  CUDA_OR_FAIL(h, cudaEventElapsedTime(&h->last_ms, h->ev0, h->ev1));
  return DLMPC_OK;
}

// Checked build: a recorded out-of-range access (dlmpc_device.cuh DCHK) fails
// the call loudly; the production build has no checks.
int check_dbg(dlmpc_handle* h) {
#ifdef DLMPC_CHECKED
  int dbg[4] = {0, 0, 0, 0};
  CUDA_OR_FAIL(h, cudaMemcpy(dbg, h->P.dbg, sizeof(dbg), cudaMemcpyDeviceToHost));
  if (dbg[0] != 0) {
    long long idx = 0;
    std::memcpy(&idx, dbg + 2, sizeof(idx));
    return fail(h, DLMPC_CUDA_ERROR, "checked build: out-of-range access, check " + std::to_string(dbg[0]) +
                                         " at index " + std::to_string(idx));
  }
#else
  (void)h;
#endif
  return DLMPC_OK;
}

int read_ctl(dlmpc_handle* h, int* ctl) {
  CUDA_OR_FAIL(h, cudaMemcpyAsync(ctl, h->P.ctl, sizeof(int) * 8, cudaMemcpyDeviceToHost, h->stream));
  CUDA_OR_FAIL(h, cudaStreamSynchronize(h->stream));
  h->cur_b = ctl[4]; h->b_valid = 1;
  return check_dbg(h);
}

// The current buffer without a round trip when the host knows it (after
// asynchronous iterations), else from the device.
int current_buffer(dlmpc_handle* h, int* b) {
  if (!h->b_valid) {
    int ctl[8];
    if (int rc = read_ctl(h, ctl)) return rc;
  }
  *b = h->cur_b;
  return DLMPC_OK;
}

// Work decomposition + shared-memory plan (offsets in doubles):
//   [class operator round8(s) x ldn][K/O tile TC x ldk][Y n08 x ldy]
//   [Y split-K partials][reduction scratch][chunk metadata][Φ patch][Φ metadata]
// exact mode: [reduction scratch][per-column scratch 5*s_pad + m_pad].
//
// Patch mode assigns CTAs to runs of consecutive same-class subsystems
// (class-aware): every CTA then stages exactly one operator per launch and
// the few chain-boundary classes get CTAs of their own instead of making one
// CTA the straggler of every iteration.
int plan(dlmpc_handle* h, const dlmpc_problem* pr) {
  DevProblem& P = h->P;
  CUDA_OR_FAIL(h, cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, h->device));
  int optin = 0;
  CUDA_OR_FAIL(h, cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
  const long long limit = (optin - 1024) / 8;   // doubles
  P.off_ctab = -1;   // patch plans set it
  const int G = pr->grid_ctas > 0 ? std::min(pr->grid_ctas, h->sm_count) : h->sm_count;
  h->grid = G;
  {
    const char* e = getenv("DLMPC_G1_MROW");
    P.g1_mrow = (e && e[0] == '0') ? 0 : 1;
  }
  const char* force = getenv("DLMPC_FORCE_TWOPHASE");
  h->mode = pr->exact ? kExact : ((pr->contiguous && !(force && force[0] == '1')) ? kPatch : kTwoPhase);
  if (h->mode == kExact) {
    P.off_red = 0; P.off_meta = 32; P.off_ex = 32 + 64;
    P.opr_cap = 0;
    h->smem_bytes = (int)((P.off_ex + 5LL * pr->s_pad + pr->m_pad) * 8);
    if (h->smem_bytes > limit * 8) return fail(h, DLMPC_BAD_ARGUMENT, "support too long for the exact kernel");
  } else {
    int s8_max = 8, n08_max = 8;
    long long opr_need = 0;
    for (int k = 0; k < pr->n_classes; ++k) {
      const int s8 = (pr->class_s[k] + 7) & ~7;
      s8_max = std::max(s8_max, s8);
      n08_max = std::max(n08_max, (pr->class_n0[k] + 7) & ~7);
      opr_need = std::max<long long>(opr_need, (long long)s8 * pr->class_ldn[k]);
    }
    int tc = pr->tile_cols;
    if (h->mode == kPatch) tc = (pr->n_cols > 8LL * G) ? 16 : 8;
    if (const char* e = getenv("DLMPC_TILE_COLS")) { const int v = atoi(e); if (v == 8 || v == 16) tc = v; }
    const int tc0 = tc;   // tile width the chunks below are cut for
    // --- patch work units (class-aware CTA assignment) ----------------------
    std::vector<int> cta_ptr(G + 1, 0), u_lo, u_hi, p_lo, p_hi, u_chunk(1, 0), ch_cls, ch_c0, ch_n;
    std::vector<int> part_first, part_n;
    std::vector<int64_t> part_off;
    std::vector<int> st_unit_desc, st_chunk_desc, st_cta_gop;
    std::vector<double> st_ptab;
    std::vector<int> cta_pair;   // patch mode: per CTA -1, or partner * 2 + half (K-split pairs)
    long long part_total = 0;
    long long prows_max = 0, np_max = 0;
    if (h->mode == kPatch) {
      auto bfirst = [&](int i) { return pr->ball_idx[pr->ball_ptr[i]]; };
      auto blast = [&](int i) { return pr->ball_idx[pr->ball_ptr[i + 1] - 1]; };
      auto sub_class = [&](int i) { return pr->col_class[pr->state_start[i]]; };
      // runs of consecutive same-class subsystems
      std::vector<int> run_lo, run_hi;
      const int o_lo = P.own_sub_lo, o_hi = P.own_sub_hi;
      for (int i = o_lo; i < o_hi;) {
        int j = i + 1;
        while (j < o_hi && sub_class(j) == sub_class(i)) ++j;
        run_lo.push_back(i); run_hi.push_back(j);
        i = j;
      }
      const int nr = (int)run_lo.size();
      std::vector<int> ranges;   // CTA -> [lo, hi) pairs
      if (nr <= G) {
        std::vector<int> ctas(nr, 1);
        std::vector<long long> cols(nr);
        for (int r = 0; r < nr; ++r)
          cols[r] = pr->state_start[run_hi[r] - 1] + pr->state_count[run_hi[r] - 1] - pr->state_start[run_lo[r]];
        for (int extra = G - nr; extra > 0; --extra) {
          int best = -1; double load = -1.0;
          for (int r = 0; r < nr; ++r) {
            if (ctas[r] >= run_hi[r] - run_lo[r]) continue;   // at least one subsystem per CTA
            const double l = (double)cols[r] / ctas[r];
            if (l > load) { load = l; best = r; }
          }
          if (best < 0) break;
          ctas[best]++;
        }
        // K-split pairs (C4 large bases): a run of ONE subsystem
        // whose class operator cannot be resident in shared memory (its CTA
        // streams an unshared basis from L2 and is the straggler, e.g. d=6,
        // T=30: 235 vs 187 us) gets a second CTA; the two split the support
        // rows of GEMM 1 / GEMM 2 and exchange their partial Y. The CTAs come
        // from multi-subsystem runs that can give one up without any CTA's
        // chunk count growing. Not in stream mode (duplicated units would
        // duplicate the Φ partials).
        std::vector<char> paired(nr, 0);
        {
          const bool stream_likely = (long long)P.n_cols >= 2LL * tc * G ||
                                     (getenv("DLMPC_FORCE_STREAM") && getenv("DLMPC_FORCE_STREAM")[0] == '1');
          const char* np = getenv("DLMPC_NO_PAIRS");
          // bases of >= 1.5 MB (far beyond the operator region): measured on the
          // C4 cells at N=1000 (tools/c4_pairs_ab.py) d=6,T=30 238.6 -> 196.1
          // us/iter, d=4,T=30 84.8 -> 82.9; neutral to +1% below that size
          const bool l2_fed = opr_need * 8 > 1536LL * 1024;
          if (!stream_likely && l2_fed && !(np && np[0] == '1')) {
            std::vector<int> cand;
            for (int r = 0; r < nr; ++r)
              if (run_hi[r] - run_lo[r] == 1 && ctas[r] == 1) cand.push_back(r);
            auto work = [&](int r) {
              const int k = sub_class(run_lo[r]);
              return (long long)pr->class_s[k] * pr->class_n0[k];
            };
            std::sort(cand.begin(), cand.end(), [&](int a, int b) { return work(a) > work(b); });
            int spare = 0;
            if (!cand.empty()) {
              for (int r = 0; r < nr; ++r) {
                const int n = run_hi[r] - run_lo[r];
                if (n <= 1) continue;
                const long long spc = (cols[r] + n - 1) / n;
                auto chunks = [&](int c) { return ((n + c - 1) / c * spc + tc - 1) / tc; };
                const long long want = chunks(ctas[r]);
                int c = ctas[r];
                while (c > 1 && chunks(c - 1) == want) --c;
                spare += ctas[r] - c;
                ctas[r] = c;
              }
            }
            for (int r : cand)
              if (spare > 0) { paired[r] = 1; ctas[r] = 2; --spare; }
            for (; spare > 0; --spare) {   // the rest back to the most loaded runs
              int best = -1; double load = -1.0;
              for (int r = 0; r < nr; ++r) {
                if (paired[r] || ctas[r] >= run_hi[r] - run_lo[r]) continue;
                const double l = (double)cols[r] / ctas[r];
                if (l > load) { load = l; best = r; }
              }
              if (best < 0) break;
              ctas[best]++;
            }
          }
        }
        for (int r = 0; r < nr; ++r) {
          const int n = run_hi[r] - run_lo[r];
          if (paired[r]) {   // both CTAs run the same unit, halves 0 and 1 of the support rows
            const int q0 = (int)ranges.size() / 2;
            for (int half = 0; half < 2; ++half) {
              ranges.push_back(run_lo[r]);
              ranges.push_back(run_hi[r]);
            }
            if ((int)cta_pair.size() < q0) cta_pair.resize(q0, -1);
            cta_pair.push_back(2 * (q0 + 1) + 0);
            cta_pair.push_back(2 * q0 + 1);
            continue;
          }
          for (int q = 0; q < ctas[r]; ++q) {
            ranges.push_back(run_lo[r] + (int)((long long)n * q / ctas[r]));
            ranges.push_back(run_lo[r] + (int)((long long)n * (q + 1) / ctas[r]));
          }
        }
        if (!cta_pair.empty()) cta_pair.resize(G, -1);
      } else {
        const int n_own = o_hi - o_lo;
        for (int q = 0; q < G; ++q) {
          ranges.push_back(o_lo + (int)((long long)n_own * q / G));
          ranges.push_back(o_lo + (int)((long long)n_own * (q + 1) / G));
        }
      }
      // subsystems per full chunk when every subsystem has the same column count
      int gran = 1;
      {
        int smin = 1 << 30, smax = 0;
        for (int i = o_lo; i < o_hi; ++i) { smin = std::min(smin, pr->state_count[i]); smax = std::max(smax, pr->state_count[i]); }
        if (smin == smax && smax > 0 && tc % smax == 0) gran = tc / smax;
      }
      auto build_units = [&](long long cap_rows) {
        std::fill(cta_ptr.begin(), cta_ptr.end(), 0);
        u_lo.clear(); u_hi.clear(); p_lo.clear(); p_hi.clear(); u_chunk.assign(1, 0);
        ch_cls.clear(); ch_c0.clear(); ch_n.clear();
        prows_max = 0; np_max = 0;
        int b = 0;
        for (size_t q = 0; q + 1 < ranges.size(); q += 2, ++b) {
          const int lo = ranges[q], hi = ranges[q + 1];
          int i = lo;
          while (i < hi) {
            int plo = bfirst(i), phi = blast(i) + 1, j = i + 1;
            while (j < hi) {
              const int nlo = std::min(plo, bfirst(j)), nhi = std::max(phi, blast(j) + 1);
              if (pr->row_start[nhi] - pr->row_start[nlo] > cap_rows) break;
              plo = nlo; phi = nhi; ++j;
            }
            // cut units at whole chunks: a unit that stops before its range
            // ends keeps a multiple of `gran` subsystems (no ragged chunk)
            if (j < hi && j - i > gran) {
              j = i + (j - i) / gran * gran;
              plo = bfirst(i); phi = blast(i) + 1;
              for (int q = i + 1; q < j; ++q) { plo = std::min(plo, bfirst(q)); phi = std::max(phi, blast(q) + 1); }
            }
            u_lo.push_back(i); u_hi.push_back(j); p_lo.push_back(plo); p_hi.push_back(phi);
            prows_max = std::max<long long>(prows_max, pr->row_start[phi] - pr->row_start[plo]);
            np_max = std::max<long long>(np_max, phi - plo);
            const int c_lo = pr->state_start[i], c_hi = pr->state_start[j - 1] + pr->state_count[j - 1];
            for (int c = c_lo; c < c_hi;) {
              const int k = pr->col_class[c];
              int n = 1;
              while (c + n < c_hi && n < tc && pr->col_class[c + n] == k) ++n;
              ch_cls.push_back(k); ch_c0.push_back(c); ch_n.push_back(n);
              c += n;
            }
            u_chunk.push_back((int)ch_cls.size());
            i = j;
          }
          cta_ptr[b + 1] = (int)u_lo.size();
        }
        for (++b; b <= G; ++b) cta_ptr[b] = cta_ptr[b - 1];
      };
      build_units(4096);
      // stream mode: whole network owned, every class operator resident in
      // shared memory; the units' Φ-dot partial slots per subsystem
      // measured crossover (tools/stream_ab.py): a CTA needs >= 2 chunks for
      // the streamed chunk pipeline to pay (N=3000 at d=3: 29.8 vs 30.1 us/iter;
      // N=1e4: 94.5 vs 109.5; N=1e5: 897 vs 1170)
      const char* nostream = getenv("DLMPC_NO_STREAM");
      const char* forcestream = getenv("DLMPC_FORCE_STREAM");
      const bool stream_pays = (long long)P.n_cols >= 2LL * tc * G || (forcestream && forcestream[0] == '1');
      // (a partitioned sub-problem streams too: patch subsystems whose ball
      // holds another rank's columns -- no unit here produces their partials
      // -- recompute the full Φ every iteration, flagged in the patch table)
      if (!(nostream && nostream[0] == '1') && stream_pays) {
        // ψ/λ staging: TMA bulk copies with smem rows at the global column
        // stride when s_pad % 16 is 4 or 12 (FP64 fragment loads stay conflict
        // free; one copy per chunk and array), else 16-byte cp.async
        const bool bulk = P.s_pad % 16 == 4 || P.s_pad % 16 == 12;   // stream mode requires it
        const int ldk = bulk ? P.s_pad : ld_frag(s8_max), ldy = ld_frag(tc);
        const int sp_max = 1;   // GEMM 1 tile-parallel for every class (no partials buffer)
        // operator region sized for the classes carrying >= 5% of the columns;
        // CTAs holding a larger (rare, chain-end) class read it from L2 in a
        // separate kernel instantiation (their work is a chunk or two)
        long long opr_main = 0;
        {
          std::vector<long long> cnt(pr->n_classes, 0);
          for (int c = 0; c < P.n_cols; ++c) cnt[pr->col_class[c]]++;
          for (int k = 0; k < pr->n_classes; ++k)
            if (cnt[k] * 20 >= P.n_cols)
              opr_main = std::max<long long>(opr_main, (long long)((pr->class_s[k] + 7) & ~7) * pr->class_ldn[k]);
          const char* e = getenv("DLMPC_OPR_ALL");
          if (opr_main == 0 || (e && e[0] == '1')) opr_main = opr_need;
        }
        // λ stash stride: 2*ldl % 16 in {4, 12} keeps the register epilogue conflict free
        int ldl = P.s_pad;
        while ((2 * ldl) % 16 != 4 && (2 * ldl) % 16 != 12) ldl += 2;
        const long long fixed = ((opr_main + 1) & ~1LL) + 2LL * tc * ldk + (long long)tc * ldl + (long long)n08_max * ldy +
                                (sp_max > 1 ? (long long)sp_max * n08_max * tc : 0) + 34 + 8 * tc + 8;
        // patch rows per unit: 2048 measured 1.3% faster than 4096 at N=1e6
        // (fewer, better-balanced units once the tables fit at the first try)
        long long cap = std::min<long long>(2048, (limit - fixed) / 2);
        if (const char* e = getenv("DLMPC_STREAM_CAP")) cap = std::min<long long>(cap, atoll(e));
        long long ch_max = 0, extra = 0;
        bool ok = false;
        for (int attempt = 0; attempt < 8 && cap > 0; ++attempt) {
          build_units(cap);
          ch_max = 0;
          for (size_t u = 0; u + 1 < u_chunk.size(); ++u) ch_max = std::max<long long>(ch_max, u_chunk[u + 1] - u_chunk[u]);
          // chunk table [ch][8 ints], patch table [q][6 doubles], row map [rows] ints
          // the unit tables twice (the next unit's are prefetched), with the
          // raw ‖a‖² copy beside the reciprocals
          extra = 2 * (((((ch_max + 1) * (8 + 2 * tc) / 2 + 1) & ~1LL) + 6 * ((np_max + 1) & ~1LL) +
                        2 * ((np_max + 1) & ~1LL) + 2)) + (cap + 2) / 2 + 32;
          const long long need = fixed + 2 * ((cap + 1) & ~1LL) + extra;
          if (need <= limit) { ok = prows_max <= cap; break; }
          cap -= (need - limit + 1) / 2 + 16;
        }
        if (ok) {
          int s_max = 1;
          for (int k = 0; k < pr->n_classes; ++k) s_max = std::max(s_max, pr->class_s[k]);
          ok = bulk && ldk >= P.s_pad && ldk >= ((s_max + 3) & ~3);
          std::vector<int> unit_of(P.n_sub, -1);
          for (size_t u = 0; u < u_lo.size(); ++u)
            for (int i = u_lo[u]; i < u_hi[u]; ++i) unit_of[i] = (int)u;
          part_first.assign(P.n_sub, 0); part_n.assign(P.n_sub, 0); part_off.assign(P.n_sub, 0);
          long long tot = 0;
          // slots of subsystem i: the units owning a subsystem of its ball
          // (on a partitioned sub-problem only the owned part of the ball;
          // subsystems outside every patch get none)
          std::vector<char> in_patch(P.n_sub, 0);
          for (size_t u = 0; u < u_lo.size(); ++u)
            for (int i = p_lo[u]; i < p_hi[u]; ++i) in_patch[i] = 1;
          for (int i = 0; ok && i < P.n_sub; ++i) {
            part_off[i] = tot;
            if (!in_patch[i]) continue;
            const int f = std::max(bfirst(i), o_lo), l = std::min(blast(i), o_hi - 1);
            const int a = f <= l ? unit_of[f] : -1, z = f <= l ? unit_of[l] : -1;
            ok = a >= 0 && z >= a;
            part_first[i] = a; part_n[i] = z - a + 1;
            tot += (long long)(z - a + 1) * (pr->row_start[i + 1] - pr->row_start[i]);
          }
          part_total = tot;
          P.part_cap = std::max<long long>(1, tot);
          if (ok) {
            h->mode = kStream;
            // host-built control tables (see DevProblem)
            const int chw = 8 + 2 * tc;
            const size_t nu = u_lo.size();
            st_unit_desc.assign(nu * 16, 0);
            st_chunk_desc.assign(ch_cls.size() * chw, 0);
            st_ptab.clear();
            int pt_off = 0;
            for (size_t u = 0; u < nu; ++u) {
              const long long prow0 = pr->row_start[p_lo[u]];
              int* ud = &st_unit_desc[u * 16];
              ud[0] = u_lo[u]; ud[1] = u_hi[u]; ud[2] = p_lo[u]; ud[3] = p_hi[u];
              ud[4] = (int)(prow0 & 0xffffffffLL); ud[5] = (int)(prow0 >> 32);
              ud[6] = (int)(pr->row_start[p_hi[u]] - prow0); ud[7] = u_chunk[u]; ud[8] = u_chunk[u + 1];
              ud[9] = pt_off;
              if (u_chunk[u + 1] > u_chunk[u]) { ud[10] = ch_n[u_chunk[u]]; ud[11] = ch_c0[u_chunk[u]]; }
              if (u_chunk[u + 1] > u_chunk[u] + 1) ud[12] = ch_n[u_chunk[u] + 1];
              for (int ch = u_chunk[u]; ch < u_chunk[u + 1]; ++ch) {
                int* cd = &st_chunk_desc[(size_t)ch * chw];
                const int k = ch_cls[ch];
                cd[0] = k; cd[1] = ch_c0[ch]; cd[2] = ch_n[ch]; cd[3] = pr->class_s[k];
                cd[4] = (pr->class_n0[k] + 7) & ~7; cd[5] = pr->class_ldn[k];
                // paired: columns (2q, 2q+1) of the chunk share their support rows
                bool paired = true;
                for (int t = 0; t + 1 < ch_n[ch]; t += 2)
                  paired = paired && pr->col_rowbase[ch_c0[ch] + t] == pr->col_rowbase[ch_c0[ch] + t + 1];
                cd[6] = paired ? 1 : 0;
                for (int t = 0; t < ch_n[ch]; ++t) {
                  const int c = ch_c0[ch] + t;
                  cd[8 + t] = (int)(pr->col_rowbase[c] - prow0);
                  cd[8 + tc + t] = pr->col_vec[c];
                }
              }
              for (int i = p_lo[u]; i < p_hi[u]; ++i) {
                double e[6] = {0, 0, 0, 0, 0, 0};
                int* ei = reinterpret_cast<int*>(e);
                ei[0] = (int)(pr->row_start[i] - prow0);
                ei[1] = (int)(pr->row_start[i + 1] - pr->row_start[i]);
                ei[2] = part_n[i];
                ei[3] = (int)u - part_first[i];
                reinterpret_cast<long long*>(e)[2] = part_off[i];
                reinterpret_cast<long long*>(e)[4] = pr->row_start[i];
                ei[10] = (i >= u_lo[u] && i < u_hi[u]) ? 1 : 0;
                ei[11] = (bfirst(i) < o_lo || blast(i) >= o_hi) ? 1 : 0;   // full Φ every iteration
                st_ptab.insert(st_ptab.end(), e, e + 6);
                ++pt_off;
              }
            }
            P.ldk = ldk; P.ldy = ldy; P.split_max = sp_max;
            P.s8_max = s8_max; P.n08_max = n08_max;
            long long off = (opr_main + 1) & ~1LL;
            P.opr_cap = (int)opr_main;
            P.off_k = (int)off; off += 2LL * tc * ldk + (long long)tc * ldl;
            P.ldl = ldl;
            // producer/consumer warp specialisation needs one class per unit
            // (the operator is staged once, before the chunk pipeline)
            {
              bool one_class = true;
              for (size_t u = 0; one_class && u + 1 < u_chunk.size(); ++u)
                for (int ch = u_chunk[u] + 1; ch < u_chunk[u + 1]; ++ch)
                  if (ch_cls[ch] != ch_cls[u_chunk[u]]) { one_class = false; break; }
              const char* e = getenv("DLMPC_WARP_SPEC");
              P.warp_spec = (one_class && !(e && e[0] == '0')) ? 1 : 0;
            }
            P.off_y = (int)off; off += (long long)n08_max * ldy;
            P.off_yp = (int)off; off += sp_max > 1 ? (long long)sp_max * n08_max * tc : 0;
            P.off_red = (int)off; off += 34;   // + the CTA's unit range (2 ints, stream_iteration)
            P.off_meta = (int)off; off += 8 * tc;
            P.off_patch = (int)off; off += (cap + 1) & ~1LL;
            P.off_cpatch = (int)off; off += (cap + 1) & ~1LL;
            P.patch_cap = (int)cap;
            {   // unit tables [chunk table | patch table | 1/‖a‖² | raw ‖a‖²], two copies tab_alt apart
              const long long np_e = (np_max + 1) & ~1LL;
              const long long tab0 = off;
              P.off_chtab = (int)off; off += ((ch_max + 1) * (8 + 2 * tc) / 2 + 1) & ~1LL; P.ch_cap = (int)(ch_max + 1);
              P.off_ptab = (int)off; off += 6 * np_e; P.np_cap = (int)np_e;
              P.off_pada = (int)off; off += 2 * np_e + 2;
              P.tab_alt = (int)(off - tab0);
              off += P.tab_alt;
            }
            P.off_rowq = (int)off; off += (cap + 2) / 2;
            off = (off + 1) & ~1LL;
            P.off_udesc = (int)off; off += 16;
            P.off_bar = (int)off; off += 4;
            // CTAs with a class operator larger than the region
            st_cta_gop.assign(G, 0);
            bool any_gop = false;
            for (int q = 0; q < G; ++q)
              for (int u = cta_ptr[q]; u < cta_ptr[q + 1]; ++u)
                for (int ch = u_chunk[u]; ch < u_chunk[u + 1]; ++ch) {
                  const int k = ch_cls[ch];
                  if ((long long)((pr->class_s[k] + 7) & ~7) * pr->class_ldn[k] > opr_main) {
                    st_cta_gop[q] = 1; any_gop = true;
                  }
                }
            if (!any_gop) st_cta_gop.clear();
            P.cache_phi = 0; P.stash_bufs = 0; P.off_stash = (int)off; P.off_phimeta = (int)off;
            P.off_ex = (int)off;
            h->smem_bytes = (int)(off * 8);
            P.tile_cols = tc;
          } else {
            build_units(4096);
          }
        } else {
          build_units(4096);
        }
      }
      h->n_units = (int)u_lo.size();
      // patch mode: trailing CTAs without a unit would only join the barriers
      // (C2: 100 units on 148 SMs); the launch leaves them out (tools/grid_ab.py,
      // C2 closed loops: 14.62 -> 14.74 M subsystem-iters/s, bitwise the same)
      const char* keep = getenv("DLMPC_KEEP_IDLE_CTAS");
      if (h->mode == kPatch && cta_pair.empty() && !(keep && keep[0] == '1')) {
        int gl = G;
        while (gl > 1 && cta_ptr[gl - 1] == cta_ptr[gl]) --gl;
        cta_ptr.resize(gl + 1);
        h->grid = gl;
      }
    }
    bool one_unit = true;
    for (int q = 0; q < h->grid; ++q) one_unit = one_unit && (cta_ptr[q + 1] - cta_ptr[q] <= 1);
    bool rb_off = false;   // the register-blocked GEMV pair was planned but did not fit
    for (; h->mode != kStream;) {
      const int ldk = ld_frag(s8_max), ldy = ld_frag(tc);
      // 16-column tiles run GEMM 1 tile-parallel for every class: no split-K
      // partials (measured on the C4 cells at N=1000: 8-16% faster than
      // split-K for the classes with < 12 tiles)
      int split_max = 1;
      const char* esk = getenv("DLMPC_SPLITK_ALL");
      const bool no_split = tc == 16 && !(esk && esk[0] == '1');
      for (int k = 0; k < pr->n_classes; ++k) {
        if (no_split) continue;
        const int groups1 = (((pr->class_n0[k] + 7) / 8) + kMG1 - 1) / kMG1;
        int sp = 1;
        while (groups1 * sp * 2 <= kWarps && sp < 4) sp <<= 1;
        split_max = std::max(split_max, sp);
      }
      const long long meta_phi = np_max * pr->d_pad * 2 + np_max + 3 * prows_max + (np_max + 1) / 2 + np_max + 8 + 2;
      // patch mode, TC 8: room for the register-blocked GEMV pair (thread-major
      // operator, 16 warps' Y partials) when the classes fit its blocking
      // (every chunk <= 2 columns; measured on C2: 8.4 vs 9.6 us per ADMM
      // iteration against the DFMA GEMV + DMMA GEMM pair). That path needs no K tile and stages
      // two columns, which keeps the plan inside the 196 KB carveout (a larger
      // one leaves too little L1 for the kernel's table loads: -25% measured).
      bool rb = h->mode == kPatch && tc == 8 && !rb_off && cta_pair.empty();
      const int rb_al = RB_AL_MAX;
      for (int n : ch_n) rb = rb && n <= 2;
      for (int k = 0; k < pr->n_classes && rb; ++k) {
        const int s8 = (pr->class_s[k] + 7) & ~7, n08 = (pr->class_n0[k] + 7) & ~7;
        rb = s8 <= 32 * RB_PL && n08 <= 16 * RB_AL_MAX;
      }
      if (const char* e = getenv("DLMPC_RB_GEMV")) rb = rb && e[0] != '0';
      const long long rb_opr = rb ? (long long)RB_PL * rb_al * kThreads : 0;
      const long long rb_part = rb ? 2LL * 16 * rb_al * kWarps : 0;
      const int kt_cols = rb ? 0 : tc, st_cols = rb ? 2 : tc;
      auto part = [&](int sp) { return std::max<long long>(sp > 1 ? (long long)sp * n08_max * tc : 0, rb_part); };
      // partial Φ cache (no per-row scales and bounds; phi_rows_pcached)
      const long long meta_part = meta_phi - 3 * prows_max;
      auto total = [&](long long opr, int sp, long long meta) {
        return opr + (long long)kt_cols * ldk + (long long)n08_max * ldy + part(sp)
               + 34 + 4 * tc + prows_max + meta + 4;
      };
      while (split_max > 1 && total(0, split_max, 0) > limit) split_max >>= 1;
      if (total(0, split_max, 0) > limit) {
        if (tc == 16) { tc = 8; continue; }
        return fail(h, DLMPC_BAD_ARGUMENT, "column tile does not fit in shared memory");
      }
      long long opr = total(opr_need, split_max, 0) <= limit ? opr_need : 0;
      if (rb && opr > 0 && opr < rb_opr && total(rb_opr, split_max, 0) <= limit) opr = rb_opr;
      const bool cache = h->mode == kPatch && one_unit && total(opr, split_max, meta_phi) <= limit;
      // where the full cache does not fit (the largest C4 cells), the partial
      // one: d=6, T=30 at N=1000 (measured in DESIGN §5)
      // (DLMPC_PARTIAL_PHI=0 disables it, =2 takes it in place of the full
      // cache -- tests: the partial-cache kernels on small problems)
      const char* epc = getenv("DLMPC_PARTIAL_PHI");
      const bool force_pc = epc && epc[0] == '2' && !rb;
      const bool pcache = (!cache || force_pc) && !rb && h->mode == kPatch && one_unit && !(epc && epc[0] == '0') &&
                          total(opr, split_max, meta_part) <= limit;
      const long long meta_sz = pcache ? meta_part : (cache ? meta_phi : 0);
      // cp.async staging buffers for chunk ψ,λ (patch mode): 2 if they fit, else 1, else none
      const long long stash_one = 2LL * st_cols * ldk;
      int stash_bufs = 0;
      if (h->mode == kPatch) {
        // staging buffers within ~200 KB of shared memory in all: a larger
        // carveout leaves too little L1 for the kernel's table loads (d=3,
        // T=10 at N=1000: 1.4% slower with a buffer that took it to 208 KB)
        const long long base = total(opr, split_max, meta_sz);
        const char* esl = getenv("DLMPC_STASH_LIM_KB");   // A/B of the carveout rule
        const long long lim_kb = esl ? atoll(esl) : 200;
        const long long lim = std::min<long long>(limit, (no_split ? lim_kb * 1024 : 1LL << 40) / 8);
        stash_bufs = base + 2 * stash_one + 2 <= lim ? 2 : (base + stash_one + 2 <= lim ? 1 : 0);
      }
      if (rb && (stash_bufs == 0 || opr < rb_opr)) { rb_off = true; continue; }
      long long off = (opr + 1) & ~1LL;
      P.opr_cap = (int)opr;
      P.s8_max = s8_max; P.n08_max = n08_max; P.ldk = ldk; P.ldy = ldy; P.split_max = split_max;
      P.off_k = (int)off; off += (long long)kt_cols * ldk;
      P.off_y = (int)off; off += (long long)n08_max * ldy;
      P.off_yp = (int)off; off += part(split_max);
      {   // GEMV partials of small chunks share the split-K partials region
        const char* e = getenv("DLMPC_SMALL_GEMV");
        P.small_gemv = (split_max > 1 && (long long)split_max * tc >= 10 && !(e && e[0] == '0')) ? 1 : 0;
      }
      P.off_red = (int)off; off += 34;   // + the CTA's unit range (2 ints, patch_iteration)
      P.off_meta = (int)off; off += 4 * tc;
      P.off_patch = (int)off; off += (prows_max + 1) & ~1LL;
      P.patch_cap = (int)prows_max;
      P.off_phimeta = (int)off; off += meta_sz;
      P.off_ublk = (int)(off - (np_max + 8 + 2));   // tail of the Φ metadata block (cache only)
      P.cache_phi = pcache ? 2 : (cache ? 1 : 0);
      off = (off + 1) & ~1LL;   // 16-byte alignment for cp.async
      P.off_stash = (int)off; off += stash_bufs * stash_one;
      P.stash_bufs = stash_bufs;
      P.stash_cols = st_cols;
      P.rb_gemv = rb ? 1 : 0;
      // patch plans (the DMMA chunks read them; the two-phase kernel shares
      // this planner but not the table): class sizes in shared memory
      // (class_dims), 3 doubles per class
      if (h->mode == kPatch && !rb && pr->n_classes <= 256 && off + 3LL * pr->n_classes <= limit) {
        P.off_ctab = (int)off;
        off += 3LL * pr->n_classes;
      }
      P.off_ex = (int)off;
      h->smem_bytes = (int)(off * 8);
      P.tile_cols = tc;
      break;
    }
    // chunks were cut for the initial tile width; re-cut if it shrank
    if ((h->mode == kPatch || h->mode == kStream) && P.tile_cols != tc0) {
      std::vector<int> nc_cls, nc_c0, nc_n, nu(1, 0);
      for (size_t u = 0; u + 1 < u_chunk.size(); ++u) {
        for (int ch = u_chunk[u]; ch < u_chunk[u + 1]; ++ch)
          for (int q = 0; q < ch_n[ch]; q += P.tile_cols) {
            nc_cls.push_back(ch_cls[ch]); nc_c0.push_back(ch_c0[ch] + q);
            nc_n.push_back(std::min(P.tile_cols, ch_n[ch] - q));
          }
        nu.push_back((int)nc_cls.size());
      }
      ch_cls.swap(nc_cls); ch_c0.swap(nc_c0); ch_n.swap(nc_n); u_chunk.swap(nu);
    }
    // closed loops with the Φ cache of one unit per CTA: the MPC-step
    // transition inside each CTA (fused_transition) over its window, from
    // step-invariant tables (layout: FuseTab in dlmpc_device.cuh)
    std::vector<int> ft_iptr(1, 0), ft_int, ft_dptr(1, 0);
    std::vector<double> ft_dbl;
    P.fuse_steps = 0;
    {
      // on by default for the register-blocked GEMV plans (C2-sized networks:
      // measured +3.1% on the C2 closed loops; N=1000 d=3 T=10 even, N=300
      // d=2 T=5 -2%: the fused kernel of the DMMA plans spills);
      // DLMPC_FUSE_STEPS=1 forces it for any eligible plan, =0 disables it
      const char* e = getenv("DLMPC_FUSE_STEPS");
      const bool force = e && e[0] == '1', off_env = e && e[0] == '0';
      const bool want = h->mode == kPatch && P.cache_phi == 1 && cta_pair.empty() && P.own_sub_lo == 0 &&
                        P.own_sub_hi == pr->n_sub && pr->a_ptr && pr->b_ptr && !off_env &&
                        (P.rb_gemv || force) &&
                        (long long)pr->n_cols * pr->s_pad < INT_MAX && pr->row_start[pr->n_sub] < INT_MAX &&
                        pr->n_cols < (1 << 29) && pr->n_inputs < (1 << 29);
      if (want) {
        long long imax = 0, dmax = 0, w2max = 0, wmax = 0, umax = 0;
        std::vector<int> wl, ul, w2, blob;
        std::vector<double> dbl;
        auto idx = [](const std::vector<int>& v, int x) { return (int)(std::lower_bound(v.begin(), v.end(), x) - v.begin()); };
        for (size_t u = 0; u < u_lo.size(); ++u) {
          const int ulo = u_lo[u], uhi = u_hi[u];
          wl.clear(); ul.clear(); w2.clear(); blob.assign(FuseTab::kHeader, 0); dbl.clear();
          for (int i = p_lo[u]; i < p_hi[u]; ++i)
            for (int k = 0; k < pr->supp_len[i]; ++k) wl.push_back(pr->supp_col[(size_t)i * pr->d_pad + k]);
          std::sort(wl.begin(), wl.end());
          wl.erase(std::unique(wl.begin(), wl.end()), wl.end());
          for (int r : wl) {
            for (int64_t q = pr->b_ptr[r]; q < pr->b_ptr[r + 1]; ++q) ul.push_back(pr->b_idx[q]);
            for (int64_t q = pr->a_ptr[r]; q < pr->a_ptr[r + 1]; ++q) w2.push_back(pr->a_idx[q]);
          }
          for (int k = 0; k < pr->n_inputs; ++k)
            if (pr->input_owner[k] >= ulo && pr->input_owner[k] < uhi) ul.push_back(k);
          for (auto* v : {&ul, &w2}) { std::sort(v->begin(), v->end()); v->erase(std::unique(v->begin(), v->end()), v->end()); }
          const int nw = (int)wl.size(), nu = (int)ul.size(), nw2 = (int)w2.size();
          blob[FuseTab::kNw] = nw; blob[FuseTab::kNu] = nu; blob[FuseTab::kNw2] = nw2;
          blob[FuseTab::kWcol] = (int)blob.size();      // window states: r * 2 + own
          for (int r : wl) blob.push_back(r * 2 + (pr->col_owner[r] >= ulo && pr->col_owner[r] < uhi ? 1 : 0));
          blob[FuseTab::kW2] = (int)blob.size();        // states whose x the window's A rows read
          blob.insert(blob.end(), w2.begin(), w2.end());
          blob[FuseTab::kSupp] = (int)blob.size();      // per patch-subsystem support slot: window index
          for (int i = p_lo[u]; i < p_hi[u]; ++i)
            for (int k = 0; k < pr->d_pad; ++k)
              blob.push_back(k < pr->supp_len[i] ? idx(wl, pr->supp_col[(size_t)i * pr->d_pad + k]) : 0);
          blob[FuseTab::kMx] = (int)blob.size();        // the single chunk's columns: window index
          if (u_chunk[u + 1] - u_chunk[u] == 1)
            for (int t = 0; t < ch_n[u_chunk[u]]; ++t) blob.push_back(idx(wl, ch_c0[u_chunk[u]] + t));
          blob[FuseTab::kUhead] = (int)blob.size();     // per input: k * 2 + own, s_row index, support length, entry offset
          const int uh = (int)blob.size();
          blob.resize(blob.size() + 4 * (size_t)nu);
          blob[FuseTab::kUent] = (int)blob.size();      // per support slot of an input's row: ψ/λ position, column
          for (int j = 0; j < nu; ++j) {
            const int k = ul[j], i = pr->input_owner[k], l = pr->input_local[k];
            blob[uh + 4 * j] = k * 2 + (i >= ulo && i < uhi ? 1 : 0);
            blob[uh + 4 * j + 1] = (int)(pr->row_start[i] + l);
            blob[uh + 4 * j + 2] = pr->supp_len[i];
            blob[uh + 4 * j + 3] = (int)blob.size() - blob[FuseTab::kUent];
            for (int q = 0; q < pr->supp_len[i]; ++q) {
              const size_t e2 = (size_t)i * pr->d_pad + q;
              blob.push_back((int)((long long)pr->supp_col[e2] * pr->s_pad + pr->supp_off[e2] + l));
              blob.push_back(pr->supp_col[e2]);
            }
          }
          blob[FuseTab::kAoff] = (int)blob.size();      // per window state: A entries [aoff, aoff+1), B entries likewise
          const int ao = (int)blob.size();
          blob.resize(blob.size() + 2 * ((size_t)nw + 1));
          blob[FuseTab::kAent] = (int)blob.size();      // A entry: index into W2 (values: doubles [0, na))
          int na = 0;
          for (int j = 0; j < nw; ++j) {
            blob[ao + j] = na;
            for (int64_t q = pr->a_ptr[wl[j]]; q < pr->a_ptr[wl[j] + 1]; ++q, ++na) {
              blob.push_back(idx(w2, pr->a_idx[q])); dbl.push_back(pr->a_val[q]);
            }
          }
          blob[ao + nw] = na;
          blob[FuseTab::kBent] = (int)blob.size();      // B entry: index into U (values: doubles [na, na+nb))
          int nb = 0;
          for (int j = 0; j < nw; ++j) {
            blob[ao + nw + 1 + j] = nb;
            for (int64_t q = pr->b_ptr[wl[j]]; q < pr->b_ptr[wl[j] + 1]; ++q, ++nb) {
              blob.push_back(idx(ul, pr->b_idx[q])); dbl.push_back(pr->b_val[q]);
            }
          }
          blob[ao + 2 * nw + 1] = nb;
          blob[FuseTab::kNa] = na;
          blob[FuseTab::kNint] = (int)blob.size();
          ft_int.insert(ft_int.end(), blob.begin(), blob.end());
          ft_dbl.insert(ft_dbl.end(), dbl.begin(), dbl.end());
          ft_iptr.push_back((int)ft_int.size()); ft_dptr.push_back((int)ft_dbl.size());
          imax = std::max<long long>(imax, (long long)blob.size());
          dmax = std::max<long long>(dmax, (long long)dbl.size());
          w2max = std::max<long long>(w2max, nw2); wmax = std::max<long long>(wmax, nw); umax = std::max<long long>(umax, nu);
        }
        // shared memory: table doubles | x of W2 | x+ of W | u of U | row weights of the patch | table ints
        const long long need = dmax + w2max + wmax + umax + prows_max + (imax + 1) / 2 + 2;
        const long long off = (P.off_ex + 1) & ~1LL;
        if (off + need <= limit) {
          P.fuse_steps = 1;
          P.off_fw = (int)off;
          P.ft_dcap = (int)dmax; P.ft_w2cap = (int)w2max; P.ft_wcap = (int)wmax; P.ft_ucap = (int)umax;
          P.off_ex = (int)(off + need);
          h->smem_bytes = (int)(P.off_ex * 8);
        }
      }
    }
    // patch mode, C2-sized networks: the register-blocked GEMV pair when every
    // chunk has <= 2 columns and every class operator fits its thread blocking
    // (measured on C2: GEMV pair 1.3 us vs 2.1 us for the DFMA GEMV + DMMA GEMM)
    if (getenv("DLMPC_DEBUG_PLAN"))
      fprintf(stderr, "plan: mode %d tc %d stash %d opr %d split %d n08 %d ldy %d rb %d chunks %zu cache %d fuse %d smem %d\n", h->mode,
              P.tile_cols, P.stash_bufs, P.opr_cap, P.split_max, P.n08_max, P.ldy, P.rb_gemv, ch_n.size(), P.cache_phi, P.fuse_steps, h->smem_bytes);
    if (h->mode == kPatch || h->mode == kStream) {
      int rc;
      if ((rc = upload(h, cta_ptr.data(), cta_ptr.size(), &P.cta_unit_ptr)) ||
          (rc = upload(h, u_lo.data(), u_lo.size(), &P.unit_sub_lo)) ||
          (rc = upload(h, u_hi.data(), u_hi.size(), &P.unit_sub_hi)) ||
          (rc = upload(h, p_lo.data(), p_lo.size(), &P.unit_patch_lo)) ||
          (rc = upload(h, p_hi.data(), p_hi.size(), &P.unit_patch_hi)) ||
          (rc = upload(h, u_chunk.data(), u_chunk.size(), &P.unit_chunk_ptr)) ||
          (rc = upload(h, ch_cls.data(), ch_cls.size(), &P.chunk_class)) ||
          (rc = upload(h, ch_c0.data(), ch_c0.size(), &P.chunk_col0)) ||
          (rc = upload(h, ch_n.data(), ch_n.size(), &P.chunk_n)))
        return rc;
      if (h->mode == kPatch && (rc = alloc(h, 1, &P.gbar))) return rc;
      if (P.fuse_steps) {
        if (ft_dbl.empty()) ft_dbl.push_back(0.0);
        if ((rc = upload(h, ft_iptr.data(), ft_iptr.size(), &P.ft_iptr)) ||
            (rc = upload(h, ft_int.data(), ft_int.size(), &P.ft_int)) ||
            (rc = upload(h, ft_dptr.data(), ft_dptr.size(), &P.ft_dptr)) ||
            (rc = upload(h, ft_dbl.data(), ft_dbl.size(), &P.ft_dbl)))
          return rc;
      }
      if (h->mode == kPatch && !cta_pair.empty()) {
        if ((rc = upload(h, cta_pair.data(), cta_pair.size(), &P.cta_pair)) ||
            (rc = alloc(h, (size_t)G, &P.pair_flag)) ||
            (rc = alloc(h, (size_t)2 * G * P.n08_max * P.tile_cols, &P.ypair)))
          return rc;
        if (getenv("DLMPC_DEBUG_PLAN")) {
          int np = 0;
          for (int v : cta_pair) np += v >= 0;
          fprintf(stderr, "plan: %d CTAs in K-split pairs\n", np);
        }
      }
      if (h->mode == kStream) {
        if ((rc = upload(h, st_cta_gop.data(), st_cta_gop.size(), &P.cta_gop)) ||
            (rc = upload(h, st_unit_desc.data(), st_unit_desc.size(), &P.unit_desc)) ||
            (rc = upload(h, st_chunk_desc.data(), st_chunk_desc.size(), &P.chunk_desc)) ||
            (rc = upload(h, st_ptab.data(), st_ptab.size(), &P.unit_ptab)) ||
            (rc = upload(h, part_first.data(), part_first.size(), &P.part_first)) ||
            (rc = upload(h, part_n.data(), part_n.size(), &P.part_n)) ||
            (rc = upload(h, part_off.data(), part_off.size(), &P.part_off)))
          return rc;
        for (int q = 0; q < 2; ++q) {
          void* ptr = nullptr;
          CUDA_OR_FAIL(h, cudaMalloc(&ptr, sizeof(double) * std::max<long long>(1, part_total)));
          h->allocs.push_back(ptr);
          P.part_buf[q] = static_cast<double*>(ptr);
        }
        {
          void* ptr = nullptr;
          CUDA_OR_FAIL(h, cudaMalloc(&ptr, sizeof(double) * std::max<long long>(1, P.n_rows)));
          h->allocs.push_back(ptr);
          P.row_invden = static_cast<double*>(ptr);
        }
      }
    }
  }
  P.smem_doubles = h->smem_bytes / 8;
  P.vbase = 0;          // the whole launch (dlmpc_multi_solve shifts it per rank)
  P.vgrid = h->grid;
  KernelFn fn = pick_kernel(h->mode, P.tile_cols, P.rb_gemv);
  CUDA_OR_FAIL(h, cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, h->smem_bytes));
  int per_sm = 0;
  CUDA_OR_FAIL(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, reinterpret_cast<const void*>(fn),
                                                                kThreads, h->smem_bytes));
  if (per_sm < 1) return fail(h, DLMPC_CUDA_ERROR, "persistent kernel cannot be resident");
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
  if (pr->tile_cols != 8 && pr->tile_cols != 16)
    return fail(nullptr, DLMPC_BAD_ARGUMENT, "tile_cols must be 8 or 16");
  auto* h = new dlmpc_handle();
  h->device = device;
  if (cudaSetDevice(device) != cudaSuccess) { delete h; return fail(nullptr, DLMPC_CUDA_ERROR, "cudaSetDevice failed"); }
  int rc = DLMPC_OK;
#define UP(field, n) do { if ((rc = upload(h, pr->field, (size_t)(n), &P.field)) != DLMPC_OK) goto bad; } while (0)
  {
    DevProblem& P = h->P;
    P.n_sub = pr->n_sub; P.n_rows = pr->n_rows; P.n_cols = pr->n_cols; P.n_inputs = pr->n_inputs;
    P.own_sub_lo = pr->own_sub_lo; P.own_sub_hi = pr->own_sub_hi;
    P.own_col_lo = pr->own_col_lo; P.own_col_hi = pr->own_col_hi;
    if (P.own_sub_hi <= P.own_sub_lo) { P.own_sub_lo = 0; P.own_sub_hi = pr->n_sub; P.own_col_lo = 0; P.own_col_hi = pr->n_cols; }
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
    P.d_pad = pr->d_pad;
    UP(supp_col, (size_t)pr->n_sub * pr->d_pad); UP(supp_off, (size_t)pr->n_sub * pr->d_pad); UP(supp_len, pr->n_sub);
    UP(row_w, pr->n_rows); UP(row_lo, pr->n_rows); UP(row_hi, pr->n_rows);
    UP(col_owner, pr->n_cols); UP(col_len, pr->n_cols); UP(col_class, pr->n_cols); UP(col_vec, pr->n_cols);
    if (!pr->contiguous) UP(col_irow, (size_t)pr->n_sub * pr->s_pad);
    UP(col_rowbase, pr->n_cols);
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
    if (pr->g0_pool && pr->perm_pool && pr->col_pin) {
      UP(class_ntouch, pr->n_classes); UP(class_g0_off, pr->n_classes + 1);
      UP(g0_pool, pr->class_g0_off[pr->n_classes]); UP(class_perm_off, pr->n_classes + 1);
      UP(perm_pool, pr->class_perm_off[pr->n_classes]); UP(col_pin, pr->n_cols);
    }
    const size_t ncell = (size_t)pr->n_cols * pr->s_pad;
    for (int q = 0; q < 2; ++q) {
      if ((rc = alloc(h, ncell, &P.psi[q])) != DLMPC_OK) goto bad;
      if ((rc = alloc(h, ncell, &P.lam[q])) != DLMPC_OK) goto bad;
      if ((rc = alloc(h, (size_t)pr->n_cols, &P.x[q])) != DLMPC_OK) goto bad;
    }
    if ((rc = alloc(h, (size_t)pr->n_rows, &P.s_row)) != DLMPC_OK) goto bad;
    if ((rc = alloc(h, (size_t)pr->n_sub + 2, &P.ada)) != DLMPC_OK) goto bad;
    if ((rc = alloc(h, (size_t)(pr->n_inputs ? pr->n_inputs : 1), &P.u)) != DLMPC_OK) goto bad;
    if ((rc = alloc(h, 8, &P.ctl)) != DLMPC_OK) goto bad;
    if ((rc = alloc(h, 4, &P.dbg)) != DLMPC_OK) goto bad;
    if ((rc = alloc(h, ncell, &h->d_scratch)) != DLMPC_OK) goto bad;
    if ((rc = alloc(h, 16 * 1024, &P.phase_ns)) != DLMPC_OK) goto bad;
    if (cudaMemset(P.ctl + 2, 0x7f, sizeof(int) * 2) != cudaSuccess) { rc = fail(h, DLMPC_CUDA_ERROR, "memset"); goto bad; }

    if ((rc = plan(h, pr)) != DLMPC_OK) goto bad;
    if (cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&h->ev0) != cudaSuccess || cudaEventCreate(&h->ev1) != cudaSuccess) {
      rc = fail(h, DLMPC_CUDA_ERROR, "stream/event creation failed"); goto bad;
    }
    h->stream = h->own_stream;
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
  if (h->d_scratch2) cudaFree(h->d_scratch2);
  if (h->d_audit) cudaFree(h->d_audit);
  if (h->d_send_cells) cudaFree(h->d_send_cells);
  if (h->d_recv_cells) cudaFree(h->d_recv_cells);
  if (h->d_halo) cudaFree(h->d_halo);
  if (h->P.resid) cudaFree(h->P.resid);
  if (h->h_stage) cudaFreeHost(h->h_stage);
  if (h->d_stage) cudaFree(h->d_stage);
  if (h->d_step_iters) cudaFree(h->d_step_iters);
  if (h->d_states) cudaFree(h->d_states);
  if (h->d_inputs) cudaFree(h->d_inputs);
  if (h->ev0) cudaEventDestroy(h->ev0);
  if (h->ev1) cudaEventDestroy(h->ev1);
  if (h->own_stream) cudaStreamDestroy(h->own_stream);
  delete h;
}

int dlmpc_set_x(dlmpc_handle* h, const double* x, int64_t* bad_row) {
  if (h) h->it_cont = 0;
  if (!h || !x) return fail(h, DLMPC_BAD_ARGUMENT, "null argument");
  cudaSetDevice(h->device);
  CUDA_OR_FAIL(h, cudaMemcpyAsync(h->P.x[0], x, sizeof(double) * h->P.n_cols, cudaMemcpyHostToDevice, h->stream));
  CUDA_OR_FAIL(h, cudaMemsetAsync(h->P.ctl + 2, 0x7f, sizeof(int), h->stream));
  set_x_kernel<<<std::max(1, std::min(h->sm_count * 8, (h->P.n_sub + 7) / 8)), 256, 0, h->stream>>>(h->P);   // a warp per subsystem
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
  R.it_base = h->it_cont;
  if (int rc = launch(h, R)) return rc;
  if (int rc = finish_timing(h)) return rc;
  CUDA_OR_FAIL(h, cudaGetLastError());
  int ctl[8];
  if (int rc = read_ctl(h, ctl)) return rc;
  int n = 0;
  CUDA_OR_FAIL(h, cudaMemcpy(&n, h->d_step_iters, sizeof(int), cudaMemcpyDeviceToHost));
  if (ctl[0] == DLMPC_NOT_CONVERGED) n = ctl[5];
  h->it_cont += n;
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

namespace {
// The closed-loop launch with x0 already in P.x[0].
int launch_closed_loop(dlmpc_handle* h, int t_sim, int warm_start, int cold_start, int max_iters, double eps_pri,
                       double eps_dual, double* states_dev, double* inputs_dev, int* step_iters_dev,
                       int* status_dev) {
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
}  // namespace

int dlmpc_simulate_device(dlmpc_handle* h, const double* x0_dev, int t_sim, int warm_start, int cold_start,
                          int max_iters, double eps_pri, double eps_dual, double* states_dev,
                          double* inputs_dev, int* step_iters_dev, int* status_dev) {
  if (h) h->it_cont = 0;
  if (!h || !x0_dev || t_sim < 1 || max_iters < 1) return fail(h, DLMPC_BAD_ARGUMENT, "bad argument");
  cudaSetDevice(h->device);
  if (int rc = ensure_run_buffers(h, max_iters, t_sim)) return rc;
  CUDA_OR_FAIL(h, cudaMemcpyAsync(h->P.x[0], x0_dev, sizeof(double) * h->P.n_cols, cudaMemcpyDeviceToDevice, h->stream));
  return launch_closed_loop(h, t_sim, warm_start, cold_start, max_iters, eps_pri, eps_dual, states_dev, inputs_dev,
                            step_iters_dev, status_dev);
}

int dlmpc_simulate(dlmpc_handle* h, const double* x0, int t_sim, int warm_start, int cold_start,
                   int max_iters, double eps_pri, double eps_dual, double* states, double* inputs,
                   int* step_iters, int* fail_step, int64_t* bad_row, int* fail_iters, double* fail_hist) {
  if (h) h->it_cont = 0;
  if (!h || !x0 || t_sim < 1 || max_iters < 1) return fail(h, DLMPC_BAD_ARGUMENT, "bad argument");
  cudaSetDevice(h->device);
  if (int rc = ensure_run_buffers(h, max_iters, t_sim)) return rc;
  // pinned staging: x0 in, then status, iteration counts, trajectory out in
  // one batch of async copies and a single stream synchronisation
  const size_t nc = (size_t)h->P.n_cols, ni = (size_t)h->P.n_inputs;
  const size_t o_ctl = nc * 8, o_it = o_ctl + 64, o_st = o_it + (((size_t)t_sim * 4 + 15) & ~(size_t)15);
  const size_t o_in = o_st + (size_t)(t_sim + 1) * nc * 8, need = o_in + (size_t)t_sim * ni * 8 + 8;
  if (need > h->stage_cap) {
    if (h->h_stage) cudaFreeHost(h->h_stage);
    if (h->d_stage) cudaFree(h->d_stage);
    h->h_stage = nullptr; h->d_stage = nullptr; h->stage_cap = 0;
    CUDA_OR_FAIL(h, cudaMallocHost(reinterpret_cast<void**>(&h->h_stage), need));
    CUDA_OR_FAIL(h, cudaMalloc(reinterpret_cast<void**>(&h->d_stage), need));
    h->stage_cap = need;
  }
  // the kernel writes iteration counts, states and inputs straight into the
  // device mirror of the staging layout and the status joins them with one
  // small D2D copy, so the results come back in a single D2H copy
  char* hs = h->h_stage;
  char* ds = h->d_stage;
  std::memcpy(hs, x0, nc * 8);
  CUDA_OR_FAIL(h, cudaMemcpyAsync(h->P.x[0], hs, nc * 8, cudaMemcpyHostToDevice, h->stream));
  if (int rc = launch_closed_loop(h, t_sim, warm_start, cold_start, max_iters, eps_pri, eps_dual,
                                  reinterpret_cast<double*>(ds + o_st), reinterpret_cast<double*>(ds + o_in),
                                  reinterpret_cast<int*>(ds + o_it), reinterpret_cast<int*>(ds + o_ctl))) return rc;
  CUDA_OR_FAIL(h, cudaMemcpyAsync(hs + o_ctl, ds + o_ctl, need - o_ctl, cudaMemcpyDeviceToHost, h->stream));
  CUDA_OR_FAIL(h, cudaStreamSynchronize(h->stream));
  CUDA_OR_FAIL(h, cudaEventElapsedTime(&h->last_ms, h->ev0, h->ev1));
  int ctl[8];
  std::memcpy(ctl, hs + o_ctl, sizeof(ctl));
  int done = t_sim;
  if (ctl[0] != DLMPC_OK) done = ctl[1];
  if (fail_step) *fail_step = ctl[0] == DLMPC_OK ? -1 : ctl[1];
  if (bad_row) *bad_row = ctl[0] == DLMPC_ROW_INFEASIBLE ? ctl[2 + (ctl[1] & 1)] : -1;
  if (fail_iters) *fail_iters = ctl[0] == DLMPC_NOT_CONVERGED ? ctl[5] : 0;
  if (states) {   // row 0 is x0 (the kernel stores it only once step 0 has been solved)
    std::memcpy(states, x0, nc * 8);
    if (done > 0) std::memcpy(states + nc, hs + o_st + nc * 8, (size_t)done * nc * 8);
  }
  if (inputs && done > 0 && ni) std::memcpy(inputs, hs + o_in, (size_t)done * ni * 8);
  if (step_iters && done > 0) std::memcpy(step_iters, hs + o_it, sizeof(int) * done);
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
  if (h) h->it_cont = 0;
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

int dlmpc_get_cols(dlmpc_handle* h, int which, int c0, int n, double* dst) {
  if (!h || !dst || c0 < 0 || n < 0 || c0 + n > h->P.n_cols) return fail(h, DLMPC_BAD_ARGUMENT, "bad column range");
  cudaSetDevice(h->device);
  int ctl[8];
  if (int rc = read_ctl(h, ctl)) return rc;
  const int b = ctl[4];
  const double* src = which == DLMPC_PSI ? h->P.psi[b] : which == DLMPC_LAM ? h->P.lam[b] : nullptr;
  if (!src) return fail(h, DLMPC_BAD_ARGUMENT, "only PSI / LAM column ranges");
  CUDA_OR_FAIL(h, cudaMemcpyAsync(dst, src + (size_t)c0 * h->P.s_pad, sizeof(double) * (size_t)n * h->P.s_pad,
                                  cudaMemcpyDefault, h->stream));
  CUDA_OR_FAIL(h, cudaStreamSynchronize(h->stream));
  return DLMPC_OK;
}

int dlmpc_put_cols(dlmpc_handle* h, int which, int c0, int n, const double* src) {
  if (h) h->it_cont = 0;
  if (!h || !src || c0 < 0 || n < 0 || c0 + n > h->P.n_cols) return fail(h, DLMPC_BAD_ARGUMENT, "bad column range");
  cudaSetDevice(h->device);
  int ctl[8];
  if (int rc = read_ctl(h, ctl)) return rc;
  const int b = ctl[4];
  double* dst = which == DLMPC_PSI ? h->P.psi[b] : which == DLMPC_LAM ? h->P.lam[b] : nullptr;
  if (!dst) return fail(h, DLMPC_BAD_ARGUMENT, "only PSI / LAM column ranges");
  CUDA_OR_FAIL(h, cudaMemcpyAsync(dst + (size_t)c0 * h->P.s_pad, src, sizeof(double) * (size_t)n * h->P.s_pad,
                                  cudaMemcpyDefault, h->stream));
  CUDA_OR_FAIL(h, cudaStreamSynchronize(h->stream));
  return DLMPC_OK;
}

int dlmpc_set_halo(dlmpc_handle* h, const int64_t* send_cells, int64_t n_send,
                   const int64_t* recv_cells, int64_t n_recv) {
  if (!h || n_send < 0 || n_recv < 0 || (n_send && !send_cells) || (n_recv && !recv_cells))
    return fail(h, DLMPC_BAD_ARGUMENT, "bad halo cell lists");
  const int64_t n_cell = (int64_t)h->P.n_cols * h->P.s_pad;
  for (int64_t k = 0; k < n_send; ++k)
    if (send_cells[k] < 0 || send_cells[k] >= n_cell) return fail(h, DLMPC_BAD_ARGUMENT, "send cell out of range");
  for (int64_t k = 0; k < n_recv; ++k)
    if (recv_cells[k] < 0 || recv_cells[k] >= n_cell) return fail(h, DLMPC_BAD_ARGUMENT, "recv cell out of range");
  cudaSetDevice(h->device);
  CUDA_OR_FAIL(h, cudaStreamSynchronize(h->stream));
  for (int64_t** p : {&h->d_send_cells, &h->d_recv_cells})
    if (*p) { cudaFree(*p); *p = nullptr; }
  if (h->d_halo) { cudaFree(h->d_halo); h->d_halo = nullptr; }
  h->n_send = n_send; h->n_recv = n_recv;
  if (n_send) {
    CUDA_OR_FAIL(h, cudaMalloc(&h->d_send_cells, sizeof(int64_t) * n_send));
    CUDA_OR_FAIL(h, cudaMemcpy(h->d_send_cells, send_cells, sizeof(int64_t) * n_send, cudaMemcpyHostToDevice));
  }
  if (n_recv) {
    CUDA_OR_FAIL(h, cudaMalloc(&h->d_recv_cells, sizeof(int64_t) * n_recv));
    CUDA_OR_FAIL(h, cudaMemcpy(h->d_recv_cells, recv_cells, sizeof(int64_t) * n_recv, cudaMemcpyHostToDevice));
  }
  const int64_t nb = std::max<int64_t>(1, std::max(n_send, n_recv));
  CUDA_OR_FAIL(h, cudaMalloc(&h->d_halo, sizeof(double) * 2 * nb));
  return DLMPC_OK;
}

int dlmpc_halo_pack(dlmpc_handle* h, double* out) {
  if (!h || (h->n_send && !out)) return fail(h, DLMPC_BAD_ARGUMENT, "null halo buffer");
  if (!h->n_send) return DLMPC_OK;
  cudaSetDevice(h->device);
  int b = 0;
  if (int rc = current_buffer(h, &b)) return rc;
  const int blocks = (int)std::min<int64_t>(h->sm_count * 4, (h->n_send + 255) / 256);
  halo_pack_kernel<<<blocks, 256, 0, h->stream>>>(h->P.psi[b], h->P.lam[b], h->d_send_cells, h->n_send,
                                                  reinterpret_cast<double2*>(h->d_halo));
  CUDA_OR_FAIL(h, cudaGetLastError());
  CUDA_OR_FAIL(h, cudaMemcpyAsync(out, h->d_halo, sizeof(double) * 2 * h->n_send, cudaMemcpyDefault, h->stream));
  CUDA_OR_FAIL(h, cudaStreamSynchronize(h->stream));
  return DLMPC_OK;
}

int dlmpc_halo_pack_async(dlmpc_handle* h, double* out_dev) {
  if (!h || (h->n_send && !out_dev)) return fail(h, DLMPC_BAD_ARGUMENT, "null halo buffer");
  if (!h->n_send) return DLMPC_OK;
  cudaSetDevice(h->device);
  int b = 0;
  if (int rc = current_buffer(h, &b)) return rc;
  const int blocks = (int)std::min<int64_t>(h->sm_count * 4, (h->n_send + 255) / 256);
  halo_pack_kernel<<<blocks, 256, 0, h->stream>>>(h->P.psi[b], h->P.lam[b], h->d_send_cells, h->n_send,
                                                  reinterpret_cast<double2*>(out_dev));
  CUDA_OR_FAIL(h, cudaGetLastError());
  return DLMPC_OK;
}

int dlmpc_halo_unpack_async(dlmpc_handle* h, const double* in_dev) {
  if (!h || (h->n_recv && !in_dev)) return fail(h, DLMPC_BAD_ARGUMENT, "null halo buffer");
  if (!h->n_recv) return DLMPC_OK;
  cudaSetDevice(h->device);
  int b = 0;
  if (int rc = current_buffer(h, &b)) return rc;
  const int blocks = (int)std::min<int64_t>(h->sm_count * 4, (h->n_recv + 255) / 256);
  halo_unpack_kernel<<<blocks, 256, 0, h->stream>>>(h->P.psi[b], h->P.lam[b], h->d_recv_cells, h->n_recv,
                                                    reinterpret_cast<const double2*>(in_dev));
  CUDA_OR_FAIL(h, cudaGetLastError());
  return DLMPC_OK;
}

int dlmpc_iterate_async(dlmpc_handle* h, int n, double* resid_dev) {
  if (!h || n < 1 || !resid_dev) return fail(h, DLMPC_BAD_ARGUMENT, "bad argument");
  cudaSetDevice(h->device);
  int b = 0;
  if (int rc = current_buffer(h, &b)) return rc;   // (a round trip only after a stop-tested launch)
  if (int rc = ensure_run_buffers(h, n, 1)) return rc;
  RunArgs R{};
  R.t_sim = 1; R.closed_loop = 0; R.warm_start = 1; R.cold_start = 0;
  R.max_iters = n; R.stop_on_conv = 0;
  R.hist = h->d_hist; R.step_iters = h->d_step_iters; R.states = h->d_states; R.inputs = h->d_inputs;
  R.it_base = h->it_cont;
  if (int rc = launch(h, R)) return rc;
  CUDA_OR_FAIL(h, cudaMemcpyAsync(resid_dev, h->d_hist + 2 * (n - 1), sizeof(double) * 2, cudaMemcpyDeviceToDevice,
                                  h->stream));
  CUDA_OR_FAIL(h, cudaGetLastError());
  h->it_cont += n;
  h->cur_b = b ^ (n & 1); h->b_valid = 1;   // no stop test: exactly n buffer swaps
  return DLMPC_OK;
}

int dlmpc_set_stream(dlmpc_handle* h, void* stream) {
  if (!h) return fail(h, DLMPC_BAD_ARGUMENT, "null handle");
  cudaSetDevice(h->device);
  CUDA_OR_FAIL(h, cudaStreamSynchronize(h->stream));   // work queued on the old stream first
  h->stream = stream ? static_cast<cudaStream_t>(stream) : h->own_stream;
  return DLMPC_OK;
}

int dlmpc_halo_unpack(dlmpc_handle* h, const double* in) {
  if (!h || (h->n_recv && !in)) return fail(h, DLMPC_BAD_ARGUMENT, "null halo buffer");
  if (!h->n_recv) return DLMPC_OK;
  // (the stream kernel's Φ-dot partials stay valid: they hold only owned
  // columns' contributions, and rows reading halo columns recompute their
  // full Φ every iteration)
  cudaSetDevice(h->device);
  int b = 0;
  if (int rc = current_buffer(h, &b)) return rc;
  CUDA_OR_FAIL(h, cudaMemcpyAsync(h->d_halo, in, sizeof(double) * 2 * h->n_recv, cudaMemcpyDefault, h->stream));
  const int blocks = (int)std::min<int64_t>(h->sm_count * 4, (h->n_recv + 255) / 256);
  halo_unpack_kernel<<<blocks, 256, 0, h->stream>>>(h->P.psi[b], h->P.lam[b], h->d_recv_cells, h->n_recv,
                                                    reinterpret_cast<const double2*>(h->d_halo));
  CUDA_OR_FAIL(h, cudaGetLastError());
  CUDA_OR_FAIL(h, cudaStreamSynchronize(h->stream));
  return DLMPC_OK;
}

int dlmpc_finish_step(dlmpc_handle* h, double* u_out, double* x_next_out) {
  if (!h) return fail(h, DLMPC_BAD_ARGUMENT, "null handle");
  cudaSetDevice(h->device);
  int ctl[8];
  if (int rc = read_ctl(h, ctl)) return rc;
  const int pb = ctl[4] ^ 1;
  const int blocks = std::max(1, std::min(h->sm_count * 8, (std::max(h->P.n_cols, h->P.n_inputs) + 7) / 8));   // a warp per item
  if (h->P.exact) control_kernel<true><<<blocks, 256, 0, h->stream>>>(h->P, pb);
  else control_kernel<false><<<blocks, 256, 0, h->stream>>>(h->P, pb);
  CUDA_OR_FAIL(h, cudaGetLastError());
  plant_kernel<<<blocks, 256, 0, h->stream>>>(h->P);
  CUDA_OR_FAIL(h, cudaGetLastError());
  if (u_out && h->P.n_inputs)
    CUDA_OR_FAIL(h, cudaMemcpyAsync(u_out, h->P.u, sizeof(double) * h->P.n_inputs, cudaMemcpyDeviceToHost, h->stream));
  if (x_next_out)
    CUDA_OR_FAIL(h, cudaMemcpyAsync(x_next_out, h->P.x[1], sizeof(double) * h->P.n_cols, cudaMemcpyDeviceToHost, h->stream));
  CUDA_OR_FAIL(h, cudaStreamSynchronize(h->stream));
  h->last_launches = 2;
  return DLMPC_OK;
}

int dlmpc_zero(dlmpc_handle* h) {
  if (h) h->it_cont = 0;
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
  return check_dbg(h);
}

int dlmpc_audit(dlmpc_handle* h, const double* phi_host, double* out3) {
  if (!h || !out3) return fail(h, DLMPC_BAD_ARGUMENT, "null argument");
  if (!h->P.g0_pool) return fail(h, DLMPC_BAD_ARGUMENT, "problem was created without audit tables");
  cudaSetDevice(h->device);
  int ctl[8];
  if (int rc = read_ctl(h, ctl)) return rc;
  const int b = ctl[4];
  if (!h->d_audit) CUDA_OR_FAIL(h, cudaMalloc(&h->d_audit, sizeof(double) * ((size_t)h->P.n_rows + 4)));
  double* s_fresh = h->d_audit;       // fresh Φ scale per row
  double* out = h->d_audit + h->P.n_rows;
  CUDA_OR_FAIL(h, cudaMemsetAsync(out, 0, sizeof(double) * 3, h->stream));
  const double* phi_dev = nullptr;
  if (phi_host) {   // audit a caller-provided φ (internal layout) instead of the recomputed one
    const size_t ncell = (size_t)h->P.n_cols * h->P.s_pad;
    if (!h->d_scratch2) CUDA_OR_FAIL(h, cudaMalloc(&h->d_scratch2, sizeof(double) * ncell));
    CUDA_OR_FAIL(h, cudaMemcpyAsync(h->d_scratch2, phi_host, sizeof(double) * ncell, cudaMemcpyHostToDevice, h->stream));
    phi_dev = h->d_scratch2;
  }
  const int warps = 16, blocks = (h->P.n_sub + warps - 1) / warps;
  const double* x = h->P.x[0];
  if (h->P.exact) audit_phi_kernel<true><<<blocks, 32 * warps, 0, h->stream>>>(h->P, b, x, s_fresh);
  else audit_phi_kernel<false><<<blocks, 32 * warps, 0, h->stream>>>(h->P, b, x, s_fresh);
  CUDA_OR_FAIL(h, cudaGetLastError());
  if (h->P.exact) audit_entries_kernel<true><<<h->sm_count * 4, 512, 0, h->stream>>>(h->P, b, x, s_fresh, phi_dev, out);
  else audit_entries_kernel<false><<<h->sm_count * 4, 512, 0, h->stream>>>(h->P, b, x, s_fresh, phi_dev, out);
  CUDA_OR_FAIL(h, cudaGetLastError());
  audit_dynamics_kernel<<<h->sm_count * 4, 256, 0, h->stream>>>(h->P, b, out);
  CUDA_OR_FAIL(h, cudaGetLastError());
  CUDA_OR_FAIL(h, cudaMemcpyAsync(out3, out, sizeof(double) * 3, cudaMemcpyDeviceToHost, h->stream));
  CUDA_OR_FAIL(h, cudaStreamSynchronize(h->stream));
  h->last_launches = 3;
  return DLMPC_OK;
}

int dlmpc_phase_times(dlmpc_handle* h, uint64_t* out, int reset) {
  if (!h || !out) return DLMPC_BAD_ARGUMENT;
  CUDA_OR_FAIL(h, cudaMemcpy(out, h->P.phase_ns, sizeof(uint64_t) * 16 * h->grid, cudaMemcpyDeviceToHost));
  if (reset) CUDA_OR_FAIL(h, cudaMemset(h->P.phase_ns, 0, sizeof(uint64_t) * 16 * h->grid));
  return DLMPC_OK;
}

// ---------------------------------------------------------------------------
// Graph-partitioned solve with the exchange on the device (include/dlmpc.h)
// ---------------------------------------------------------------------------
int dlmpc_dist_alloc(dlmpc_handle* h, int world, void** out7) {
  if (!h || !out7 || world < 1) return fail(h, DLMPC_BAD_ARGUMENT, "bad argument");
  if (h->mode == kPatch || h->mode == kPatchRb)
    return fail(h, DLMPC_BAD_ARGUMENT, "the device exchange needs a non-patch kernel mode (stream, two-phase, exact)");
  cudaSetDevice(h->device);
  DevProblem& P = h->P;
  if (h->dist_world != world) {
    int rc;
    unsigned* flag; unsigned* rflag; unsigned long long* slots; int* abort_;
    if ((rc = alloc(h, 1, &flag)) || (rc = alloc(h, 1, &rflag)) || (rc = alloc(h, (size_t)4 * world, &slots)) ||
        (rc = alloc(h, 1, &abort_)))
      return rc;
    P.d_flag = flag; P.d_rflag = rflag; P.d_slots = slots; P.d_abort = abort_;
    h->dist_world = world;
    h->dist_epoch = 0;
  }
  out7[0] = P.psi[0]; out7[1] = P.psi[1]; out7[2] = P.lam[0]; out7[3] = P.lam[1];
  out7[4] = P.d_flag; out7[5] = P.d_slots; out7[6] = P.d_rflag;
  return DLMPC_OK;
}

int dlmpc_dist_setup(dlmpc_handle* h, int rank, int world, int n_peers, int64_t n_send,
                     const int64_t* send_src, const int64_t* send_dst, const int32_t* send_peer,
                     void* const* peer_psi, void* const* peer_lam, void* const* peer_flag,
                     uint32_t halo_per_iter, void* const* all_slots, void* const* all_rflag) {
  if (!h || world != h->dist_world || rank < 0 || rank >= world || n_peers < 0 || n_send < 0 ||
      (n_send > 0 && (!send_src || !send_dst || !send_peer)) || (n_peers > 0 && (!peer_psi || !peer_lam || !peer_flag)) ||
      !all_slots || !all_rflag)
    return fail(h, DLMPC_BAD_ARGUMENT, "bad argument (call dlmpc_dist_alloc first)");
  for (int64_t i = 0; i < n_send; ++i)
    if (send_peer[i] < 0 || send_peer[i] >= n_peers || send_src[i] < 0 ||
        send_src[i] >= (int64_t)h->P.n_cols * h->P.s_pad || send_dst[i] < 0)
      return fail(h, DLMPC_BAD_ARGUMENT, "send list entry out of range");
  cudaSetDevice(h->device);
  DevProblem& P = h->P;
  int rc;
  std::vector<double*> pp(2 * (size_t)std::max(1, n_peers)), pl(2 * (size_t)std::max(1, n_peers));
  std::vector<unsigned*> pf(std::max(1, n_peers));
  for (int q = 0; q < n_peers; ++q) {
    for (int k = 0; k < 2; ++k) {
      pp[2 * q + k] = static_cast<double*>(peer_psi[2 * q + k]);
      pl[2 * q + k] = static_cast<double*>(peer_lam[2 * q + k]);
    }
    pf[q] = static_cast<unsigned*>(peer_flag[q]);
  }
  std::vector<unsigned long long*> as(world);
  std::vector<unsigned*> ar(world);
  for (int r = 0; r < world; ++r) {
    as[r] = static_cast<unsigned long long*>(all_slots[r]);
    ar[r] = static_cast<unsigned*>(all_rflag[r]);
  }
  const long long* src64 = reinterpret_cast<const long long*>(send_src);
  const long long* dst64 = reinterpret_cast<const long long*>(send_dst);
  const long long* dsrc; const long long* ddst; const int* dpeer;
  double* const* dpp; double* const* dpl; unsigned* const* dpf;
  unsigned long long* const* das; unsigned* const* dar;
  if ((rc = upload(h, src64, (size_t)n_send, &dsrc)) || (rc = upload(h, dst64, (size_t)n_send, &ddst)) ||
      (rc = upload(h, send_peer, (size_t)n_send, &dpeer)) ||
      (rc = upload(h, pp.data(), pp.size(), &dpp)) || (rc = upload(h, pl.data(), pl.size(), &dpl)) ||
      (rc = upload(h, pf.data(), pf.size(), &dpf)) ||
      (rc = upload(h, as.data(), as.size(), &das)) || (rc = upload(h, ar.data(), ar.size(), &dar)))
    return rc;
  P.d_send_src = dsrc; P.d_send_dst = ddst; P.d_send_peer = dpeer;
  P.d_peer_psi = dpp; P.d_peer_lam = dpl; P.d_peer_flag = dpf;
  P.d_all_slots = das; P.d_all_rflag = dar;
  P.d_rank = rank; P.d_world = world; P.d_npeer = n_peers; P.d_nsend = n_send;
  P.d_halo_per_iter = halo_per_iter;
  P.dist = 1;
  return DLMPC_OK;
}

namespace {
RunArgs solve_args(dlmpc_handle* h, int max_iters, double eps_pri, double eps_dual) {
  RunArgs R{};
  R.t_sim = 1; R.closed_loop = 0; R.warm_start = 1; R.cold_start = 0;
  R.max_iters = max_iters; R.stop_on_conv = 1; R.eps_pri = eps_pri; R.eps_dual = eps_dual;
  R.hist = h->d_hist; R.step_iters = h->d_step_iters; R.states = h->d_states; R.inputs = h->d_inputs;
  R.it_base = h->it_cont;
  R.dist_epoch = h->dist_epoch;
  return R;
}

// after a dist launch: status, iterations, history; the counters' base moves on
int finish_dist(dlmpc_handle* h, int* iters, double* hist) {
  int ctl[8];
  if (int rc = read_ctl(h, ctl)) return rc;
  int n = 0;
  CUDA_OR_FAIL(h, cudaMemcpy(&n, h->d_step_iters, sizeof(int), cudaMemcpyDeviceToHost));
  if (ctl[0] != 0) n = ctl[5];
  if (ctl[0] == 4) return fail(h, DLMPC_CUDA_ERROR, "device exchange timed out (a neighbour rank did not arrive)");
  h->dist_epoch += (unsigned)n;
  h->it_cont += n;
  if (iters) *iters = n;
  if (hist && n > 0) CUDA_OR_FAIL(h, cudaMemcpy(hist, h->d_hist, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost));
  return ctl[0];
}
}  // namespace

int dlmpc_dist_solve(dlmpc_handle* h, int max_iters, double eps_pri, double eps_dual, int* iters, double* hist) {
  if (!h || max_iters < 1) return fail(h, DLMPC_BAD_ARGUMENT, "bad argument");
  if (!h->P.dist) return fail(h, DLMPC_BAD_ARGUMENT, "dlmpc_dist_setup first");
  cudaSetDevice(h->device);
  if (int rc = ensure_run_buffers(h, max_iters, 1)) return rc;
  RunArgs R = solve_args(h, max_iters, eps_pri, eps_dual);
  if (int rc = launch(h, R, kVarDist)) return rc;
  if (int rc = finish_timing(h)) return rc;
  CUDA_OR_FAIL(h, cudaGetLastError());
  return finish_dist(h, iters, hist);
}

int dlmpc_multi_solve(dlmpc_handle* const* hs, int n, int max_iters, double eps_pri, double eps_dual,
                      int* iters, double* hist) {
  if (!hs || n < 1 || max_iters < 1) return fail(nullptr, DLMPC_BAD_ARGUMENT, "bad argument");
  dlmpc_handle* h0 = hs[0];
  for (int r = 0; r < n; ++r) {
    if (!hs[r] || hs[r]->device != h0->device || hs[r]->mode != h0->mode || hs[r]->P.tile_cols != h0->P.tile_cols)
      return fail(h0, DLMPC_BAD_ARGUMENT, "the ranks must share device, kernel mode and tile width");
    if (!hs[r]->P.dist) return fail(h0, DLMPC_BAD_ARGUMENT, "dlmpc_dist_setup first on every rank");
  }
  if (h0->mode != kExact && h0->mode != kStream && h0->mode != kTwoPhase)
    return fail(h0, DLMPC_BAD_ARGUMENT, "no multi-rank kernel for this mode");
  cudaSetDevice(h0->device);
  std::vector<DevProblem> probs(n);
  std::vector<RunArgs> runs(n);
  std::vector<int> base(n + 1, 0);
  int smem = 0;
  for (int r = 0; r < n; ++r) {
    dlmpc_handle* h = hs[r];
    if (int rc = ensure_run_buffers(h, max_iters, 1)) return rc;
    CUDA_OR_FAIL(h, cudaStreamSynchronize(h->stream));
    probs[r] = h->P;
    probs[r].vbase = base[r];
    probs[r].vgrid = h->grid;
    runs[r] = solve_args(h, max_iters, eps_pri, eps_dual);
    base[r + 1] = base[r] + h->grid;
    smem = std::max(smem, h->smem_bytes);
  }
  DevProblem* dprobs = nullptr; RunArgs* druns = nullptr; int* dbase = nullptr;
  CUDA_OR_FAIL(h0, cudaMalloc(&dprobs, sizeof(DevProblem) * n));
  CUDA_OR_FAIL(h0, cudaMalloc(&druns, sizeof(RunArgs) * n));
  CUDA_OR_FAIL(h0, cudaMalloc(&dbase, sizeof(int) * (n + 1)));
  cudaError_t e = cudaMemcpy(dprobs, probs.data(), sizeof(DevProblem) * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(druns, runs.data(), sizeof(RunArgs) * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(dbase, base.data(), sizeof(int) * (n + 1), cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = launch_multi_kernel(h0->mode, h0->P.tile_cols, dprobs, druns, dbase, n, base[n], smem, h0->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h0->stream);
  cudaFree(dprobs); cudaFree(druns); cudaFree(dbase);
  if (e != cudaSuccess) return fail(h0, DLMPC_CUDA_ERROR, std::string("multi-rank launch: ") + cudaGetErrorString(e));
  int status = DLMPC_OK;
  for (int r = 0; r < n; ++r) {
    hs[r]->b_valid = 0;
    const int rc = finish_dist(hs[r], r == 0 ? iters : nullptr, r == 0 ? hist : nullptr);
    if (rc != DLMPC_OK && status == DLMPC_OK) status = rc;
  }
  return status;
}

int dlmpc_ipc_get(const void* dev_ptr, void* handle64) {
  if (!dev_ptr || !handle64) return fail(nullptr, DLMPC_BAD_ARGUMENT, "null argument");
  cudaIpcMemHandle_t hd;
  const cudaError_t e = cudaIpcGetMemHandle(&hd, const_cast<void*>(dev_ptr));
  if (e != cudaSuccess) return fail(nullptr, DLMPC_CUDA_ERROR, std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e));
  std::memcpy(handle64, &hd, sizeof(hd));
  return DLMPC_OK;
}

int dlmpc_ipc_open(const void* handle64, int device, void** dev_ptr) {
  if (!handle64 || !dev_ptr) return fail(nullptr, DLMPC_BAD_ARGUMENT, "null argument");
  cudaSetDevice(device);
  cudaIpcMemHandle_t hd;
  std::memcpy(&hd, handle64, sizeof(hd));
  const cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, hd, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail(nullptr, DLMPC_CUDA_ERROR, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
  return DLMPC_OK;
}

int dlmpc_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return DLMPC_OK;
  const cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
  return e == cudaSuccess ? DLMPC_OK : fail(nullptr, DLMPC_CUDA_ERROR, cudaGetErrorString(e));
}

// FP64 tensor-core peak of this GPU, measured live (the roofline denominator
// of the FP64 fraction; MEASURED_PEAKS.json carries HBM and bf16 only): every
// warp runs 8 independent m8n8k4 DMMA accumulation chains, 4 CTAs x 256
// threads per SM, best of 3 launches of ~20 ms.
__global__ void fp64_dmma_probe_kernel(double* out, int iters) {
  const double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;   // keeps the chains live
}

int dlmpc_fp64_peak(int device, double* tflops) {
  if (!tflops) return fail(nullptr, DLMPC_BAD_ARGUMENT, "null argument");
  if (cudaSetDevice(device) != cudaSuccess) return fail(nullptr, DLMPC_NO_DEVICE, "cudaSetDevice failed");
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess)
    return fail(nullptr, DLMPC_CUDA_ERROR, "device attribute");
  double* out = nullptr;
  cudaEvent_t e0, e1;
  if (cudaMalloc(&out, 64) != cudaSuccess) return fail(nullptr, DLMPC_CUDA_ERROR, "cudaMalloc");
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = sms * 4, threads = 256, iters = 4000;
  fp64_dmma_probe_kernel<<<blocks, threads>>>(out, 64);
  double best = 0.0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    fp64_dmma_probe_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    if (cudaEventSynchronize(e1) != cudaSuccess) break;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flop = 2.0 * 256 * 8 * (double)iters * blocks * (threads / 32);   // 8x8x4 MACs per DMMA
    best = std::max(best, flop / (ms * 1e-3) / 1e12);
  }
  const cudaError_t err = cudaGetLastError();
  cudaEventDestroy(e0); cudaEventDestroy(e1); cudaFree(out);
  if (err != cudaSuccess || best <= 0.0) return fail(nullptr, DLMPC_CUDA_ERROR, "fp64 probe failed");
  *tflops = best;
  return DLMPC_OK;
}

int dlmpc_info(const dlmpc_handle* h, int64_t* out) {
  if (!h || !out) return DLMPC_BAD_ARGUMENT;
  out[0] = h->P.n_rows; out[1] = h->P.n_cols; out[2] = h->P.s_pad; out[3] = h->P.n_sub;
  out[4] = h->grid; out[5] = h->P.tile_cols; out[6] = h->smem_bytes;
  out[7] = h->mode; out[8] = h->n_units;
  return DLMPC_OK;
}

int dlmpc_plan_flags(const dlmpc_handle* h, int64_t* out, int n) {
  if (!h || !out || n < 0) return DLMPC_BAD_ARGUMENT;
  const int64_t v[5] = {h->P.cache_phi, h->P.fuse_steps, h->P.rb_gemv, h->P.stash_bufs, h->P.cta_pair ? 1 : 0};
  for (int i = 0; i < n && i < 5; ++i) out[i] = v[i];
  return DLMPC_OK;
}

}  // extern "C"

// ===========================================================================
// The reference's device schedules (dlmpc_schedules.cuh) and its scalar stage
// functions as standalone device operators.
// ===========================================================================
#include "dlmpc_schedules.cuh"

struct dlmpc_sched {
  int device = 0;
  cudaStream_t stream = nullptr;
  sched::RefDev R{};
  std::vector<void*> allocs;
  std::string err;
  int sm_count = 0;
  int smem_psi = 0;       // dynamic shared memory of the Ψ-carrying kernels (k [s] + r [m])
  long long n_x = 0;      // state dimension (max column index + 1)
  double* d_x = nullptr;  // measured state of the current step
  double* d_out = nullptr; size_t out_cap = 0;   // _phi_compute scratch
  bool has_patch = false;
};

namespace {

int sfail(dlmpc_sched* h, int code, const std::string& msg) {
  if (h) h->err = msg; else g_global_error = msg;
  return code;
}

#define SCUDA(h, expr)                                                                 \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return sfail((h), DLMPC_CUDA_ERROR, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

template <class T>   // T from dst only: src may be nullptr (zeroed allocation)
int supload(dlmpc_sched* h, const typename std::common_type<T>::type* src, size_t n, T** dst) {
  *dst = nullptr;
  void* p = nullptr;
  SCUDA(h, cudaMalloc(&p, (n ? n : 1) * sizeof(T)));
  h->allocs.push_back(p);
  if (src && n) SCUDA(h, cudaMemcpy(p, src, n * sizeof(T), cudaMemcpyHostToDevice));
  else SCUDA(h, cudaMemset(p, 0, (n ? n : 1) * sizeof(T)));
  *dst = static_cast<T*>(p);
  return DLMPC_OK;
}

double* sched_array(dlmpc_sched* h, int which, size_t* n) {
  sched::RefDev& R = h->R;
  const size_t nr = (size_t)R.n_rows * R.d_row, nc = (size_t)R.n_cols * R.d_col;
  switch (which) {
    case DLMPC_SCHED_PHI_R: *n = nr; return R.phi_r;
    case DLMPC_SCHED_PSI_R: *n = nr; return R.psi_r;
    case DLMPC_SCHED_LAM_R: *n = nr; return R.lam_r;
    case DLMPC_SCHED_PHI_C: *n = nc; return R.phi_c;
    case DLMPC_SCHED_PSI_C: *n = nc; return R.psi_c;
    case DLMPC_SCHED_LAM_C: *n = nc; return R.lam_c;
    case DLMPC_SCHED_PSI_PREV_C: *n = nc; return R.prev_c;
    case DLMPC_SCHED_PRI_C: *n = R.n_cols; return R.pri_c;
    case DLMPC_SCHED_DUAL_C: *n = R.n_cols; return R.dual_c;
    case DLMPC_SCHED_A_PAD: *n = nr; return R.a_pad;
    case DLMPC_SCHED_ADA: *n = R.n_rows; return R.ada;
    case DLMPC_SCHED_ROW_W: *n = R.n_rows; return R.w;
    case DLMPC_SCHED_ROW_LO: *n = R.n_rows; return R.lo;
    case DLMPC_SCHED_ROW_HI: *n = R.n_rows; return R.hi;
    default: *n = 0; return nullptr;
  }
}

// Host-pointer operands of one standalone operator call: device copies freed
// on scope exit.
struct OpBufs {
  std::vector<void*> p;
  ~OpBufs() { for (void* q : p) cudaFree(q); }
  template <class T>
  T* up(const T* src, size_t n) {
    void* q = nullptr;
    if (cudaMalloc(&q, (n ? n : 1) * sizeof(T)) != cudaSuccess) return nullptr;
    p.push_back(q);
    if (src && n && cudaMemcpy(q, src, n * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
    return static_cast<T*>(q);
  }
};

int op_begin(int device) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return sfail(nullptr, DLMPC_NO_DEVICE, "no CUDA device visible");
  if (device < 0 || device >= ndev) return sfail(nullptr, DLMPC_BAD_ARGUMENT, "device out of range");
  if (cudaSetDevice(device) != cudaSuccess) return sfail(nullptr, DLMPC_CUDA_ERROR, "cudaSetDevice failed");
  return DLMPC_OK;
}

int op_end(double* host_out, const double* dev_out, size_t n) {
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess && n) e = cudaMemcpy(host_out, dev_out, n * sizeof(double), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return sfail(nullptr, DLMPC_CUDA_ERROR, std::string("operator: ") + cudaGetErrorString(e));
  return DLMPC_OK;
}

int grid_for(long long n, int per_block) {
  return (int)std::max<long long>(1, std::min<long long>((n + per_block - 1) / per_block, 148LL * 16));
}

}  // namespace

extern "C" {

int dlmpc_sched_create(const dlmpc_sched_problem* pr, int device, dlmpc_sched** out) {
  if (!pr || !out) return sfail(nullptr, DLMPC_BAD_ARGUMENT, "null argument");
  *out = nullptr;
  if (int rc = op_begin(device)) return rc;
  if (pr->n_rows < 1 || pr->n_cols < 1 || pr->d_row < 1 || pr->d_col < 1)
    return sfail(nullptr, DLMPC_BAD_ARGUMENT, "empty layout");
  auto* h = new dlmpc_sched();
  h->device = device;
  sched::RefDev& R = h->R;
  R.n_rows = pr->n_rows; R.n_cols = pr->n_cols; R.d_row = pr->d_row; R.d_col = pr->d_col;
  R.n_elems = pr->n_elems; R.rho = pr->rho;
  const size_t nr = (size_t)R.n_rows * R.d_row, nc = (size_t)R.n_cols * R.d_col;
  int rc = DLMPC_OK;
  int m_max = 1, s_max = 1;
  for (int k = 0; k < pr->n_classes; ++k) { m_max = std::max(m_max, pr->class_m[k]); s_max = std::max(s_max, pr->class_s[k]); }
  h->smem_psi = (m_max + s_max) * 8;
  long long nx = 0;
  for (size_t q = 0; q < nr; ++q) nx = std::max<long long>(nx, pr->rs[q] + 1);
  h->n_x = nx;
#define SUP(field, src, n) do { if ((rc = supload(h, src, (size_t)(n), &field)) != DLMPC_OK) goto bad; } while (0)
  {
    int* row_len; int* col_len; long long* rs; long long* c2r; long long* r2c; long long* ef;
    int* col_class; int* class_m; long long* g_off; double* g_pool; long long* p_off; double* p_pool;
    long long* rhs_off; double* rhs_pool;
    SUP(row_len, pr->row_len, R.n_rows); SUP(col_len, pr->col_len, R.n_cols);
    SUP(rs, reinterpret_cast<const long long*>(pr->rs), nr);
    SUP(c2r, reinterpret_cast<const long long*>(pr->c2r_flat), nc);
    SUP(r2c, reinterpret_cast<const long long*>(pr->r2c_flat), nr);
    SUP(ef, reinterpret_cast<const long long*>(pr->elem_flat_col), R.n_elems);
    SUP(col_class, pr->col_class, R.n_cols); SUP(class_m, pr->class_m, pr->n_classes);
    SUP(g_off, reinterpret_cast<const long long*>(pr->class_g_off), pr->n_classes + 1);
    SUP(g_pool, pr->g_pool, pr->class_g_off[pr->n_classes]);
    SUP(p_off, reinterpret_cast<const long long*>(pr->class_p_off), pr->n_classes + 1);
    SUP(p_pool, pr->p_pool, pr->class_p_off[pr->n_classes]);
    SUP(rhs_off, reinterpret_cast<const long long*>(pr->col_rhs_off), R.n_cols + 1);
    SUP(rhs_pool, pr->rhs_pool, pr->col_rhs_off[R.n_cols]);
    SUP(R.w, pr->row_w, R.n_rows); SUP(R.lo, pr->row_lo, R.n_rows); SUP(R.hi, pr->row_hi, R.n_rows);
    R.row_len = row_len; R.col_len = col_len; R.rs = rs; R.c2r = c2r; R.r2c = r2c; R.elem_flat = ef;
    R.col_class = col_class; R.class_m = class_m; R.g_off = g_off; R.g_pool = g_pool; R.p_off = p_off;
    R.p_pool = p_pool; R.rhs_off = rhs_off; R.rhs_pool = rhs_pool;
    if (pr->n_patch > 0 && pr->patch_off && pr->patch_rows && pr->patch_slot && pr->patch_owned) {
      long long* po; long long* prw; int* ps; int* pw;
      SUP(po, reinterpret_cast<const long long*>(pr->patch_off), R.n_cols + 1);
      SUP(prw, reinterpret_cast<const long long*>(pr->patch_rows), pr->n_patch);
      SUP(ps, pr->patch_slot, pr->n_patch); SUP(pw, pr->patch_owned, pr->n_patch);
      R.patch_off = po; R.patch_rows = prw; R.patch_slot = ps; R.patch_owned = pw;
      h->has_patch = true;
    }
    SUP(R.phi_r, nullptr, nr); SUP(R.psi_r, nullptr, nr); SUP(R.lam_r, nullptr, nr);
    SUP(R.psi_r_nx, nullptr, nr); SUP(R.lam_r_nx, nullptr, nr);
    SUP(R.phi_c, nullptr, nc); SUP(R.psi_c, nullptr, nc); SUP(R.lam_c, nullptr, nc); SUP(R.prev_c, nullptr, nc);
    SUP(R.pri_c, nullptr, R.n_cols); SUP(R.dual_c, nullptr, R.n_cols);
    SUP(R.a_pad, nullptr, nr); SUP(R.ada, nullptr, R.n_rows);
    SUP(R.resid, nullptr, 2); SUP(R.bad, nullptr, 1); SUP(h->d_x, nullptr, std::max<long long>(1, nx));
    if (h->smem_psi > 48 * 1024) {
      const void* fns[] = {reinterpret_cast<const void*>(sched::psi_cols_kernel),
                           reinterpret_cast<const void*>(sched::fused_cols_kernel),
                           reinterpret_cast<const void*>(sched::patch_cols_kernel<false>),
                           reinterpret_cast<const void*>(sched::patch_cols_kernel<true>)};
      for (const void* f : fns)
        if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, h->smem_psi) != cudaSuccess) {
          rc = sfail(h, DLMPC_BAD_ARGUMENT, "column operator too large for shared memory"); goto bad;
        }
    }
    if (cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, device) != cudaSuccess ||
        cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess) {
      rc = sfail(h, DLMPC_CUDA_ERROR, "stream creation failed"); goto bad;
    }
  }
#undef SUP
  *out = h;
  return DLMPC_OK;
bad:
  g_global_error = h->err;
  dlmpc_sched_destroy(h);
  return rc;
}

void dlmpc_sched_destroy(dlmpc_sched* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (void* p : h->allocs) cudaFree(p);
  if (h->d_out) cudaFree(h->d_out);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

const char* dlmpc_sched_last_error(const dlmpc_sched* h) { return h ? h->err.c_str() : g_global_error.c_str(); }

int dlmpc_sched_put(dlmpc_sched* h, int which, const double* src) {
  if (!h || !src) return sfail(h, DLMPC_BAD_ARGUMENT, "null argument");
  size_t n = 0;
  double* dst = sched_array(h, which, &n);
  if (!dst) return sfail(h, DLMPC_BAD_ARGUMENT, "unknown array");
  cudaSetDevice(h->device);
  SCUDA(h, cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  SCUDA(h, cudaStreamSynchronize(h->stream));
  return DLMPC_OK;
}

int dlmpc_sched_get(dlmpc_sched* h, int which, double* dst) {
  if (!h || !dst) return sfail(h, DLMPC_BAD_ARGUMENT, "null argument");
  size_t n = 0;
  double* src = sched_array(h, which, &n);
  if (!src) return sfail(h, DLMPC_BAD_ARGUMENT, "unknown array");
  cudaSetDevice(h->device);
  SCUDA(h, cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  SCUDA(h, cudaStreamSynchronize(h->stream));
  return DLMPC_OK;
}

int dlmpc_sched_set_x(dlmpc_sched* h, const double* x, int64_t n_x, int64_t* bad_row) {
  if (!h || !x) return sfail(h, DLMPC_BAD_ARGUMENT, "null argument");
  if (n_x < h->n_x) return sfail(h, DLMPC_BAD_ARGUMENT, "state shorter than the layout's columns");
  cudaSetDevice(h->device);
  SCUDA(h, cudaMemcpyAsync(h->d_x, x, h->n_x * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  SCUDA(h, cudaMemsetAsync(h->R.bad, 0x7f, sizeof(int), h->stream));
  sched::set_x_kernel<<<grid_for(h->R.n_rows, 256), 256, 0, h->stream>>>(h->R, h->d_x);
  SCUDA(h, cudaGetLastError());
  int bad = 0;
  SCUDA(h, cudaMemcpyAsync(&bad, h->R.bad, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  SCUDA(h, cudaStreamSynchronize(h->stream));
  if (bad_row) *bad_row = bad == kBadNone ? -1 : bad;
  return bad == kBadNone ? DLMPC_OK : DLMPC_ROW_INFEASIBLE;
}

int dlmpc_sched_stage(dlmpc_sched* h, int stage, int64_t lo, int64_t hi) {
  if (!h) return sfail(h, DLMPC_BAD_ARGUMENT, "null handle");
  sched::RefDev& R = h->R;
  const bool rows = stage == DLMPC_STAGE_PHI_ROWS || stage == DLMPC_STAGE_PHI_ROWS_PADDED;
  const long long n_items = rows ? R.n_rows : (stage == DLMPC_STAGE_LAMBDA_ELEMS ? R.n_elems : R.n_cols);
  if (lo < 0 || hi > n_items || lo > hi) return sfail(h, DLMPC_BAD_ARGUMENT, "item range out of bounds");
  if ((stage == DLMPC_STAGE_PATCH_COLS || stage == DLMPC_STAGE_PATCH_COLS_PADDED) && !h->has_patch)
    return sfail(h, DLMPC_BAD_ARGUMENT, "no patch tables");
  cudaSetDevice(h->device);
  const int cols_grid = (int)std::max<long long>(1, std::min<long long>(hi - lo, (long long)h->sm_count * 8));
  switch (stage) {
    case DLMPC_STAGE_PHI_ROWS:
      sched::phi_rows_kernel<false><<<grid_for(hi - lo, 128), 128, 0, h->stream>>>(R, lo, hi, nullptr); break;
    case DLMPC_STAGE_PHI_ROWS_PADDED:
      sched::phi_rows_kernel<true><<<grid_for(hi - lo, 128), 128, 0, h->stream>>>(R, lo, hi, nullptr); break;
    case DLMPC_STAGE_EXCHANGE_PHI:
      sched::exchange_phi_kernel<<<grid_for((long long)R.n_cols * R.d_col, 256), 256, 0, h->stream>>>(R); break;
    case DLMPC_STAGE_PSI_COLS:
      sched::psi_cols_kernel<<<cols_grid, 256, h->smem_psi, h->stream>>>(R, (int)lo, (int)hi); break;
    case DLMPC_STAGE_LAMBDA_COLS:
      sched::lambda_cols_kernel<<<cols_grid, 128, 0, h->stream>>>(R, (int)lo, (int)hi); break;
    case DLMPC_STAGE_LAMBDA_ELEMS:
      sched::lambda_elems_kernel<<<grid_for(hi - lo, 256), 256, 0, h->stream>>>(R, lo, hi); break;
    case DLMPC_STAGE_CONV_COLS:
      sched::conv_cols_kernel<<<cols_grid, 128, 0, h->stream>>>(R, (int)lo, (int)hi); break;
    case DLMPC_STAGE_EXCHANGE_PSI_LAM:
      sched::exchange_psi_lam_kernel<<<grid_for((long long)R.n_rows * R.d_row, 256), 256, 0, h->stream>>>(R); break;
    case DLMPC_STAGE_FUSED_COLS:
      sched::fused_cols_kernel<<<cols_grid, 256, h->smem_psi, h->stream>>>(R, (int)lo, (int)hi); break;
    case DLMPC_STAGE_PATCH_COLS:
      sched::patch_cols_kernel<false><<<cols_grid, 256, h->smem_psi, h->stream>>>(R, (int)lo, (int)hi); break;
    case DLMPC_STAGE_PATCH_COLS_PADDED:
      sched::patch_cols_kernel<true><<<cols_grid, 256, h->smem_psi, h->stream>>>(R, (int)lo, (int)hi); break;
    default:
      return sfail(h, DLMPC_BAD_ARGUMENT, "unknown stage");
  }
  SCUDA(h, cudaGetLastError());
  return DLMPC_OK;
}

int dlmpc_sched_sync(dlmpc_sched* h) {
  if (!h) return sfail(h, DLMPC_BAD_ARGUMENT, "null handle");
  cudaSetDevice(h->device);
  SCUDA(h, cudaStreamSynchronize(h->stream));
  return DLMPC_OK;
}

int dlmpc_sched_read_residuals(dlmpc_sched* h, double* pri_dual) {
  if (!h || !pri_dual) return sfail(h, DLMPC_BAD_ARGUMENT, "null argument");
  cudaSetDevice(h->device);
  unsigned long long bits[2];
  SCUDA(h, cudaMemcpyAsync(bits, h->R.resid, sizeof(bits), cudaMemcpyDeviceToHost, h->stream));
  SCUDA(h, cudaMemsetAsync(h->R.resid, 0, sizeof(bits), h->stream));
  SCUDA(h, cudaStreamSynchronize(h->stream));
  std::memcpy(pri_dual, bits, sizeof(bits));   // the ordered bits are the doubles' own patterns
  return DLMPC_OK;
}

int dlmpc_sched_phi_compute(dlmpc_sched* h, int64_t lo, int64_t hi, double* out_host) {
  if (!h || !out_host) return sfail(h, DLMPC_BAD_ARGUMENT, "null argument");
  if (lo < 0 || hi > h->R.n_rows || lo > hi) return sfail(h, DLMPC_BAD_ARGUMENT, "row range out of bounds");
  cudaSetDevice(h->device);
  const size_t n = (size_t)h->R.n_rows * h->R.d_row;
  if (!h->d_out) {
    SCUDA(h, cudaMalloc(&h->d_out, n * sizeof(double)));
    h->out_cap = n;
  }
  sched::phi_rows_kernel<false><<<grid_for(hi - lo, 128), 128, 0, h->stream>>>(h->R, lo, hi, h->d_out);
  SCUDA(h, cudaGetLastError());
  const size_t off = (size_t)lo * h->R.d_row, cnt = (size_t)(hi - lo) * h->R.d_row;
  SCUDA(h, cudaMemcpyAsync(out_host, h->d_out + off, cnt * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  SCUDA(h, cudaStreamSynchronize(h->stream));
  return DLMPC_OK;
}

int dlmpc_sched_swap_rows(dlmpc_sched* h) {
  if (!h) return sfail(h, DLMPC_BAD_ARGUMENT, "null handle");
  std::swap(h->R.psi_r, h->R.psi_r_nx);
  std::swap(h->R.lam_r, h->R.lam_r_nx);
  return DLMPC_OK;
}

int dlmpc_op_phi_rows(int device, int n, int d, const int32_t* len, const double* a, const double* v,
                      const double* ada, const double* w, const double* lo, const double* hi, double rho,
                      double* out) {
  if (n < 0 || d < 1 || !len || !a || !v || !ada || !w || !lo || !hi || !out)
    return sfail(nullptr, DLMPC_BAD_ARGUMENT, "bad argument");
  if (n == 0) return DLMPC_OK;
  if (int rc = op_begin(device)) return rc;
  OpBufs B;
  const size_t nd = (size_t)n * d;
  int* dl = B.up(len, n); double* da = B.up(a, nd); double* dv = B.up(v, nd); double* dd = B.up(ada, n);
  double* dw = B.up(w, n); double* dlo = B.up(lo, n); double* dhi = B.up(hi, n); double* dout = B.up<double>(nullptr, nd);
  if (!dl || !da || !dv || !dd || !dw || !dlo || !dhi || !dout) return sfail(nullptr, DLMPC_CUDA_ERROR, "operator buffers");
  sched::op_phi_rows_kernel<<<grid_for(n, 128), 128>>>(n, d, dl, da, dv, dd, dw, dlo, dhi, rho, dout);
  return op_end(out, dout, nd);
}

int dlmpc_op_psi_cols(int device, int n, int m, int s, const double* g, const double* P, const double* rhs,
                      const double* k, double* out) {
  if (n < 0 || m < 1 || s < 1 || !g || !P || !rhs || !k || !out) return sfail(nullptr, DLMPC_BAD_ARGUMENT, "bad argument");
  if (n == 0) return DLMPC_OK;
  if (int rc = op_begin(device)) return rc;
  if ((size_t)m * 8 > 200 * 1024) return sfail(nullptr, DLMPC_BAD_ARGUMENT, "too many constraint rows");
  OpBufs B;
  double* dg = B.up(g, (size_t)n * m * s); double* dp = B.up(P, (size_t)n * s * m);
  double* dr = B.up(rhs, (size_t)n * m); double* dk = B.up(k, (size_t)n * s); double* dout = B.up<double>(nullptr, (size_t)n * s);
  if (!dg || !dp || !dr || !dk || !dout) return sfail(nullptr, DLMPC_CUDA_ERROR, "operator buffers");
  const int smem = m * 8;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(reinterpret_cast<const void*>(sched::op_psi_cols_kernel), cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  sched::op_psi_cols_kernel<<<std::min(n, 148 * 8), 256, smem>>>(n, m, s, dg, dp, dr, dk, dout);
  return op_end(out, dout, (size_t)n * s);
}

int dlmpc_op_lambda(int device, int64_t n, const double* lam, const double* phi, const double* psi, double* out) {
  if (n < 0 || !lam || !phi || !psi || !out) return sfail(nullptr, DLMPC_BAD_ARGUMENT, "bad argument");
  if (n == 0) return DLMPC_OK;
  if (int rc = op_begin(device)) return rc;
  OpBufs B;
  double* dl = B.up(lam, n); double* df = B.up(phi, n); double* ds = B.up(psi, n); double* dout = B.up<double>(nullptr, n);
  if (!dl || !df || !ds || !dout) return sfail(nullptr, DLMPC_CUDA_ERROR, "operator buffers");
  sched::op_lambda_kernel<<<grid_for(n, 256), 256>>>(n, dl, df, ds, dout);
  return op_end(out, dout, n);
}

int dlmpc_op_residuals(int device, int n, int d, const int32_t* len, const double* phi, const double* psi,
                       const double* prev, double rho, double* out2) {
  if (n < 0 || d < 1 || !len || !phi || !psi || !prev || !out2) return sfail(nullptr, DLMPC_BAD_ARGUMENT, "bad argument");
  if (n == 0) return DLMPC_OK;
  if (int rc = op_begin(device)) return rc;
  OpBufs B;
  const size_t nd = (size_t)n * d;
  int* dl = B.up(len, n); double* df = B.up(phi, nd); double* ds = B.up(psi, nd); double* dp = B.up(prev, nd);
  double* dout = B.up<double>(nullptr, 2 * (size_t)n);
  if (!dl || !df || !ds || !dp || !dout) return sfail(nullptr, DLMPC_CUDA_ERROR, "operator buffers");
  sched::op_residuals_kernel<<<grid_for(n, 128), 128>>>(n, d, dl, df, ds, dp, rho, dout);
  return op_end(out2, dout, 2 * (size_t)n);
}

int dlmpc_op_row_dots(int device, int n, int d, const int32_t* len, const double* vals, const int64_t* idx,
                      int64_t n_x, const double* x, double* out) {
  if (n < 0 || d < 1 || n_x < 0 || !len || !vals || !idx || !x || !out) return sfail(nullptr, DLMPC_BAD_ARGUMENT, "bad argument");
  if (n == 0) return DLMPC_OK;
  for (size_t q = 0; q < (size_t)n * d; ++q)
    if (q % d < (size_t)len[q / d] && (idx[q] < 0 || idx[q] >= n_x)) return sfail(nullptr, DLMPC_BAD_ARGUMENT, "index out of range");
  if (int rc = op_begin(device)) return rc;
  OpBufs B;
  const size_t nd = (size_t)n * d;
  int* dl = B.up(len, n); double* dv = B.up(vals, nd);
  long long* di = B.up(reinterpret_cast<const long long*>(idx), nd); double* dx = B.up(x, n_x);
  double* dout = B.up<double>(nullptr, n);
  if (!dl || !dv || !di || !dx || !dout) return sfail(nullptr, DLMPC_CUDA_ERROR, "operator buffers");
  sched::op_row_dots_kernel<<<grid_for(n, 128), 128>>>(n, d, dl, dv, di, dx, dout);
  return op_end(out, dout, n);
}

int dlmpc_op_plant_step(int device, int n_x, int n_u, const int64_t* a_ptr, const int32_t* a_idx, const double* a_val,
                        const int64_t* b_ptr, const int32_t* b_idx, const double* b_val, const double* x,
                        const double* u, double* out) {
  if (n_x < 0 || n_u < 0 || !a_ptr || !b_ptr || !x || !out || (n_u > 0 && !u)) return sfail(nullptr, DLMPC_BAD_ARGUMENT, "bad argument");
  if (n_x == 0) return DLMPC_OK;
  if (int rc = op_begin(device)) return rc;
  OpBufs B;
  const size_t na = (size_t)a_ptr[n_x], nb = (size_t)b_ptr[n_x];
  long long* ap = B.up(reinterpret_cast<const long long*>(a_ptr), n_x + 1); int* ai = B.up(a_idx, na); double* av = B.up(a_val, na);
  long long* bp = B.up(reinterpret_cast<const long long*>(b_ptr), n_x + 1); int* bi = B.up(b_idx, nb); double* bv = B.up(b_val, nb);
  double* dx = B.up(x, n_x); double* du = B.up(u, n_u); double* dout = B.up<double>(nullptr, n_x);
  if (!ap || !ai || !av || !bp || !bi || !bv || !dx || !du || !dout) return sfail(nullptr, DLMPC_CUDA_ERROR, "operator buffers");
  sched::op_plant_kernel<<<grid_for(n_x, 128), 128>>>(n_x, ap, ai, av, bp, bi, bv, dx, du, dout);
  return op_end(out, dout, n_x);
}

}  // extern "C"
