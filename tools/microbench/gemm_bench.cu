// Microbenchmark of the Ψ-projection GEMMs of dlmpc_device.cuh on one chunk
// resident in shared memory (class shape S=203, n0=47 or 55; TC=16), one CTA
// of 512 threads per SM, REPS back-to-back calls. Prints achieved FP64 rate.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2103_14990_b200/csrc gemm_bench.cu
#include <cstdio>
#include "dlmpc_device.cuh"
using namespace dlmpc;

constexpr int TC = 16;


// V1: per-column metadata hoisted into registers once per GEMM-2 call
template <int TC, bool DUAL, bool GSTORE = true>
struct EpiV1 {
  static constexpr int NTN = TC / 8;
  double* psi_n; double* lam_n; const double* q_pool;
  const long long* m_pos; const long long* m_s; const long long* m_q; const double* m_x;
  const double* s_patch; const double* kt; double* lt; int ldk, S, nt;
  double pri_m, dual_m;
  double qv[kMG2][NTN][2];
  long long cpos[NTN][2]; int cs0[NTN][2]; double cx[NTN][2];
  bool init = false;
  __device__ __forceinline__ void prefetch(int m, int mt) {
    const int lane = threadIdx.x & 31, g = lane >> 2, tig = lane & 3;
    if (!init) {
      init = true;
#pragma unroll
      for (int nn = 0; nn < NTN; ++nn)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int t = nn * 8 + 2 * tig + e;
          cpos[nn][e] = m_pos[t]; cs0[nn][e] = (int)m_s[t]; cx[nn][e] = m_x[t];
        }
    }
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
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int t = nn * 8 + 2 * tig + e;
      if (p < S && t < nt) {
        const double kv = kt[t * ldk + p], lm = lt[t * ldk + p];
        const double pn = qv[m][nn][e] + (e ? c1 : c0);
        const double ln = __dsub_rn(kv, pn);
        if (GSTORE) {
          psi_n[cpos[nn][e] + p] = pn;
          lam_n[cpos[nn][e] + p] = ln;
        } else {
          dual_m += pn * ln;
        }
        pri_m = fmax(pri_m, fabs(__dsub_rn(ln, lm)));
        if (DUAL) {
          const double ps = fma(-s_patch[cs0[nn][e] + p], cx[nn][e], kv);
          dual_m = fmax(dual_m, fabs(__dsub_rn(pn, ps)));
        }
        lt[t * ldk + p] = __dsub_rn(pn, ln);
      }
    }
  }
};

template <int WHICH>
__global__ void __launch_bounds__(kThreads, 1) bench(DevProblem P, int S, int n0, int reps, double* sink,
                                                     double* gout, const double* qpool) {
  extern __shared__ __align__(16) double smem[];
  const int S8 = (S + 7) & ~7, n08 = (n0 + 7) & ~7;
  const int ldn = P.class_ldn[0];
  double* nop = smem;
  double* kt = smem + P.off_k;
  double* yb = smem + P.off_y;
  double* yp = smem + P.off_yp;
  for (int i = threadIdx.x; i < P.off_k; i += kThreads) nop[i] = 1e-3 * ((i * 37) % 101);
  for (int i = threadIdx.x; i < TC * P.ldk; i += kThreads) kt[i] = 1e-3 * ((i * 53) % 97);
  for (int i = threadIdx.x; i < n08 * P.ldy; i += kThreads) yb[i] = 1e-3 * ((i * 29) % 89);
  __syncthreads();
  double acc = 0.0;
  for (int r = 0; r < reps; ++r) {
    if (WHICH == 1) {
      gemm1<TC>(P, S8, n08, ldn, nop, kt, P.ldk, yb, P.ldy, yp);
    } else if (WHICH >= 3) {
      // GEMM 2 + the stream kernel's fused epilogue (stores into a per-CTA
      // global slab, λ/v' buffer and metadata in shared memory)
      double* lt = smem + P.off_yp + 4 * n08 * TC;
      double* s_patch = lt + TC * P.ldk;
      long long* m_pos = reinterpret_cast<long long*>(s_patch + 512);
      long long* m_s = m_pos + TC; long long* m_q = m_pos + 2 * TC;
      double* m_x = reinterpret_cast<double*>(m_pos + 3 * TC);
      if (r == 0) {
        for (int i = threadIdx.x; i < TC * P.ldk; i += kThreads) lt[i] = 1e-3 * (i % 91);
        for (int i = threadIdx.x; i < 512; i += kThreads) s_patch[i] = 1e-3 * (i % 83);
        if (threadIdx.x < TC) {
          const int t = threadIdx.x;
          m_pos[t] = (long long)(blockIdx.x * TC + t) * 204; m_s[t] = (t / 2) * 29; m_q[t] = (t & 1) * 204;
          m_x[t] = 0.5 + 0.01 * t;
        }
        __syncthreads();
      }
      if (WHICH == 3) {
        StreamEpi<TC> epi{gout, gout + (size_t)gridDim.x * TC * 204, qpool, m_pos, m_s, m_q, m_x,
                          s_patch, kt, lt, P.ldk, S, TC, 0.0, 0.0};
        gemm2<TC>(S8, n08, ldn, nop, yb, P.ldy, epi);
        acc += epi.pri_m + epi.dual_m;
      } else if (WHICH == 4) {
        EpiV1<TC, true> epi{gout, gout + (size_t)gridDim.x * TC * 204, qpool, m_pos, m_s, m_q, m_x,
                            s_patch, kt, lt, P.ldk, S, TC, 0.0, 0.0};
        gemm2<TC>(S8, n08, ldn, nop, yb, P.ldy, epi);
        acc += epi.pri_m + epi.dual_m;
      } else if (WHICH == 5) {
        EpiV1<TC, true, false> epi{gout, gout + (size_t)gridDim.x * TC * 204, qpool, m_pos, m_s, m_q, m_x,
                             s_patch, kt, lt, P.ldk, S, TC, 0.0, 0.0};
        gemm2<TC>(S8, n08, ldn, nop, yb, P.ldy, epi);
        acc += epi.pri_m + epi.dual_m;
      }
      __syncthreads();
    } else {
      StoreO epi{kt, P.ldk};
      gemm2<TC>(S8, n08, ldn, nop, yb, P.ldy, epi);
      __syncthreads();
    }
  }
  acc = kt[threadIdx.x] + yb[threadIdx.x];
  if (acc == 12345.0) sink[0] = acc;
}

int ld_frag(int n) { int ld = n; while (ld % 16 != 4) ++ld; return ld; }

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* sink; cudaMalloc(&sink, 8);
  double* gout; cudaMalloc(&gout, sizeof(double) * 2 * 148 * 16 * 204);
  double* qpool; cudaMalloc(&qpool, sizeof(double) * 2 * 204);
  cudaMemset(qpool, 0, sizeof(double) * 2 * 204);
  for (int n0 : {47}) {
    for (int split_max : {1}) {
      const int S = 203, S8 = 208, n08 = (n0 + 7) & ~7;
      DevProblem P{};
      int* cls_ldn; cudaMalloc(&cls_ldn, 4);
      const int ldn = ld_frag(n08);
      cudaMemcpy(cls_ldn, &ldn, 4, cudaMemcpyHostToDevice);
      P.class_ldn = cls_ldn;
      P.ldk = ld_frag(S8); P.ldy = ld_frag(TC); P.split_max = split_max; P.n08_max = n08;
      P.off_k = S8 * ldn; P.off_y = P.off_k + TC * P.ldk; P.off_yp = P.off_y + n08 * P.ldy;
      const int smem = (P.off_yp + 4 * n08 * TC + TC * P.ldk + 512 + 4 * TC) * 8;
      const int reps = 2000;
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      for (int which : {1, 2, 3, 4, 5}) {
        auto fn = which == 1 ? bench<1> : which == 2 ? bench<2> : which == 3 ? bench<3> : which == 4 ? bench<4> : bench<5>;
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        fn<<<sms, kThreads, smem>>>(P, S, n0, 10, sink, gout, qpool);
        cudaEventRecord(e0);
        fn<<<sms, kThreads, smem>>>(P, S, n0, reps, sink, gout, qpool);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double flop = 2.0 * n0 * S * TC * (double)reps * sms;
        printf("n0=%d split_max=%d GEMM%d: %.3f us/call  %.2f TFLOP/s (useful)  err=%s\n", n0, split_max, which,
               1e3 * ms / reps, flop / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
      }
      cudaFree(cls_ldn);
    }
  }
  return 0;
}
