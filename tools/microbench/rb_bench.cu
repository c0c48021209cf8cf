// Small-chunk (<= 2 columns) Ψ projection, C2 interior class (S=203, n0=47):
// the patch kernel's DFMA GEMV 1 + DMMA GEMM 2 vs the register-blocked GEMV
// pair (gemv_pair_rb). One CTA of 512 threads per SM, clock64 per call; the
// outputs are checked against a CPU double loop.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2103_14990_b200/csrc \
//        -o tools/microbench/rb_bench tools/microbench/rb_bench.cu
#include <cstdio>
#include <cmath>
#include <vector>
#include "dlmpc_device.cuh"
using namespace dlmpc;

constexpr int TC = 8;
constexpr int RB_AL = 3;   // the microbenchmark's fixed blocking (the kernel uses RB_AL_MAX)
constexpr int S = 203, N0 = 47, S8 = 208, N08 = 48;

struct KtRead {
  const double* kt; int ldk;
  __device__ __forceinline__ double operator()(int t, int p) const { return kt[t * ldk + p]; }
};
struct StoreOut {
  double* out;
  __device__ __forceinline__ void operator()(int p, int t, double o) const { out[t * S8 + p] = o; }
};


template <int STAGE, class Epi>
__device__ __forceinline__ void rb_staged(int S, const double (&op)[RB_PL][RB_AL], const double* kt, int ldk,
                                          double* ypart, double* yb2, int nt, const Epi& epi) {
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31, h = l >> 4, j = l & 15;
  const int PB = (((S + 7) & ~7) + 15) >> 4;
  const int prow0 = w * PB + h * RB_PL;
  const int nrow = max(0, min(RB_PL, min(PB - h * RB_PL, S - prow0)));
  double y0[RB_AL], y1[RB_AL];
#pragma unroll
  for (int c = 0; c < RB_AL; ++c) { y0[c] = 0.0; y1[c] = 0.0; }
#pragma unroll
  for (int i = 0; i < RB_PL; ++i) {
    const double k0 = i < nrow ? kt[prow0 + i] : 0.0;
    const double k1 = i < nrow ? kt[ldk + prow0 + i] : 0.0;
#pragma unroll
    for (int c = 0; c < RB_AL; ++c) { y0[c] = fma(op[i][c], k0, y0[c]); y1[c] = fma(op[i][c], k1, y1[c]); }
  }
  if (STAGE == 1) { for (int c = 0; c < RB_AL; ++c) ypart[tid * 8 + c] = y0[c] + y1[c]; return; }
#pragma unroll
  for (int c = 0; c < RB_AL; ++c) {
    const double keep = h ? y1[c] : y0[c], send = h ? y0[c] : y1[c];
    ypart[(w * 2 + h) * (16 * RB_AL) + j * RB_AL + c] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
  __syncthreads();
  if (STAGE == 2) return;
  if (tid < 2 * 16 * RB_AL) {
    double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
#pragma unroll
    for (int q = 0; q < kWarps; q += 4) {
      const int t = tid / (16 * RB_AL), a = tid - t * (16 * RB_AL);
      v0 += ypart[((q + 0) * 2 + t) * (16 * RB_AL) + a];
      v1 += ypart[((q + 1) * 2 + t) * (16 * RB_AL) + a];
      v2 += ypart[((q + 2) * 2 + t) * (16 * RB_AL) + a];
      v3 += ypart[((q + 3) * 2 + t) * (16 * RB_AL) + a];
    }
    yb2[tid] = (tid / (16 * RB_AL) < nt) ? (v0 + v1) + (v2 + v3) : 0.0;
  }
  __syncthreads();
  if (STAGE == 3) return;
  double ya[RB_AL], yc[RB_AL];
#pragma unroll
  for (int c = 0; c < RB_AL; ++c) { ya[c] = yb2[j * RB_AL + c]; yc[c] = yb2[16 * RB_AL + j * RB_AL + c]; }
  double v[16];
#pragma unroll
  for (int i = 0; i < RB_PL; ++i) {
    double o0 = 0.0, o1 = 0.0;
#pragma unroll
    for (int c = 0; c < RB_AL; ++c) { o0 = fma(op[i][c], ya[c], o0); o1 = fma(op[i][c], yc[c], o1); }
    v[i] = o0; v[8 + i] = o1;
  }
  if (STAGE == 4) { double a = 0; for (int k = 0; k < 16; ++k) a += (k == 7 || k == 15) ? 0.0 : v[k]; ypart[tid] = a; return; }
  v[7] = 0.0; v[15] = 0.0;
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

template <int WHICH>
__global__ void __launch_bounds__(kThreads, 1) bench(DevProblem P, const double* gop, const double* gk, int reps,
                                                     double* out, unsigned long long* cyc) {
  extern __shared__ __align__(16) double smem[];
  const int ldn = P.class_ldn[0];
  double* nop = smem;
  double* kt = smem + P.off_k;
  double* yb = smem + P.off_y;
  double* yp = smem + P.off_yp;
  for (int i = threadIdx.x; i < S8 * ldn; i += kThreads) nop[i] = gop[i];
  for (int i = threadIdx.x; i < TC * P.ldk; i += kThreads) kt[i] = 0.0;
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * S; i += kThreads) kt[(i / S) * P.ldk + i % S] = gk[i];
  __syncthreads();
  if (WHICH == 2) {   // thread-major copy replaces the [S8][ldn] operator
    P.class_null_off = nullptr;
    __syncthreads();
  }
  double* opT = smem + P.off_yp + 4 * N08 * TC;   // separate region for the thread-major copy
  if (WHICH >= 2) {
    const int tid = threadIdx.x, w = tid >> 5, l = tid & 31, h = l >> 4, j = l & 15;
    const int PB = (S8 + 15) >> 4;
    for (int i = 0; i < RB_PL; ++i)
      for (int c = 0; c < RB_AL; ++c) {
        const int pr = h * RB_PL + i, p = w * PB + pr, a = j * RB_AL + c;
        opT[(i * RB_AL + c) * kThreads + tid] = (pr < PB && p < S && a < N0) ? nop[p * ldn + a] : 0.0;
      }
    __syncthreads();
  }
  double opr[RB_PL][RB_AL];
  if (WHICH >= 3) load_operator_rb<RB_AL>(opT, opr);
  unsigned long long t0 = 0, best = ~0ull;
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    t0 = clock64();
    if (WHICH == 1) {
      gemv1_small<TC>(S, N08, ldn, nop, kt, P.ldk, yp, yb, P.ldy, 2);
      StoreO epi{kt + 2 * P.ldk, P.ldk};   // O into columns 2,3 (K kept)
      gemm2<TC>(S8, N08, ldn, nop, yb, P.ldy, epi);
      __syncthreads();
    } else if (WHICH == 2) {
      double op[RB_PL][RB_AL];
      load_operator_rb<RB_AL>(opT, op);
      gemv_pair_rb<RB_AL>(S, op, KtRead{kt, P.ldk}, yp, yb, 2, StoreOut{kt + 2 * P.ldk});
      __syncthreads();
    } else if (WHICH == 3) {
      gemv_pair_rb<RB_AL>(S, opr, KtRead{kt, P.ldk}, yp, yb, 2, StoreOut{kt + 2 * P.ldk});
      __syncthreads();
    } else {
      rb_staged<WHICH - 3>(S, opr, kt, P.ldk, yp, yb, 2, StoreOut{kt + 2 * P.ldk});
      __syncthreads();
    }
    const unsigned long long dt = clock64() - t0;
    if (dt < best) best = dt;
  }
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < 2 * S; i += kThreads) {
      const int t = i / S, p = i % S;
      out[i] = WHICH == 1 ? kt[(2 + t) * P.ldk + p] : kt[2 * P.ldk + t * S8 + p];
    }
    if (threadIdx.x == 0) cyc[0] = best;
  }
}

int ld_frag(int n) { int ld = n; while (ld % 16 != 4 && ld % 16 != 12) ++ld; return ld; }

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  DevProblem P{};
  int* cls_ldn; cudaMalloc(&cls_ldn, 4);
  const int ldn = ld_frag(N08);
  cudaMemcpy(cls_ldn, &ldn, 4, cudaMemcpyHostToDevice);
  P.class_ldn = cls_ldn;
  P.ldk = ld_frag(S8); P.ldy = ld_frag(TC); P.split_max = 4; P.n08_max = N08;
  P.off_k = S8 * ldn; P.off_y = P.off_k + TC * P.ldk; P.off_yp = P.off_y + N08 * P.ldy;
  const int smem = (P.off_yp + 4 * N08 * TC + RB_PL * RB_AL * kThreads + 64) * 8;
  std::vector<double> op(S8 * ldn, 0.0), k(2 * S);
  for (int p = 0; p < S; ++p) for (int a = 0; a < N0; ++a) op[p * ldn + a] = std::sin(0.37 * p + 1.3 * a) / 7.0;
  for (int i = 0; i < 2 * S; ++i) k[i] = std::cos(0.11 * i);
  std::vector<double> ref(2 * S);
  for (int t = 0; t < 2; ++t) {
    double y[N0];
    for (int a = 0; a < N0; ++a) { y[a] = 0; for (int p = 0; p < S; ++p) y[a] += op[p * ldn + a] * k[t * S + p]; }
    for (int p = 0; p < S; ++p) { double o = 0; for (int a = 0; a < N0; ++a) o += op[p * ldn + a] * y[a]; ref[t * S + p] = o; }
  }
  double *gop, *gk, *out; unsigned long long* cyc;
  cudaMalloc(&gop, op.size() * 8); cudaMalloc(&gk, k.size() * 8); cudaMalloc(&out, 2 * S * 8); cudaMalloc(&cyc, 8);
  cudaMemcpy(gop, op.data(), op.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(gk, k.data(), k.size() * 8, cudaMemcpyHostToDevice);
  const char* names[8] = {"", "GEMV1 DFMA + GEMM2 DMMA (patch kernel today)", "register-blocked GEMV pair",
                          "register-blocked, operator register-resident", "  stage: GEMV1 FMAs", "  stage: + scatter, sync",
                          "  stage: + warp sum, sync", "  stage: + GEMV2 FMAs"};
  for (int which = 1; which <= 7; ++which) {
    auto fn = which == 1 ? bench<1> : which == 2 ? bench<2> : which == 3 ? bench<3> : which == 4 ? bench<4>
            : which == 5 ? bench<5> : which == 6 ? bench<6> : bench<7>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    fn<<<sms, kThreads, smem>>>(P, gop, gk, 200, out, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    std::vector<double> o(2 * S); cudaMemcpy(o.data(), out, 2 * S * 8, cudaMemcpyDeviceToHost);
    double err = 0, mx = 0;
    for (int i = 0; i < 2 * S; ++i) { err = std::fmax(err, std::fabs(o[i] - ref[i])); mx = std::fmax(mx, std::fabs(ref[i])); }
    printf("%-48s best %6llu cycles = %.3f us  rel err %.2e  (%s)\n", names[which], c, c / 1965.0, err / mx,
           cudaGetErrorString(e));
  }
  return 0;
}
