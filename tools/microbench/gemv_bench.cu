// Small-chunk (1-2 columns) Ψ projection: DMMA GEMMs (TC=8, as the patch
// kernel runs C2) vs DFMA GEMVs on an operator stored with an odd leading
// dimension (conflict-free row walks). One CTA of 512 threads per SM.
#include <cstdio>
#include "dlmpc_device.cuh"
using namespace dlmpc;

constexpr int TC = 8;
constexpr int S = 203, N0 = 47, S8 = 208, S4 = 204, N08 = 48;

// Y[a][t] = sum_p N[p][a] K[t][p]; 5-way p split, partials reduced in smem
__device__ __forceinline__ void gemv1(const double* nop, int ldo, const double* kt, int ldk, double* part,
                                      double* yb, int ldy, int nt) {
  constexpr int PS = 5, PL = (S + PS - 1) / PS;
  const int tid = threadIdx.x;
  const int a = tid % 48, rest = tid / 48;           // 48 x (t, ps) = 480 threads
  const int t = rest % 2, ps = rest / 2;
  if (rest < 2 * PS && a < N0 && t < nt) {
    const int p0 = ps * PL, p1 = min(S, p0 + PL);
    double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
    const double* kr = kt + t * ldk;
    int p = p0;
#pragma unroll 2
    for (; p + 3 < p1; p += 4) {
      c0 = fma(nop[p * ldo + a], kr[p], c0);
      c1 = fma(nop[(p + 1) * ldo + a], kr[p + 1], c1);
      c2 = fma(nop[(p + 2) * ldo + a], kr[p + 2], c2);
      c3 = fma(nop[(p + 3) * ldo + a], kr[p + 3], c3);
    }
    for (; p < p1; ++p) c0 = fma(nop[p * ldo + a], kr[p], c0);
    c0 = (c0 + c1) + (c2 + c3);
    part[(ps * 2 + t) * 48 + a] = c0;
  }
  __syncthreads();
  if (tid < 48 * 2) {
    const int aa = tid % 48, tt = tid / 48;
    double v = 0.0;
    if (aa < N0 && tt < nt)
      for (int q = 0; q < PS; ++q) v += part[(q * 2 + tt) * 48 + aa];
    yb[aa * ldy + tt] = v;
  }
  __syncthreads();
}

// O[t][p] = sum_a N[p][a] Y[a][t]: thread per (p, t) pair-of-columns
__device__ __forceinline__ void gemv2(const double* nop, int ldo, const double* yb, int ldy, double* kt, int ldk,
                                      int nt) {
  const int p = threadIdx.x;
  if (p < S) {
    double o0a = 0.0, o0b = 0.0, o1a = 0.0, o1b = 0.0, o0c = 0.0, o1c = 0.0, o0d = 0.0, o1d = 0.0;
    const double* row = nop + p * ldo;
    int a = 0;
#pragma unroll 3
    for (; a + 3 < N0; a += 4) {
      const double n0v = row[a], n1v = row[a + 1], n2v = row[a + 2], n3v = row[a + 3];
      o0a = fma(n0v, yb[a * ldy], o0a);       o1a = fma(n0v, yb[a * ldy + 1], o1a);
      o0b = fma(n1v, yb[(a + 1) * ldy], o0b); o1b = fma(n1v, yb[(a + 1) * ldy + 1], o1b);
      o0c = fma(n2v, yb[(a + 2) * ldy], o0c); o1c = fma(n2v, yb[(a + 2) * ldy + 1], o1c);
      o0d = fma(n3v, yb[(a + 3) * ldy], o0d); o1d = fma(n3v, yb[(a + 3) * ldy + 1], o1d);
    }
    for (; a < N0; ++a) { o0a = fma(row[a], yb[a * ldy], o0a); o1a = fma(row[a], yb[a * ldy + 1], o1a); }
    o0a = (o0a + o0b) + (o0c + o0d); o1a = (o1a + o1b) + (o1c + o1d);
    o0b = 0.0; o1b = 0.0;
    kt[p] = o0a + o0b;
    if (nt > 1) kt[ldk + p] = o1a + o1b;
  }
  __syncthreads();
}

template <int WHICH>
__global__ void __launch_bounds__(kThreads, 1) bench(DevProblem P, int ldo, int reps, double* sink) {
  extern __shared__ __align__(16) double smem[];
  const int ldn = P.class_ldn[0];
  double* nop = smem;
  double* kt = smem + P.off_k;
  double* yb = smem + P.off_y;
  double* yp = smem + P.off_yp;
  for (int i = threadIdx.x; i < P.off_k; i += kThreads) nop[i] = 1e-3 * ((i * 37) % 101);
  for (int i = threadIdx.x; i < TC * P.ldk; i += kThreads) kt[i] = 1e-3 * ((i * 53) % 97);
  for (int i = threadIdx.x; i < N08 * P.ldy; i += kThreads) yb[i] = 1e-3 * ((i * 29) % 89);
  __syncthreads();
  for (int r = 0; r < reps; ++r) {
    if (WHICH == 1) gemm1<TC>(P, S8, N08, ldn, nop, kt, P.ldk, yb, P.ldy, yp);
    if (WHICH == 2) { StoreO epi{kt, P.ldk}; gemm2<TC>(S8, N08, ldn, nop, yb, P.ldy, epi); __syncthreads(); }
    if (WHICH == 3) gemv1(nop, ldo, kt, P.ldk, yp, yb, P.ldy, 2);
    if (WHICH == 4) gemv2(nop, ldo, yb, P.ldy, kt, P.ldk, 2);
  }
  if (kt[threadIdx.x] == 12345.0) sink[0] = 1.0;
}

int ld_frag(int n) { int ld = n; while (ld % 16 != 4 && ld % 16 != 12) ++ld; return ld; }

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* sink; cudaMalloc(&sink, 8);
  DevProblem P{};
  int* cls_ldn; cudaMalloc(&cls_ldn, 4);
  const int ldn = ld_frag(N08);
  cudaMemcpy(cls_ldn, &ldn, 4, cudaMemcpyHostToDevice);
  P.class_ldn = cls_ldn;
  P.ldk = ld_frag(S8); P.ldy = ld_frag(TC); P.split_max = 4; P.n08_max = N08;
  P.off_k = S8 * 52; P.off_y = P.off_k + TC * P.ldk; P.off_yp = P.off_y + N08 * P.ldy;
  const int smem = (P.off_yp + 4 * N08 * TC + 1024) * 8;
  const int reps = 4000;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[5] = {"", "DMMA GEMM1 (split-K)", "DMMA GEMM2", "DFMA GEMV1 ldo=49", "DFMA GEMV2 ldo=49"};
  for (int which = 1; which <= 4; ++which) {
    auto fn = which == 1 ? bench<1> : which == 2 ? bench<2> : which == 3 ? bench<3> : bench<4>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    fn<<<sms, kThreads, smem>>>(P, 49, 10, sink);
    cudaEventRecord(e0);
    fn<<<sms, kThreads, smem>>>(P, 49, reps, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-24s %.3f us/call  (%s)\n", names[which], 1e3 * ms / reps, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
