// Microbenchmarks that size the design of the DLMPC persistent kernel on B200:
//  (1) FP64 DFMA throughput on CUDA cores, (2) FP64 DMMA (mma.sync m8n8k4 f64)
//  throughput, (3) grid-barrier latency (cooperative groups vs. a hand-rolled
//  sense-reversing barrier), (4) cluster barrier latency.
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double r[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) r[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i] = fma(r[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += r[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void cg_barrier_kernel(int iters, int* sink) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) g.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = iters;
}

// Hand-rolled barrier: one arrival counter + generation word.
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__global__ void my_barrier_kernel(int iters, unsigned* bar, int* sink) {
  unsigned nb = gridDim.x;
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned gen = ld_acquire(bar + 1);
      unsigned arrived;
      asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(arrived) : "l"(bar) : "memory");
      if (arrived == nb - 1) {
        bar[0] = 0;
        asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(bar + 1), "r"(gen + 1) : "memory");
      } else {
        while (ld_acquire(bar + 1) == gen) { }
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = iters;
}

__global__ void __cluster_dims__(16, 1, 1) cluster_barrier_kernel(int iters, int* sink) {
  cg::cluster_group cl = cg::this_cluster();
  for (int i = 0; i < iters; ++i) cl.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = iters;
}

int main() {
  int dev = 0; cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  printf("device %s SMs %d clock %d kHz smemOptin %zu\n", prop.name, prop.multiProcessorCount, prop.clockRate, prop.sharedMemPerBlockOptin);
  double* out; CK(cudaMalloc(&out, 64)); int* sink; CK(cudaMalloc(&sink, 64));
  unsigned* bar; CK(cudaMalloc(&bar, 64)); CK(cudaMemset(bar, 0, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = prop.multiProcessorCount;
  // DFMA
  for (int bps : {4, 8}) {
    int iters = 20000; int blocks = sms * bps, threads = 256;
    dfma_kernel<<<blocks, threads>>>(out, 100, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flop = 2.0 * 8 * iters * (double)blocks * threads;
    printf("DFMA blocks/SM %d: %.2f TFLOP/s (%.3f ms)\n", bps, flop / ms / 1e9, ms);
  }
  for (int bps : {4, 8}) {
    int iters = 5000; int blocks = sms * bps, threads = 256;
    dmma_kernel<<<blocks, threads>>>(out, 100);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); dmma_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flop = 2.0 * 256 * 8 * iters * (double)blocks * (threads / 32);
    printf("DMMA m8n8k4 blocks/SM %d: %.2f TFLOP/s (%.3f ms)\n", bps, flop / ms / 1e9, ms);
  }
  // barriers
  for (int nblk : {16, 74, 148}) {
    int iters = 2000;
    void* args[] = {&iters, &sink};
    CK(cudaLaunchCooperativeKernel((void*)cg_barrier_kernel, nblk, 256, args, 0, 0));
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    CK(cudaLaunchCooperativeKernel((void*)cg_barrier_kernel, nblk, 256, args, 0, 0));
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("cg grid.sync blocks %d: %.3f us/barrier\n", nblk, ms * 1e3 / iters);
    void* args2[] = {&iters, &bar, &sink};
    CK(cudaLaunchCooperativeKernel((void*)my_barrier_kernel, nblk, 256, args2, 0, 0));
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    CK(cudaLaunchCooperativeKernel((void*)my_barrier_kernel, nblk, 256, args2, 0, 0));
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("hand barrier blocks %d: %.3f us/barrier\n", nblk, ms * 1e3 / iters);
  }
  {
    int iters = 20000;
    cluster_barrier_kernel<<<16, 256>>>(iters, sink); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); cluster_barrier_kernel<<<16, 256>>>(iters, sink); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("cluster(16) sync: %.3f us/barrier\n", ms * 1e3 / iters);
  }
  // launch latency
  {
    int iters = 2000;
    cudaEventRecord(e0);
    for (int i = 0; i < iters; ++i) dfma_kernel<<<sms, 256>>>(out, 1, 1.0, 0.0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("back-to-back tiny launches: %.3f us/launch\n", ms * 1e3 / iters);
  }
  return 0;
}
