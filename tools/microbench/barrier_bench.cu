// Grid barrier latency on B200, 148 CTAs x 512 threads (the persistent
// kernel's shape): cooperative groups grid.sync vs a monotonic-counter
// barrier (bar.sync; one red.release.gpu per CTA; ld.acquire.gpu polling
// until the counter reaches epoch * grid; bar.sync).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench/barrier_bench tools/microbench/barrier_bench.cu
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

__global__ void cg_kernel(int iters, int* sink) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) g.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = iters;
}

__global__ void mono_kernel(int iters, unsigned* ctr, int* sink) {
  for (int i = 1; i <= iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      red_release_add(ctr, 1u);
      const unsigned target = static_cast<unsigned>(i) * gridDim.x;
      while (ld_acquire(ctr) < target) { }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = iters;
}

// same, but the polling thread re-reads with ld.relaxed + a final acquire fence
__global__ void mono_relaxed_kernel(int iters, unsigned* ctr, int* sink) {
  for (int i = 1; i <= iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      red_release_add(ctr, 1u);
      const unsigned target = static_cast<unsigned>(i) * gridDim.x;
      unsigned v;
      do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory"); } while (v < target);
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = iters;
}

// K counters in different L2 lines (CTA b arrives on counter b % K): the
// same-address atomics of 148 CTAs serialise in one L2 slice; warp 0's first
// K lanes poll one counter each until it holds its share of the arrivals.
template <int K>
__global__ void spread_kernel(int iters, unsigned* ctr, int* sink) {
  const int lane = threadIdx.x & 31;
  for (int i = 1; i <= iters; ++i) {
    __syncthreads();
    if (threadIdx.x < 32) {
      if (lane == 0) red_release_add(ctr + (blockIdx.x % K) * 64, 1u);
      if (lane < K) {
        const unsigned share = gridDim.x / K + (lane < static_cast<int>(gridDim.x % K) ? 1u : 0u);
        const unsigned target = static_cast<unsigned>(i) * share;
        while (ld_acquire(ctr + lane * 64) < target) { }
      }
      __syncwarp();
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = iters;
}

// lower bound: no release / acquire at all (not a valid barrier for data)
__global__ void relaxed_kernel(int iters, unsigned* ctr, int* sink) {
  for (int i = 1; i <= iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" :: "l"(ctr) : "memory");
      const unsigned target = static_cast<unsigned>(i) * gridDim.x;
      unsigned v;
      do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory"); } while (v < target);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = iters;
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int* sink; unsigned* ctr; CK(cudaMalloc(&sink, 4)); CK(cudaMalloc(&ctr, 4 * 64 * 32));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    for (int which = 0; which < 7; ++which) {
      CK(cudaMemset(ctr, 0, 4 * 64 * 32));
      int it = iters;
      void* a0[] = {&it, &sink};
      void* a1[] = {&it, &ctr, &sink};
      void* fn = which == 0 ? (void*)cg_kernel : which == 1 ? (void*)mono_kernel : which == 2 ? (void*)mono_relaxed_kernel
               : which == 3 ? (void*)spread_kernel<4> : which == 4 ? (void*)spread_kernel<8> : which == 5 ? (void*)spread_kernel<16> : (void*)relaxed_kernel;
      cudaEventRecord(e0);
      CK(cudaLaunchCooperativeKernel(fn, sms, 512, which == 0 ? a0 : a1, 0, 0));
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const char* nm[7] = {"cg grid.sync", "monotonic red+acquire", "monotonic red+relaxed poll", "4 counters", "8 counters", "16 counters", "relaxed (no ordering)"};
      printf("%-28s %d CTAs x 512: %.3f us/barrier\n", nm[which], sms, ms * 1e3 / iters);
    }
  }
  return 0;
}
