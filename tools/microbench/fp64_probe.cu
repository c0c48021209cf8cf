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

// Cluster barrier: no compile-time cluster shape; the launch sets it
// (cudaLaunchKernelEx + cudaLaunchAttributeClusterDimension). 16-CTA clusters
// are non-portable and need cudaFuncAttributeNonPortableClusterSizeAllowed.
__global__ void cluster_barrier_kernel(int iters, int* sink) {
  cg::cluster_group cl = cg::this_cluster();
  for (int i = 0; i < iters; ++i) cl.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = iters + (int)cl.num_blocks();
}

// Split cluster barrier as a persistent kernel would use it: arrive.release
// by every thread, wait.acquire.
__global__ void cluster_split_barrier_kernel(int iters, int* sink) {
  for (int i = 0; i < iters; ++i) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = iters;
}

// DSMEM round trip: thread 0 of CTA 0 chases a pointer ring that lives in
// the shared memory of CTA `peer` of its cluster (ld.shared::cluster).
__global__ void dsmem_latency_kernel(int iters, int peer, long long* out) {
  __shared__ unsigned ring[256];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) ring[i] = (i * 97 + 13) & 255;
  cl.sync();
  if (cl.block_rank() == 0 && threadIdx.x == 0) {
    unsigned* remote = cl.map_shared_rank(ring, peer);
    unsigned idx = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) idx = remote[idx];
    long long t1 = clock64();
    out[0] = (t1 - t0) / iters;
    out[1] = idx;
  }
  cl.sync();
}

// L2 round trip for comparison: the same chase over a global ring (ld.cg).
__global__ void l2_latency_kernel(const unsigned* ring, int iters, long long* out) {
  unsigned idx = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) idx = __ldcg(ring + idx);
  long long t1 = clock64();
  out[0] = (t1 - t0) / iters;
  out[1] = idx;
}

static cudaError_t launch_cluster(const void* fn, int grid, int block, int cluster, void** args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid); cfg.blockDim = dim3(block); cfg.dynamicSmemBytes = 0; cfg.stream = 0;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr; cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, fn, args);
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
  // cluster barriers (sizes 2..16; 16 is non-portable), one cluster and a
  // full machine of clusters, 512 threads per CTA like the persistent kernel
  CK(cudaFuncSetAttribute((const void*)cluster_barrier_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute((const void*)cluster_split_barrier_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute((const void*)dsmem_latency_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  for (int cs : {2, 4, 8, 16}) {
    for (int full : {0, 1}) {
      int grid = full ? (sms / cs) * cs : cs;
      int iters = 20000;
      void* args[] = {&iters, &sink};
      CK(launch_cluster((const void*)cluster_barrier_kernel, grid, 512, cs, args));
      CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
      int h = 0; CK(cudaMemcpy(&h, sink, 4, cudaMemcpyDeviceToHost));
      if (h != iters + cs) { printf("cluster(%d) kernel did not run (sink %d)\n", cs, h); continue; }
      cudaEventRecord(e0);
      CK(launch_cluster((const void*)cluster_barrier_kernel, grid, 512, cs, args));
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
      cudaEventRecord(e0);
      CK(launch_cluster((const void*)cluster_split_barrier_kernel, grid, 512, cs, args));
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms2; cudaEventElapsedTime(&ms2, e0, e1);
      printf("cluster(%d) x %d clusters: cg cluster.sync %.3f us/barrier, arrive.release/wait.acquire %.3f us\n",
             cs, grid / cs, ms * 1e3 / iters, ms2 * 1e3 / iters);
    }
  }
  {
    long long* lat; CK(cudaMalloc(&lat, 64));
    for (int cs : {2, 16}) {
      for (int peer : {0, 1, cs - 1}) {
        int iters = 4096;
        void* args[] = {&iters, &peer, &lat};
        CK(launch_cluster((const void*)dsmem_latency_kernel, cs, 128, cs, args));
        CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
        long long h[2]; CK(cudaMemcpy(h, lat, 16, cudaMemcpyDeviceToHost));
        printf("DSMEM load round trip, cluster %d, peer rank %d: %lld cycles\n", cs, peer, h[0]);
      }
    }
    unsigned* ring; CK(cudaMalloc(&ring, 1 << 22));
    unsigned hr[1 << 12];
    for (int i = 0; i < (1 << 12); ++i) hr[i] = ((i * 1021 + 17) & ((1 << 12) - 1)) * 64;   // 256 B apart
    unsigned* big = new unsigned[1 << 20]();
    for (int i = 0; i < (1 << 12); ++i) big[i * 64] = hr[i];
    CK(cudaMemcpy(ring, big, 1 << 22, cudaMemcpyHostToDevice));
    l2_latency_kernel<<<1, 1>>>(ring, 4096, lat); CK(cudaDeviceSynchronize());
    l2_latency_kernel<<<1, 1>>>(ring, 4096, lat); CK(cudaDeviceSynchronize());
    long long h[2]; CK(cudaMemcpy(h, lat, 16, cudaMemcpyDeviceToHost));
    printf("L2 load round trip (ld.cg, 1 MB ring, warm): %lld cycles\n", h[0]);
    delete[] big;
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
