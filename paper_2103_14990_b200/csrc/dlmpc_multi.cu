// dlmpc_multi.cu -- the multi-rank test kernel of the device-side exchange
// (dlmpc_multi_solve): the ranks of a graph-partitioned solve as contiguous
// CTA slices of ONE cooperative launch on one GPU. Its own translation unit,
// because here the persistent kernel's CTA index and count are virtual
// (DLMPC_VB_SHIFT: blockIdx.x - P.vbase, P.vgrid), which the production
// kernels in dlmpc.cu must not pay for.
#define DLMPC_VB_SHIFT 1
#define DLMPC_MULTI_TU 1
#include "dlmpc_device.cuh"

namespace dlmpc {

cudaError_t launch_multi_kernel(int mode, int tc, const DevProblem* probs, const RunArgs* runs,
                                const int* cta_base, int n_ranks, int grid, int smem, cudaStream_t stream) {
  void (*fn)(const DevProblem*, const RunArgs*, const int*, int) = nullptr;
  if (mode == kExact) fn = dlmpc_multi_kernel<8, kExact>;
  else if (mode == kStream) fn = tc == 16 ? dlmpc_multi_kernel<16, kStream> : dlmpc_multi_kernel<8, kStream>;
  else if (mode == kTwoPhase) fn = tc == 16 ? dlmpc_multi_kernel<16, kTwoPhase> : dlmpc_multi_kernel<8, kTwoPhase>;
  if (!fn) return cudaErrorInvalidValue;   // patch modes: the overlapped stop test reads the local maxima
  cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       smem);
  if (e != cudaSuccess) return e;
  void* args[] = {&probs, &runs, &cta_base, &n_ranks};
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(fn), dim3(grid), dim3(kThreads), args,
                                     static_cast<size_t>(smem), stream);
}

}  // namespace dlmpc
