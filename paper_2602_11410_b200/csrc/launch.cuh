// Programmatic dependent launch (PDL): a kernel launched with launch_pdl may start (prologue:
// barrier init, TMEM alloc, descriptor prefetch) while the previous kernel on the stream drains
// its last CTAs; it blocks in pdl_wait() until that grid has completed and its writes are visible.
// Every kernel launched this way calls pdl_wait() before its first global access; pdl_trigger()
// lets the NEXT kernel launch as soon as every CTA of this one has started.
#pragma once
#include <cuda_runtime.h>

#include <utility>

namespace cadet {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace cadet
