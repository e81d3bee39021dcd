// pdl.cuh -- programmatic dependent launch (PDL) for chains of short kernels.
//
// A kernel launched with launch_pdl may be scheduled while the previous
// kernel on its stream is still running; it must call pdl_wait() before it
// touches memory the predecessor writes (griddepcontrol.wait returns once the
// predecessor grid has completed and its writes are visible; without a
// programmatic predecessor it returns at once).  What PDL buys is the launch
// latency of each link in a dependent chain (the per-tick stream path is ~15
// kernels of a few microseconds each).  VSB_PDL=0 launches them normally.
#pragma once
#include <utility>

#include <cuda_runtime.h>

#ifndef VSB_PDL
#define VSB_PDL 1
#endif

namespace vsb {

__device__ __forceinline__ void pdl_wait() {
#if VSB_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = VSB_PDL;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace vsb
