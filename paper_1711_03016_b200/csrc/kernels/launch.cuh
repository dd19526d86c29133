// Launch configuration shared by every kernel of the library.
//
// Programmatic dependent launch (PDL): kernels are launched with
// programmatic stream serialization, so a kernel's CTAs may be scheduled
// while its predecessor in the stream drains.  Every kernel therefore calls
// pdl_wait() (griddepcontrol.wait: the predecessor has completed and its
// memory is visible) before it touches global memory the predecessor may
// write.  The successor is released when this kernel's CTAs exit (implicit
// trigger): measured on c1, an early griddepcontrol.launch_dependents
// (-DDLVM_PDL_EARLY_TRIGGER) let waiting successor CTAs take SMs the
// split-K clusters needed (40 -> 43-48 us/step), while the implicit trigger
// hides launch latency (40.7 -> 38.9 us, e2e 84 -> 74 us).  Kernels launched
// by other code (torch copies) are ordinary stream predecessors: the wait
// then returns at once.  DLVM_PDL=0 launches without the attribute.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>

namespace dlvm {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#ifdef DLVM_PDL_EARLY_TRIGGER
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#else
__device__ __forceinline__ void pdl_trigger() {}  // implicit trigger at CTA exit
#endif

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("DLVM_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

struct LaunchCfg {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[2];
  LaunchCfg(dim3 grid, dim3 block, size_t smem, cudaStream_t stream, unsigned cluster_x = 1, unsigned cluster_z = 1) {
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    int n = 0;
    if (cluster_x * cluster_z > 1) {
      attr[n].id = cudaLaunchAttributeClusterDimension;
      attr[n].val.clusterDim.x = cluster_x;
      attr[n].val.clusterDim.y = 1;
      attr[n].val.clusterDim.z = cluster_z;
      ++n;
    }
    if (pdl_enabled()) {
      attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[n].val.programmaticStreamSerializationAllowed = 1;
      ++n;
    }
    cfg.attrs = attr;
    cfg.numAttrs = n;
  }
};

}  // namespace dlvm
