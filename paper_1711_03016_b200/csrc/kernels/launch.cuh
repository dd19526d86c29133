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

#ifndef __CUDACC_RTC__
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdlib>
#endif

namespace dlvm {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#ifdef DLVM_PDL_EARLY_TRIGGER
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#else
__device__ __forceinline__ void pdl_trigger() {}  // implicit trigger at CTA exit
#endif
// tcgen05 GEMMs (DLVM_PDL_GEMM_EARLY=1): release the successor after the
// prologue, so its CTAs can start theirs on SMs this grid leaves idle.
// Measured slower (c3 0.312 -> 0.315 ms, c4 10.39-10.53 -> 10.65-10.69 ms):
// off by default.
#ifndef DLVM_PDL_GEMM_EARLY
#define DLVM_PDL_GEMM_EARLY 0
#endif
__device__ __forceinline__ void pdl_trigger_gemm() {
#if DLVM_PDL_GEMM_EARLY
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

#ifndef __CUDACC_RTC__
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
  LaunchCfg(dim3 grid, dim3 block, size_t smem, cudaStream_t stream, unsigned cluster_x = 1, unsigned cluster_z = 1,
            bool pdl = true) {
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
    if (pdl && pdl_enabled()) {
      attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[n].val.programmaticStreamSerializationAllowed = 1;
      ++n;
    }
    cfg.attrs = attr;
    cfg.numAttrs = n;
  }
};

// Launch a kernel loaded from a create-time JIT cubin (csrc/jit.cpp) with the
// configuration of `L` (same grid, cluster and PDL attributes as the
// ahead-of-time path); `smem` > 48 KB is opted in on the function first.
inline cudaError_t launch_jit(void* fn, const LaunchCfg& L, void** args) {
  static PFN_cuLaunchKernelEx_v11060 launch = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    return cudaGetDriverEntryPoint("cuLaunchKernelEx", &p, cudaEnableDefault, &q) == cudaSuccess &&
                   q == cudaDriverEntryPointSuccess
               ? reinterpret_cast<PFN_cuLaunchKernelEx_v11060>(p)
               : nullptr;
  }();
  static PFN_cuFuncSetAttribute_v9000 set_attr = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    return cudaGetDriverEntryPoint("cuFuncSetAttribute", &p, cudaEnableDefault, &q) == cudaSuccess &&
                   q == cudaDriverEntryPointSuccess
               ? reinterpret_cast<PFN_cuFuncSetAttribute_v9000>(p)
               : nullptr;
  }();
  if (!launch || !set_attr) return cudaErrorNotSupported;
  CUfunction f = static_cast<CUfunction>(fn);
  if (L.cfg.dynamicSmemBytes > 48 * 1024 &&
      set_attr(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)L.cfg.dynamicSmemBytes) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  CUlaunchAttribute at[2];
  unsigned na = 0;
  for (unsigned i = 0; i < L.cfg.numAttrs; ++i) {
    const cudaLaunchAttribute& a = L.cfg.attrs[i];
    if (a.id == cudaLaunchAttributeClusterDimension) {
      at[na].id = CU_LAUNCH_ATTRIBUTE_CLUSTER_DIMENSION;
      at[na].value.clusterDim.x = a.val.clusterDim.x;
      at[na].value.clusterDim.y = a.val.clusterDim.y;
      at[na].value.clusterDim.z = a.val.clusterDim.z;
      ++na;
    } else if (a.id == cudaLaunchAttributeProgrammaticStreamSerialization) {
      at[na].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
      at[na].value.programmaticStreamSerializationAllowed = a.val.programmaticStreamSerializationAllowed;
      ++na;
    }
  }
  CUlaunchConfig c = {};
  c.gridDimX = L.cfg.gridDim.x;
  c.gridDimY = L.cfg.gridDim.y;
  c.gridDimZ = L.cfg.gridDim.z;
  c.blockDimX = L.cfg.blockDim.x;
  c.blockDimY = L.cfg.blockDim.y;
  c.blockDimZ = L.cfg.blockDim.z;
  c.sharedMemBytes = (unsigned)L.cfg.dynamicSmemBytes;
  c.hStream = static_cast<CUstream>(L.cfg.stream);
  c.attrs = at;
  c.numAttrs = na;
  return launch(&c, f, args, nullptr) == CUDA_SUCCESS ? cudaSuccess : cudaErrorLaunchFailure;
}

#endif

}  // namespace dlvm
