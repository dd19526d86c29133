// Create-time specialisation of kernels (the B200 form of the paper's JIT,
// PAPER.md Fig. 4 "At runtime, 'dg' gets just-in-time compiled through
// DLVM"; §3.2 L322-329 code generation).  The planner's element-wise
// programs that are not in the ahead-of-time registry (spec_programs.inc)
// are compiled by NVRTC from the same kernel templates (kernels/*_kernel.cuh,
// ew_kernels.cuh) with the program as compile-time types, so every slot
// lives in registers instead of the interpreter's local-memory slots.
// Results are bit-identical to the interpreter (same vm_apply).
//
// NVRTC is loaded with dlopen; without it (or with DLVM_JIT=0) programs
// outside the registry run on the interpreter.  Cubins are cached in
// $DLVM_JIT_CACHE (default ~/.cache/dlvm-jit), keyed by a hash of the kernel
// sources, the instantiation and the options.
#pragma once

#include <string>
#include <vector>

namespace dlvm {

// one kernel instantiation, e.g. "&dlvm::kern::ew2d_kernel<4, dlvm::spec::Prog<...>>"
struct JitRequest {
  std::string expr;
  void* function = nullptr;  // CUfunction after jit_load
  std::string error;
};

bool jit_available();  // NVRTC loadable and DLVM_JIT != 0
// C++ type of an element-wise program signature (plan.cpp program_signature),
// "dlvm::spec::Prog<...>"
std::string jit_prog_type(const std::string& sig);
// compile (in parallel, through the disk cache) and load every request into
// the current CUDA context; returns false if any failed (see error)
bool jit_build(std::vector<JitRequest>& reqs);

}  // namespace dlvm
