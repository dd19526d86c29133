"""B200-native (sm_100a) hot path of DLVM (arXiv 1711.03016): straight-line
DLVM IR functions and the adjoint functions its AD pass generates, executed
by fused element-wise kernels and tcgen05 GEMMs through a C ABI
(include/dlvm.h).  `Function` is the Python binding; `dp` holds the
data-parallel driver: bucketed NCCL all-reduce of parameter gradients, or
the fused reduction of gradients into their owners' peer memory
(DLVM_F32_ADD outputs, `AddInto`)."""

from .dlvm import (DLVM_BF16, DLVM_BOOL, DLVM_F32, DLVM_F32_ADD, DLVM_GRADIENT, AddInto, DLVM_NO_FUSION, DLVM_NO_JIT, DLVM_NO_OPT, DLVM_NO_SPECIALIZE,
                   DLVM_PLAN_ONLY, DLVM_PRIMAL, DlvmError, Function, dlvm_version, lib)

__all__ = ["Function", "DlvmError", "lib", "dlvm_version", "DLVM_PLAN_ONLY", "DLVM_NO_FUSION",
           "DLVM_NO_SPECIALIZE", "DLVM_NO_OPT", "DLVM_NO_JIT", "DLVM_PRIMAL", "DLVM_GRADIENT", "DLVM_F32", "DLVM_BF16", "DLVM_BOOL", "DLVM_F32_ADD", "AddInto"]
