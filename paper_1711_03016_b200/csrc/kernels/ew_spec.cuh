// Compile-time element-wise programs.
//
// The planner's EwProgram is interpreted by the generic kernels (slots in
// local memory, one switch per op).  For the programs the benchmarked
// workloads produce, tools/gen_specializations.py writes spec_programs.inc:
// the same programs as C++ types, so every slot index is a compile-time
// constant (registers) and every op's switch folds away.  Both paths call
// the same vm_apply, so a specialised program computes bit-identical results
// to the interpreter (checked by tests/test_gpu_parity.py).
#pragma once

#include "ew_device.cuh"

namespace dlvm {
namespace spec {

template <int OP, int D, int A, int B, int C>
struct Ins {
  static constexpr int op = OP, dst = D;
};
template <int... S>
struct St {};
template <int... R>  // flattened (slot, kind) pairs
struct Rd {};

template <int NIN, int NLIT, class STs, class RDs, class... Is>
struct Prog {
  static constexpr int kIn = NIN, kLit = NLIT, kIns = (int)sizeof...(Is);
  static constexpr int kSlots = NIN + NLIT + (int)sizeof...(Is);
};

template <class P>
struct Traits;

template <int... S>
struct StArr {
  static constexpr int n = (int)sizeof...(S);
  __host__ __device__ static constexpr int at(int k) {
    constexpr int a[sizeof...(S) + 1] = {S..., 0};
    return a[k];
  }
};
template <int... R>
struct RdArr {
  static constexpr int n = (int)sizeof...(R) / 2;
  __host__ __device__ static constexpr int at(int k) {
    constexpr int a[sizeof...(R) + 1] = {R..., 0};
    return a[k];
  }
};

template <int NIN, int NLIT, int... S, int... R, class... Is>
struct Traits<Prog<NIN, NLIT, St<S...>, Rd<R...>, Is...>> {
  using Stores = StArr<S...>;
  using Reds = RdArr<R...>;
  static constexpr int kIn = NIN, kLit = NLIT;
  static constexpr int kSlots = NIN + NLIT + (int)sizeof...(Is);

  template <int VEC, int OP, int D, int A, int B, int C>
  __device__ __forceinline__ static void one(float (&v)[kSlots][VEC], Ins<OP, D, A, B, C>) {
#pragma unroll
    for (int j = 0; j < VEC; ++j) v[D][j] = vm_apply((uint8_t)OP, v[A][j], v[B][j], v[C][j]);
  }
  template <int VEC>
  __device__ __forceinline__ static void exec(float (&v)[kSlots][VEC]) {
    (one<VEC>(v, Is{}), ...);
  }
  // slot d holds only 0.0f / 1.0f: written by a compare or a cast to bool
  __host__ __device__ static constexpr bool is01(int d) {
    constexpr int ops[] = {Is::op..., -1};
    constexpr int dst[] = {Is::dst..., -1};
    for (int k = 0; k < (int)sizeof...(Is); ++k)
      if (dst[k] == d) return (ops[k] >= VM_LT && ops[k] <= VM_NE) || ops[k] == VM_TOBOOL;
    return false;
  }
};

}  // namespace spec
}  // namespace dlvm
