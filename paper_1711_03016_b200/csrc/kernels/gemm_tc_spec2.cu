// Compile-time GEMM epilogue specialisations, shard 2 of 4 (entries of
// spec_programs.inc with index % 4 == 2; sharded so nvcc builds them in
// parallel).
#include "gemm_tc.cuh"

namespace dlvm {
namespace {
template <int IDX, int BN, class PROG>
constexpr GemmLaunchFn pick_gemm() {
  if constexpr (IDX % 4 == 2)
    return &launch_prog<BN, PROG>;
  else
    return nullptr;
}
using namespace spec;
#define DLVM_SPEC_EW(VEC, SIG, ...)
#define DLVM_SPEC_GEMM(IDX, BN, SIG, ...) {SIG, BN, pick_gemm<IDX, BN, __VA_ARGS__>()},
#define DLVM_SPEC_SIMT(BM, SIG, ...)
const GemmSpecEntry kTable[] = {
#include "spec_programs.inc"
    {nullptr, 0, nullptr}};
#undef DLVM_SPEC_EW
#undef DLVM_SPEC_GEMM
#undef DLVM_SPEC_SIMT
}  // namespace

const GemmSpecEntry* gemm_spec_table_2() { return kTable; }

}  // namespace dlvm
