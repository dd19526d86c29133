// SIMT GEMM for `dot` (Table 1) under the fp32 policy (exact fp32
// operands, FFMA accumulation; K6 of SURVEY.md §2.5) and for bf16 dots whose
// shapes/strides the tensor-core path cannot take (tiny or TMA-misaligned).
// `transpose` feeding a dot is absorbed as operand strides (A/B may be row-
// or column-major).  BM x 64 tile (BM = 32 or 64, chosen by the planner),
// BK = 16, 256 threads x (BM/16)x4 outputs, next K tile prefetched into
// registers while the current one is multiplied.  Small grids split K over a thread-block cluster: each CTA sums
// its K range, rank 0 adds the peers' partial tiles from distributed shared
// memory in rank order (deterministic) and runs the fused element-wise
// epilogue program (bias, activation, activation derivative, reductions;
// P:L231-236) once over all of a thread's outputs: a compile-time program
// (spec_programs.inc) keeps every slot in registers; the interpreter
// (SimtVm) runs one output row of 4 at a time.
#include <cstdlib>
#include <cstring>

#include "gemm_simt_kernel.cuh"
#include "spec_registry.h"

namespace dlvm {

namespace {

using namespace kern::simt;

// launch geometry: tile grid and the cluster split of K (see the kernel)
LaunchCfg simt_config(const GemmParams& p, int BMv, cudaStream_t stream, int64_t* kchunk_out) {
  const int64_t gx = (p.N + BN - 1) / BN, gy = (p.M + BMv - 1) / BMv, tiles = gx * gy;
  // split K over a cluster when the tile grid leaves most SMs idle.
  // DLVM_SIMT_MAX_SPLIT caps the split (profiling experiments; default 8).
  // Each split costs a cluster barrier pair and a DSMEM pass (~2 us measured
  // by tools/simt_probe.py), so splits are used only on SM-starved grids and
  // keep >= 2 K tiles each.
  static const int64_t max_split = [] {
    const char* e = std::getenv("DLVM_SIMT_MAX_SPLIT");
    const int64_t v = e ? std::atoll(e) : 8;
    return v < 1 ? 1 : (v > 8 ? 8 : v);
  }();
  const int64_t K = p.seg[0].K;
  int64_t ks = 1;
  if (tiles < 148 && p.n_seg == 1) {
    ks = 296 / tiles;
    const int64_t kmax = (K + 2 * BK - 1) / (2 * BK);
    ks = ks < kmax ? ks : kmax;
    ks = ks < max_split ? ks : max_split;
    ks = ks > 1 ? ks : 1;
  }
  int64_t kchunk = ((K + ks - 1) / ks + BK - 1) / BK * BK;
  if (kchunk <= 0) kchunk = BK;
  ks = K > 0 ? (K + kchunk - 1) / kchunk : 1;
  *kchunk_out = kchunk;
  return LaunchCfg(dim3((unsigned)gx, (unsigned)gy, (unsigned)ks), dim3(256, 1, 1), 0, stream, 1, (unsigned)ks);
}

template <bool BF16, int BM, class PROG>
cudaError_t launch_bm(const GemmParams& p, cudaStream_t stream) {
  int64_t kchunk;
  LaunchCfg L = simt_config(p, BM, stream, &kchunk);
  return cudaLaunchKernelEx(&L.cfg, gemm_simt_kernel<BF16, BM, PROG>, p, kchunk);
}

template <int BM, class PROG>
cudaError_t launch_simt_prog(const GemmParams& p, cudaStream_t stream) {
  cudaError_t e = p.bf16 ? launch_bm<true, BM, PROG>(p, stream) : launch_bm<false, BM, PROG>(p, stream);
  return e != cudaSuccess ? e : cudaGetLastError();
}

using namespace spec;
#define DLVM_SPEC_EW(VEC, SIG, ...)
#define DLVM_SPEC_GEMM(IDX, BN, SIG, ...)
#define DLVM_SPEC_SIMT(BM, SIG, ...) {SIG, BM, &launch_simt_prog<BM, __VA_ARGS__>},
const GemmSpecEntry kSimtTable[] = {
#include "spec_programs.inc"
    {nullptr, 0, nullptr}};
#undef DLVM_SPEC_EW
#undef DLVM_SPEC_GEMM
#undef DLVM_SPEC_SIMT

}  // namespace

GemmLaunchFn find_simt_spec(const char* sig, int bm) {
  for (const GemmSpecEntry* e = kSimtTable; e->sig; ++e)
    if (e->bn == bm && std::strcmp(e->sig, sig) == 0) return e->fn;
  return nullptr;
}

int num_simt_specs() { return (int)(sizeof(kSimtTable) / sizeof(kSimtTable[0])) - 1; }

cudaError_t launch_gemm_simt_fn(void* fn, const GemmParams& p, cudaStream_t stream) {
  int64_t kchunk;
  LaunchCfg L = simt_config(p, p.bm, stream, &kchunk);
  void* args[] = {const_cast<GemmParams*>(&p), &kchunk};
  return launch_jit(fn, L, args);
}

cudaError_t launch_gemm_simt(const GemmParams& p, cudaStream_t stream) {
  if (p.bm == 32) return launch_simt_prog<32, SimtVm>(p, stream);
  if (p.bm == 64) return launch_simt_prog<64, SimtVm>(p, stream);
  return cudaErrorInvalidValue;
}

}  // namespace dlvm
