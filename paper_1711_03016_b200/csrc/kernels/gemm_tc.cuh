#pragma once
// tcgen05 tensor-core GEMM for `dot` under the bf16 policy (K5 of SURVEY.md
// §2.5; Table 1 "dot"; reading A15: bf16 operands, fp32 accumulation).
//
// C[M,N] = A[M,K] . B[K,N], bf16 operands read by TMA (cp.async.bulk.tensor,
// 128-byte swizzle) into a 4-stage shared-memory ring guarded by mbarriers;
// one elected thread issues tcgen05.mma.cta_group::1.kind::f16 (M=128,
// N=BN, K=16) accumulating in TMEM (two BN-column accumulators so the
// epilogue of tile i overlaps the main loop of tile i+1); four epilogue warps
// read TMEM with tcgen05.ld.32x32b and run the fused element-wise epilogue
// program (bias, activation, activation derivative, column/row/full partial
// sums) before storing -- "linear algebra fusion" of P:L231-236 done on the
// accumulator tile.  `transpose` of an operand is absorbed into the UMMA
// descriptor major bit (A K- or M-major, B K- or N-major), so the adjoint
// dots dY.W^T and X^T.dY read W and X in place.
//
// Warp roles (256 threads, persistent over tiles, 1 CTA/SM):
//   warp 0: TMA producer   warp 1: MMA issuer   warp 2: TMEM allocator
//   warps 4-11: epilogue (TMEM lanes 32*(warp%4) .. +31 = tile rows; two
//               warps per lane quarter split the tile's column chunks)
// Host side: tensor maps, launch configuration, registry entry points.
#include <atomic>
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "gemm_tc_kernel.cuh"
#include "spec_registry.h"

#ifdef DLVM_GEMM_TRACE
namespace dlvm {
namespace kern {
extern unsigned long long* g_gemm_trace_ptr;  // gemm_tc.cu (trace builds)
extern int g_gemm_trace_slots, g_gemm_trace_next;
}  // namespace kern
}  // namespace dlvm
#endif

namespace dlvm {

namespace {

using namespace kern;

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D bf16 tensor map: inner dim (contiguous) `inner`, outer dim `outer`
// with row pitch `ld` elements, box {64, box_outer}, 128-byte swizzle
bool encode(CUtensorMap* map, const void* ptr, int64_t inner, int64_t outer, int64_t ld, int box_outer) {
  auto fn = get_encode();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {64u, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1u, 1u};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BN, int CTAS = 1>
constexpr int smem_bytes() {
  constexpr int NST = num_stages<CTAS, BN>();
  return 1024 + NST * (A_STAGE_BYTES + (BN / CTAS) * BK * 2) + 16 * NST + 64 +
         (kEpiReds * 4 * BN + kEpiReds * 2 * BM + kEpiReds * 8 + 8 * 32 * 17) * 4;
}
static_assert(smem_bytes<256, 2>() <= 227 * 1024, "CTA-pair stages exceed shared memory");

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

bool make_params(const GemmParams& p, TcParams* tp, int ctas = 1) {
  memset(tp, 0, sizeof(*tp));
  tp->g = p;
#ifdef DLVM_GEMM_TRACE
  // launch k of the traced run writes slice k % slots of [slots][148][8]
  tp->trace = g_gemm_trace_ptr ? g_gemm_trace_ptr + (size_t)(g_gemm_trace_next++ % g_gemm_trace_slots) * 148 * 8
                               : nullptr;
#endif
  const int BN = p.bn;
  if (p.n_seg < 1 || p.n_seg > kMaxSeg) return false;
  for (int q = 0; q < p.n_seg; ++q) {
    const GemmSegParams& G = p.seg[q];
    bool ok;
    if (G.a_kmajor)  // A [M,K], K contiguous: map {K, M}, box {64, 128}
      ok = encode(&tp->tma_a[q], G.a, G.K, p.M, G.a_s0, BM);
    else  // A stored [K][M]: map {M, K}, box {64, 64}
      ok = encode(&tp->tma_a[q], G.a, p.M, G.K, G.a_s1, 64);
    if (!ok) return false;
    if (G.b_kmajor)  // B stored [N][K]: map {K, N}, box {64, BN / ctas} (a CTA's share)
      ok = encode(&tp->tma_b[q], G.b, G.K, p.N, G.b_s1, BN / ctas);
    else  // B stored [K][N]: map {N, K}, box {64, 64}
      ok = encode(&tp->tma_b[q], G.b, p.N, G.K, G.b_s0, 64);
    if (!ok) return false;
  }
  tp->tiles_m = (int)((p.M + BM * ctas - 1) / (BM * ctas));
  tp->tiles_n = (int)((p.N + BN - 1) / BN);
  // L2 policy: when one operand is small enough to stay resident (every tile
  // row re-reads all of it) and the other is streamed once, keep the small
  // one and stream the big one, so the epilogue's store stream does not evict
  // it (DLVM_GEMM_L2HINT=0 disables)
  static const int hints_on = [] {
    const char* e = std::getenv("DLVM_GEMM_L2HINT");
    return e ? std::atoi(e) : 0;  // off: measured no gain (A is re-read by every N tile too)
  }();
  double bytes_a = 0, bytes_b = 0;
  for (int q = 0; q < p.n_seg; ++q) {
    bytes_a += 2.0 * p.M * p.seg[q].K;
    bytes_b += 2.0 * p.N * p.seg[q].K;
  }
  const double keep_max = 48.0 * (1 << 20);
  tp->hint_a = tp->hint_b = 0;
  if (hints_on) {
    const int stream = hints_on == 2 ? 2 : 0;
    if (bytes_b <= keep_max && bytes_a >= 4 * bytes_b) {
      tp->hint_b = 1;
      tp->hint_a = stream;
    } else if (bytes_a <= keep_max && bytes_b >= 4 * bytes_a) {
      tp->hint_a = 1;
      tp->hint_b = stream;
    }
  }
  return true;
}

// CTA pairs for large 256-wide tiles (DLVM_GEMM_CTA2=0 forces single CTAs)
bool use_cta_pair(const GemmParams& p) {
  static const int mode = [] {
    const char* e = std::getenv("DLVM_GEMM_CTA2");
    return e ? std::atoi(e) : 1;
  }();
  return mode != 0 && p.bn == 256 && p.M >= 512;
}

template <int BN, class PROG, int CTAS>
cudaError_t launch_ctas(const GemmParams& p, cudaStream_t stream) {
  // the max-dynamic-smem attribute is per device: one bit per device ordinal
  static std::atomic<uint64_t> configured{0};
  constexpr int SMEM = smem_bytes<BN, CTAS>();
  auto kern = gemm_tc_kernel<BN, PROG, CTAS>;
  int dev = 0;
  cudaError_t e0 = cudaGetDevice(&dev);
  if (e0 != cudaSuccess) return e0;
  const uint64_t bit = 1ull << (dev & 63);
  if (!(configured.load(std::memory_order_relaxed) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    configured.fetch_or(bit);
  }
  TcParams tp;
  if (!make_params(p, &tp, CTAS)) return cudaErrorInvalidValue;
  // persistent: one CTA (pair) per SM (pair), up to one per work item
  // (tile x K split)
  const int items = tp.tiles_m * tp.tiles_n * std::max(p.ksplit, 1);
  const int grid = CTAS * std::min(items, num_sms() / CTAS);
  LaunchCfg L(dim3((unsigned)grid, 1, 1), dim3(NUM_THREADS, 1, 1), SMEM, stream, CTAS, 1);
  cudaError_t e = cudaLaunchKernelEx(&L.cfg, kern, tp);
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int BN, class PROG>
cudaError_t launch_prog(const GemmParams& p, cudaStream_t stream) {
  if constexpr (BN == 256) {
    if (use_cta_pair(p)) return launch_ctas<BN, PROG, 2>(p, stream);
  }
  return launch_ctas<BN, PROG, 1>(p, stream);
}

}  // namespace
}  // namespace dlvm
