// Element-wise program kernel (K1/K2/K3/K7/K8 of SURVEY.md §2.5): one pass
// over an [R, C] iteration space (R = product of up to three row dims)
// evaluating a fused chain of the IR's element-wise ops with broadcasting
// ("fuse compatible element-wise operators to a single
// kernel"; P:L213 broadcasting), storing results and producing
// deterministic per-CTA partial sums for `reduce` (Table 1):
//   RED_COL  partial[blockIdx.y][c]          (sum over this CTA's rows)
//   RED_ROW  partial[r][blockIdx.x]          (sum over this CTA's columns)
//   RED_ALL  partial[blockIdx.y*gx + blockIdx.x]
// A finalize launch (the same kernel over the partials, nchunks > 1) sums
// partials in a fixed order.
//
// Thread layout: blockDim = (bx, by), bx*by = 256, bx a multiple of 32;
// thread (tx, ty) owns VEC consecutive columns c = (blockIdx.x*bx + tx)*VEC
// and rows r = (blockIdx.y*rpt + k)*by + ty, k < rpt.  With VEC = 4 every
// full-stride operand moves as one 16-byte (f32) / 8-byte (bf16) / 4-byte
// (bool) access per thread, coalesced across the warp.
//
// Two instantiations of the same body: P = void interprets p.prog (slots in
// local memory); P = spec::Prog<...> is a compile-time program (registers).
#define DLVM_EW_DEFINE_FIXED_KERNELS
#include "ew_kernels.cuh"

#include <cstdlib>
#include <cstring>
#include "spec_registry.h"

namespace dlvm {

namespace {

using namespace kern;

// TMA-staged path: 256 x 1 blocks of 4-wide vectors over [R, C]; every
// row-varying input a 16-byte aligned unit-column-stride row segment, every
// store contiguous along the row (DLVM_EW_TMA=0 disables)
int tma_stages(const EwParams& p, int bx, int by, int n_in, int rows) {
  static const bool on = [] {
    const char* e = std::getenv("DLVM_EW_TMA");  // off by default: the f32 row loop of ew2d_kernel measured faster
    return e && e[0] == '1';
  }();
  if (!on || p.vec != 4 || bx != 256 || by != 1 || p.ndims != 2 || p.ncols != 1) return 0;
  int nsi = 0;
  for (int i = 0; i < n_in; ++i) {
    const EwDevIn& in = p.in[i];
    if (in.s[0] == 0) continue;
    const int es = st_bytes(in.st);
    if (in.nchunks != 1 || in.s[1] != 1 || reinterpret_cast<uintptr_t>(in.ptr) % 16 || (in.s[0] * es) % 16 ||
        (p.dims[1] * es) % 16)
      return 0;
    ++nsi;
  }
  for (int o = 0; o < p.prog.n_stores; ++o)
    if (p.out[o].s[1] != 1) return 0;
  if (nsi == 0) return 0;
  const int stage = nsi * rows * kTmaRowBytes;
  int nst = 98304 / stage;  // two CTAs (16 consumer warps) per SM
  return nst > 8 ? 8 : (nst < 2 ? 0 : nst);
}

template <class P>
cudaError_t launch_tma_ew(const EwParams& p, int nst, cudaStream_t stream) {
  int nsi = 0;
  for (int i = 0; i < spec::Traits<P>::kIn; ++i) nsi += p.in[i].s[0] != 0;
  const int smem = nst * nsi * tma_rows<P>() * kTmaRowBytes + 16 * nst;
  static int configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(ew_tma_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    configured = 227 * 1024;
  }
  const int64_t tiles = p.gx * p.gy;
  LaunchCfg L(dim3((unsigned)(tiles < 296 ? tiles : 296)), dim3(288), smem, stream);
  cudaError_t e = cudaLaunchKernelEx(&L.cfg, ew_tma_kernel<P>, p, nst);
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int VEC, class P>
cudaError_t launch_spec_ew(const EwParams& p, int bx, int by, cudaStream_t stream) {
  dim3 grid((unsigned)p.gx, (unsigned)p.gy), block(bx, by);
  if constexpr (!has_row_red<P>()) {
    if constexpr (VEC == 4) {
      const int nst = tma_stages(p, bx, by, spec::Traits<P>::kIn, tma_rows<P>());
      if (nst) return launch_tma_ew<P>(p, nst, stream);
    }
    if (p.ndims == 2 && p.ncols == 1) {
      LaunchCfg L(grid, block, 0, stream);
      cudaError_t e = cudaLaunchKernelEx(&L.cfg, ew2d_kernel<VEC, P>, p);
      return e != cudaSuccess ? e : cudaGetLastError();
    }
  }
  LaunchCfg L(grid, block, 0, stream);
  cudaError_t e = cudaLaunchKernelEx(&L.cfg, ew_kernel<VEC, P>, p);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace

// ---------------------------------------------------------- registry
#define DLVM_SPEC_EW(VEC, SIG, ...) {SIG, VEC, &launch_spec_ew<VEC, __VA_ARGS__>},
#define DLVM_SPEC_GEMM(IDX, BN, SIG, ...)
#define DLVM_SPEC_SIMT(BM, SIG, ...)
namespace {
using namespace spec;
const EwSpecEntry kEwSpecs[] = {
#include "spec_programs.inc"
    {nullptr, 0, nullptr}};
}  // namespace
#undef DLVM_SPEC_EW
#undef DLVM_SPEC_GEMM
#undef DLVM_SPEC_SIMT

EwLaunchFn find_ew_spec(const char* sig, int vec) {
  for (const EwSpecEntry* e = kEwSpecs; e->sig; ++e)
    if (e->vec == vec && std::strcmp(e->sig, sig) == 0) return e->fn;
  return nullptr;
}

int num_ew_specs() {
  int n = 0;
  for (const EwSpecEntry* e = kEwSpecs; e->sig; ++e) ++n;
  return n;
}

cudaError_t launch_ew(const EwParams& p, int bx, int by, cudaStream_t stream) {
  dim3 grid((unsigned)p.gx, (unsigned)p.gy), block(bx, by);
  LaunchCfg L(grid, block, 0, stream);
  cudaError_t e = p.vec == 4 ? cudaLaunchKernelEx(&L.cfg, ew_kernel<4, void>, p)
                             : cudaLaunchKernelEx(&L.cfg, ew_kernel<1, void>, p);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_ew_fn(void* fn, const EwParams& p, int bx, int by, cudaStream_t stream) {
  LaunchCfg L(dim3((unsigned)p.gx, (unsigned)p.gy), dim3(bx, by), 0, stream);
  void* args[] = {const_cast<EwParams*>(&p)};
  return launch_jit(fn, L, args);
}

cudaError_t launch_finalize(const EwParams& p, cudaStream_t stream) {
  const int nq = p.prog.n_in > 0 ? p.prog.n_in : 1;
  int64_t nb = 1;  // CTAs of the longest reduction (32 or 1 outputs per CTA)
  for (int q = 0; q < nq; ++q) {
    const int64_t n = p.dims[q];
    const int64_t b = n >= 32 ? (n + 31) / 32 : n;
    nb = b > nb ? b : nb;
  }
  LaunchCfg L(dim3((unsigned)nb, (unsigned)nq), dim3(256), 0, stream);
  cudaError_t e = cudaLaunchKernelEx(&L.cfg, finalize_kernel, p);
  return e != cudaSuccess ? e : cudaGetLastError();
}

// [rows, cols] f32 / bf16 -> bf16 rows of ld (multiple of 8) elements, zero
// padded: each thread writes 8 outputs (16 bytes) per step; sources whose
// rows are 16-byte aligned (bf16: cols % 8 == 0; f32: cols % 4 == 0) move
// as vectors, the rest element by element
__global__ void pack_bf16_kernel(const void* __restrict__ src, int src_f32, int64_t rows, int64_t cols,
                                 unsigned short* __restrict__ dst, int64_t ld) {
  pdl_trigger();
  pdl_wait();
  const int64_t per_row = ld / 8, total = rows * per_row;
  const bool vec = src_f32 ? (cols % 4 == 0) : (cols % 8 == 0);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / per_row, c = (i - r * per_row) * 8;
    unsigned short v[8];
    if (vec && c + 8 <= cols) {
      if (src_f32) {
        const float4* q = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(src) + r * cols + c);
        const float4 x0 = __ldg(q), x1 = __ldg(q + 1);
        v[0] = f2bf(x0.x); v[1] = f2bf(x0.y); v[2] = f2bf(x0.z); v[3] = f2bf(x0.w);
        v[4] = f2bf(x1.x); v[5] = f2bf(x1.y); v[6] = f2bf(x1.z); v[7] = f2bf(x1.w);
      } else {
        const uint4 x = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const unsigned short*>(src) + r * cols + c));
        *reinterpret_cast<uint4*>(dst + r * ld + c) = x;
        continue;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        v[j] = 0;
        if (c + j < cols)
          v[j] = src_f32 ? f2bf(__ldg(reinterpret_cast<const float*>(src) + r * cols + c + j))
                         : __ldg(reinterpret_cast<const unsigned short*>(src) + r * cols + c + j);
      }
    }
    uint4 o;
    o.x = (unsigned)v[0] | ((unsigned)v[1] << 16);
    o.y = (unsigned)v[2] | ((unsigned)v[3] << 16);
    o.z = (unsigned)v[4] | ((unsigned)v[5] << 16);
    o.w = (unsigned)v[6] | ((unsigned)v[7] << 16);
    *reinterpret_cast<uint4*>(dst + r * ld + c) = o;
  }
}

cudaError_t launch_pack_bf16(const void* src, bool src_f32, int64_t rows, int64_t cols, void* dst, int64_t ld,
                             cudaStream_t stream) {
  if (ld % 8) return cudaErrorInvalidValue;
  const int64_t total = rows * (ld / 8);
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 8);
  LaunchCfg L(dim3((unsigned)blocks), dim3(256), 0, stream);
  cudaError_t e = cudaLaunchKernelEx(&L.cfg, pack_bf16_kernel, src, src_f32 ? 1 : 0, rows, cols,
                                     reinterpret_cast<unsigned short*>(dst), ld);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_cast_bf16(const float* src, void* dst, int64_t n, cudaStream_t stream) {
  int64_t blocks = std::min<int64_t>((n / 4 + 255) / 256 + 1, 148 * 16);
  LaunchCfg L(dim3((unsigned)blocks), dim3(256), 0, stream);
  cudaError_t e = cudaLaunchKernelEx(&L.cfg, cast_bf16_kernel, src, reinterpret_cast<unsigned short*>(dst), n);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace dlvm
