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
#include <type_traits>

#include "ew_spec.cuh"
#include "launch.cuh"
#include "spec_registry.h"

namespace dlvm {

namespace {

__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = __fadd_rn(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

struct VmTraits {
  static constexpr int kSlots = kMaxSlots;
};

template <class T, bool S>
__host__ __device__ constexpr int num_red_slots() {
  if constexpr (S) return T::Reds::n; else return kMaxReduces;
}

template <int VEC, class P>
__global__ void __launch_bounds__(256) ew_kernel(const __grid_constant__ EwParams p) {
  pdl_trigger();
  pdl_wait();
  constexpr bool SPEC = !std::is_void_v<P>;
  using T = std::conditional_t<SPEC, spec::Traits<std::conditional_t<SPEC, P, spec::Prog<0, 0, spec::St<>, spec::Rd<>>>>, VmTraits>;
  constexpr int NS = T::kSlots;
  const EwProgram& Pg = p.prog;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int bx = blockDim.x, by = blockDim.y;
  const int nd = p.ndims;
  const int nrd = nd - p.ncols;  // row dims
  int64_t R = 1, C = 1;
  for (int d = 0; d < nd; ++d) (d < nrd ? R : C) *= p.dims[d];
  const int64_t c = ((int64_t)blockIdx.x * bx + tx) * VEC;
  const bool cval = c < C;
  const int64_t c_hi = p.ncols == 2 ? c / p.dims[nd - 1] : 0, c_lo = p.ncols == 2 ? c % p.dims[nd - 1] : c;
  // element offset of column c for strides s (two column dims only with VEC == 1)
  auto col_off = [&](const int64_t* s) -> int64_t { return c_lo * s[nd - 1] + (p.ncols == 2 ? c_hi * s[nd - 2] : 0); };
  const int n_in = SPEC ? 0 : Pg.n_in;
  float v[NS][VEC];
  if constexpr (SPEC) {
#pragma unroll
    for (int i = 0; i < T::kLit; ++i)
#pragma unroll
      for (int j = 0; j < VEC; ++j) v[T::kIn + i][j] = Pg.lits[i];
  } else {
    for (int i = 0; i < Pg.n_lits; ++i)
#pragma unroll
      for (int j = 0; j < VEC; ++j) v[n_in + i][j] = Pg.lits[i];
  }
  const int n_red = SPEC ? 0 : Pg.n_reduces;
  auto red_slot = [&](int q) -> int {
    if constexpr (SPEC) return T::Reds::at(2 * q); else return Pg.reduce_slot[q];
  };
  auto red_kind = [&](int q) -> int {
    if constexpr (SPEC) return T::Reds::at(2 * q + 1); else return Pg.reduce_kind[q];
  };
  constexpr int NRS = num_red_slots<T, SPEC>();
  const int nred = SPEC ? NRS : n_red;
  bool has_row = false, has_colall = false;
#pragma unroll
  for (int q = 0; q < NRS; ++q)
    if (q < nred) {
      has_row |= red_kind(q) == RED_ROW;
      has_colall |= red_kind(q) != RED_ROW;
    }
  float acc[NRS > 0 ? NRS : 1][VEC];
#pragma unroll
  for (int q = 0; q < (NRS > 0 ? NRS : 1); ++q)
#pragma unroll
    for (int j = 0; j < VEC; ++j) acc[q][j] = 0.f;
  __shared__ float red_s[256 * 4];
  __shared__ float row_s[8][8];

  // rows handled per loop iteration: specialised programs load RPI rows
  // before computing, so 2*VEC independent 16-byte loads per input are in flight
  constexpr int RPI = SPEC ? 2 : 1;
  for (int k = 0; k < p.rpt; k += RPI) {
    int64_t rrow[RPI];
    bool vrow[RPI];
#pragma unroll
    for (int i = 0; i < RPI; ++i) {
      rrow[i] = ((int64_t)blockIdx.y * p.rpt + k + i) * by + ty;
      vrow[i] = cval && (k + i) < p.rpt && rrow[i] < R;
    }
    float rowv[RPI][NRS > 0 ? NRS : 1];
#pragma unroll
    for (int i = 0; i < RPI; ++i)
#pragma unroll
      for (int q = 0; q < (NRS > 0 ? NRS : 1); ++q) rowv[i][q] = 0.f;
    // element offset of row r for a ref with strides s (2-D fast path: no div/mod)
    auto row_off = [&](const int64_t* s, int64_t r) -> int64_t {
      if (nrd == 1) return r * s[0];
      int64_t off = 0, rr = r;
      for (int d = nrd - 1; d >= 0; --d) {
        off += (rr % p.dims[d]) * s[d];
        rr /= p.dims[d];
      }
      return off;
    };
    if constexpr (SPEC) {
      float w[NS][RPI * VEC];
#pragma unroll
      for (int i = 0; i < T::kLit; ++i)
#pragma unroll
        for (int j = 0; j < RPI * VEC; ++j) w[T::kIn + i][j] = Pg.lits[i];
#pragma unroll
      for (int i = 0; i < T::kIn; ++i) {
        const EwDevIn& in = p.in[i];
        const int64_t cs = in.s[nd - 1];
#pragma unroll
        for (int u = 0; u < RPI; ++u) {
          if (vrow[u]) {
            vm_load<VEC>(in, row_off(in.s, rrow[u]) + col_off(in.s), cs, &w[i][u * VEC]);
          } else {
#pragma unroll
            for (int j = 0; j < VEC; ++j) w[i][u * VEC + j] = 0.f;
          }
        }
      }
      T::template exec<RPI * VEC>(w);
#pragma unroll
      for (int s2 = 0; s2 < T::Stores::n; ++s2) {
        const EwDevOut& o = p.out[s2];
        const int64_t cs = o.s[nd - 1];
#pragma unroll
        for (int u = 0; u < RPI; ++u)
          if (vrow[u]) vm_store<VEC>(o, row_off(o.s, rrow[u]) + col_off(o.s), cs, &w[T::Stores::at(s2)][u * VEC]);
      }
#pragma unroll
      for (int q = 0; q < NRS; ++q) {
#pragma unroll
        for (int u = 0; u < RPI; ++u) {
          if (!vrow[u]) continue;
          if (T::Reds::at(2 * q + 1) == RED_ROW) {
            float s3 = 0.f;
#pragma unroll
            for (int j = 0; j < VEC; ++j) s3 = __fadd_rn(s3, w[T::Reds::at(2 * q)][u * VEC + j]);
            rowv[u][q] = s3;
          } else {
#pragma unroll
            for (int j = 0; j < VEC; ++j) acc[q][j] = __fadd_rn(acc[q][j], w[T::Reds::at(2 * q)][u * VEC + j]);
          }
        }
      }
    } else {
      if (vrow[0]) {
        const int64_t r = rrow[0];
        for (int i = 0; i < n_in; ++i) {
          const EwDevIn& in = p.in[i];
          vm_load<VEC>(in, row_off(in.s, r) + col_off(in.s), in.s[nd - 1], v[i]);
        }
        vm_exec<VEC>(Pg, v);
        for (int s2 = 0; s2 < Pg.n_stores; ++s2) {
          const EwDevOut& o = p.out[s2];
          vm_store<VEC>(o, row_off(o.s, r) + col_off(o.s), o.s[nd - 1], v[Pg.store_slot[s2]]);
        }
        for (int q = 0; q < n_red; ++q) {
          const float* x = v[Pg.reduce_slot[q]];
          if (Pg.reduce_kind[q] == RED_ROW) {
            float s3 = 0.f;
#pragma unroll
            for (int j = 0; j < VEC; ++j) s3 = __fadd_rn(s3, x[j]);
            rowv[0][q] = s3;
          } else {
#pragma unroll
            for (int j = 0; j < VEC; ++j) acc[q][j] = __fadd_rn(acc[q][j], x[j]);
          }
        }
      }
    }
    if (has_row) {  // block-uniform: every thread takes part
#pragma unroll
      for (int u = 0; u < RPI; ++u) {
#pragma unroll
        for (int q = 0; q < NRS; ++q) {
          if (q >= nred || red_kind(q) != RED_ROW) continue;
          float s3 = warp_sum(rowv[u][q]);
          if ((tx & 31) == 0) row_s[ty][tx >> 5] = s3;
          __syncthreads();
          if (tx == 0 && (k + u) < p.rpt && rrow[u] < R) {
            float t = 0.f;
            for (int w2 = 0; w2 < (bx >> 5); ++w2) t = __fadd_rn(t, row_s[ty][w2]);
            p.red[q][rrow[u] * p.gx + blockIdx.x] = t;
          }
          __syncthreads();
        }
      }
    }
  }
  if (!has_colall) return;
#pragma unroll
  for (int q = 0; q < NRS; ++q) {
    if (q >= nred) break;
    const int kind = red_kind(q);
    if (kind == RED_ROW) continue;
    if (kind == RED_COL) {
#pragma unroll
      for (int j = 0; j < VEC; ++j) red_s[(ty * bx + tx) * VEC + j] = acc[q][j];
      __syncthreads();
      if (ty == 0 && cval) {
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
          float t = 0.f;
          for (int y = 0; y < by; ++y) t = __fadd_rn(t, red_s[(y * bx + tx) * VEC + j]);
          if (VEC == 1 || c + j < C) p.red[q][blockIdx.y * C + c + j] = t;
        }
      }
      __syncthreads();
    } else {  // RED_ALL
      float t = 0.f;
#pragma unroll
      for (int j = 0; j < VEC; ++j) t = __fadd_rn(t, acc[q][j]);
      t = warp_sum(t);
      const int lin = ty * bx + tx;
      if ((lin & 31) == 0) red_s[lin >> 5] = t;
      __syncthreads();
      if (lin == 0) {
        float u = 0.f;
        for (int w = 0; w < (bx * by) >> 5; ++w) u = __fadd_rn(u, red_s[w]);
        p.red[q][blockIdx.y * p.gx + blockIdx.x] = u;
      }
      __syncthreads();
    }
  }
}

// Deterministic finalize of reduction partials: out[e] = sum_k P[k*cs + e*es]
// in a fixed order (threadIdx.y strides the chunks, then a fixed-order sum
// over threadIdx.y), written to every home of the reduced value.
__global__ void __launch_bounds__(256) finalize_kernel(const __grid_constant__ EwParams p) {
  pdl_trigger();
  pdl_wait();
  __shared__ float part[256];
  const int ex = blockDim.x, cy = blockDim.y;
  const int64_t e = (int64_t)blockIdx.x * ex + threadIdx.x;
  const EwDevIn& in = p.in[0];
  const float* P = reinterpret_cast<const float*>(in.ptr);
  float s = 0.f;
  if (e < p.dims[0]) {
    const float* q = P + e * in.s[0];
    int k = threadIdx.y;
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    for (; k + 3 * cy < in.nchunks; k += 4 * cy) {
      a0 = __fadd_rn(a0, __ldg(q + (int64_t)k * in.chunk_stride));
      a1 = __fadd_rn(a1, __ldg(q + (int64_t)(k + cy) * in.chunk_stride));
      a2 = __fadd_rn(a2, __ldg(q + (int64_t)(k + 2 * cy) * in.chunk_stride));
      a3 = __fadd_rn(a3, __ldg(q + (int64_t)(k + 3 * cy) * in.chunk_stride));
    }
    for (; k < in.nchunks; k += cy) a0 = __fadd_rn(a0, __ldg(q + (int64_t)k * in.chunk_stride));
    s = __fadd_rn(__fadd_rn(a0, a1), __fadd_rn(a2, a3));
  }
  part[threadIdx.y * ex + threadIdx.x] = s;
  __syncthreads();
  for (int w = cy / 2; w > 0; w >>= 1) {  // fixed-order tree over threadIdx.y
    if (threadIdx.y < w) part[threadIdx.y * ex + threadIdx.x] =
        __fadd_rn(part[threadIdx.y * ex + threadIdx.x], part[(threadIdx.y + w) * ex + threadIdx.x]);
    __syncthreads();
  }
  if (threadIdx.y == 0 && e < p.dims[0]) {
    const float t = part[threadIdx.x];
    for (int o = 0; o < p.prog.n_stores; ++o) st1(p.out[o].ptr, e * p.out[o].s[0], p.out[o].st, t);
  }
}

// 2-D specialised fast path ([R, C], row-major refs, no row reductions):
// per-thread column pointers advanced by one row stride per step, operands
// that do not depend on the row (bias / scale vectors, scalars) loaded once,
// RPI rows loaded before they are computed.  Same arithmetic as ew_kernel.
template <int VEC, class P>
__global__ void __launch_bounds__(256, 3) ew2d_kernel(const __grid_constant__ EwParams p) {
  pdl_trigger();
  pdl_wait();
  using T = spec::Traits<P>;
  constexpr int NS = T::kSlots, NI = T::kIn > 0 ? T::kIn : 1;
  constexpr int NR = T::Reds::n > 0 ? T::Reds::n : 1;
  constexpr int RPI = 2;
  const EwProgram& Pg = p.prog;
  const int tx = threadIdx.x, ty = threadIdx.y, bx = blockDim.x, by = blockDim.y;
  const int64_t C = p.dims[1], R = p.dims[0];
  const int64_t c = ((int64_t)blockIdx.x * bx + tx) * VEC;
  const bool cval = c < C;
  const int64_t r0 = (int64_t)blockIdx.y * p.rpt * by + ty;
  float acc[NR][VEC];
#pragma unroll
  for (int q = 0; q < NR; ++q)
#pragma unroll
    for (int j = 0; j < VEC; ++j) acc[q][j] = 0.f;
  float inv[NI][VEC];  // row-invariant operands
  bool rinv[NI];
#pragma unroll
  for (int i = 0; i < T::kIn; ++i) {
    rinv[i] = p.in[i].s[0] == 0;
    if (rinv[i] && cval) vm_load<VEC>(p.in[i], c * p.in[i].s[1], p.in[i].s[1], inv[i]);
  }
  if (cval) {
    for (int k = 0; k < p.rpt; k += RPI) {
      float w[NS][RPI * VEC];
#pragma unroll
      for (int i = 0; i < T::kLit; ++i)
#pragma unroll
        for (int j = 0; j < RPI * VEC; ++j) w[T::kIn + i][j] = Pg.lits[i];
      int64_t rr[RPI];
      bool ok[RPI];
#pragma unroll
      for (int u = 0; u < RPI; ++u) {
        rr[u] = r0 + (int64_t)(k + u) * by;
        ok[u] = (k + u) < p.rpt && rr[u] < R;
      }
#pragma unroll
      for (int i = 0; i < T::kIn; ++i) {
        const EwDevIn& in = p.in[i];
#pragma unroll
        for (int u = 0; u < RPI; ++u) {
          if (rinv[i]) {
#pragma unroll
            for (int j = 0; j < VEC; ++j) w[i][u * VEC + j] = inv[i][j];
          } else if (ok[u]) {
            vm_load<VEC>(in, rr[u] * in.s[0] + c * in.s[1], in.s[1], &w[i][u * VEC]);
          } else {
#pragma unroll
            for (int j = 0; j < VEC; ++j) w[i][u * VEC + j] = 0.f;
          }
        }
      }
      T::template exec<RPI * VEC>(w);
#pragma unroll
      for (int s2 = 0; s2 < T::Stores::n; ++s2) {
        const EwDevOut& o = p.out[s2];
#pragma unroll
        for (int u = 0; u < RPI; ++u)
          if (ok[u]) vm_store<VEC>(o, rr[u] * o.s[0] + c * o.s[1], o.s[1], &w[T::Stores::at(s2)][u * VEC]);
      }
#pragma unroll
      for (int q = 0; q < T::Reds::n; ++q)
#pragma unroll
        for (int u = 0; u < RPI; ++u)
          if (ok[u])
#pragma unroll
            for (int j = 0; j < VEC; ++j) acc[q][j] = __fadd_rn(acc[q][j], w[T::Reds::at(2 * q)][u * VEC + j]);
    }
  }
  __shared__ float red_s[256 * 4];
#pragma unroll
  for (int q = 0; q < T::Reds::n; ++q) {
    if (T::Reds::at(2 * q + 1) == RED_COL) {
#pragma unroll
      for (int j = 0; j < VEC; ++j) red_s[(ty * bx + tx) * VEC + j] = acc[q][j];
      __syncthreads();
      if (ty == 0 && cval) {
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
          float t = 0.f;
          for (int y = 0; y < by; ++y) t = __fadd_rn(t, red_s[(y * bx + tx) * VEC + j]);
          if (VEC == 1 || c + j < C) p.red[q][blockIdx.y * C + c + j] = t;
        }
      }
      __syncthreads();
    } else {  // RED_ALL
      float t = 0.f;
#pragma unroll
      for (int j = 0; j < VEC; ++j) t = __fadd_rn(t, acc[q][j]);
      t = warp_sum(t);
      const int lin = ty * bx + tx;
      if ((lin & 31) == 0) red_s[lin >> 5] = t;
      __syncthreads();
      if (lin == 0) {
        float u2 = 0.f;
        for (int w2 = 0; w2 < (bx * by) >> 5; ++w2) u2 = __fadd_rn(u2, red_s[w2]);
        p.red[q][blockIdx.y * p.gx + blockIdx.x] = u2;
      }
      __syncthreads();
    }
  }
}

template <class P>
constexpr bool has_row_red() {
  using T = spec::Traits<P>;
  for (int q = 0; q < T::Reds::n; ++q)
    if (T::Reds::at(2 * q + 1) == RED_ROW) return true;
  return false;
}

__global__ void cast_bf16_kernel(const float* __restrict__ src, unsigned short* __restrict__ dst, int64_t n) {
  pdl_trigger();
  pdl_wait();
  int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
  for (; i + 3 < n; i += stride) {
    float4 x = __ldg(reinterpret_cast<const float4*>(src + i));
    uint2 o;
    o.x = (unsigned)f2bf(x.x) | ((unsigned)f2bf(x.y) << 16);
    o.y = (unsigned)f2bf(x.z) | ((unsigned)f2bf(x.w) << 16);
    *reinterpret_cast<uint2*>(dst + i) = o;
  }
  for (; i < n; ++i) dst[i] = f2bf(src[i]);
}

template <int VEC, class P>
cudaError_t launch_spec_ew(const EwParams& p, int bx, int by, cudaStream_t stream) {
  dim3 grid((unsigned)p.gx, (unsigned)p.gy), block(bx, by);
  if constexpr (!has_row_red<P>()) {
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

cudaError_t launch_finalize(const EwParams& p, cudaStream_t stream) {
  const int64_t n = p.dims[0];
  dim3 block = n >= 32 ? dim3(32, 8) : dim3(1, 256);
  dim3 grid((unsigned)((n + block.x - 1) / block.x));
  LaunchCfg L(grid, block, 0, stream);
  cudaError_t e = cudaLaunchKernelEx(&L.cfg, finalize_kernel, p);
  return e != cudaSuccess ? e : cudaGetLastError();
}

__global__ void pack_bf16_kernel(const void* __restrict__ src, int src_f32, int64_t rows, int64_t cols,
                                 unsigned short* __restrict__ dst, int64_t ld) {
  pdl_trigger();
  pdl_wait();
  const int64_t r = blockIdx.y * (int64_t)blockDim.y + threadIdx.y;
  if (r >= rows) return;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ld; c += (int64_t)gridDim.x * blockDim.x) {
    unsigned short v = 0;
    if (c < cols)
      v = src_f32 ? f2bf(__ldg(reinterpret_cast<const float*>(src) + r * cols + c))
                  : __ldg(reinterpret_cast<const unsigned short*>(src) + r * cols + c);
    dst[r * ld + c] = v;
  }
}

cudaError_t launch_pack_bf16(const void* src, bool src_f32, int64_t rows, int64_t cols, void* dst, int64_t ld,
                             cudaStream_t stream) {
  dim3 block(128, 4), grid((unsigned)std::min<int64_t>((ld + 127) / 128, 8), (unsigned)((rows + 3) / 4));
  LaunchCfg L(grid, block, 0, stream);
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
