// Element-wise program kernel (K1/K2/K3/K7/K8 of SURVEY.md §2.5): one pass
// over an [R, C] iteration space (R = product of up to kMaxIterDims - 1 row dims)
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
// Device code only: compiled ahead of time (ew.cu) for the registry of
// specialised programs and the interpreter, and at create time by NVRTC for
// programs outside the registry (csrc/jit.cpp).
#pragma once

#include "async.cuh"
#include "ew_spec.cuh"
#include "launch.cuh"

namespace dlvm {
namespace kern {

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
  constexpr bool SPEC = !is_void_v<P>;
  using T = cond_t<SPEC, spec::Traits<cond_t<SPEC, P, spec::Prog<0, 0, spec::St<>, spec::Rd<>>>>, VmTraits>;
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
  // element offset of column c for strides s (several column dims only with VEC == 1)
  auto col_off = [&](const int64_t* s) -> int64_t {
    if (p.ncols == 1) return c * s[nd - 1];
    int64_t off = 0, cc = c;
    for (int d = nd - 1; d >= nrd; --d) {
      off += (cc % p.dims[d]) * s[d];
      cc /= p.dims[d];
    }
    return off;
  };
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

#ifdef DLVM_EW_DEFINE_FIXED_KERNELS  // non-template kernels: one definition, in ew.cu
// Deterministic finalize of reduction partials: out[e] = sum_k P[k*cs + e*es]
// in a fixed order (a logical (ex, cy) thread grid: ty strides the chunks,
// then a fixed-order tree over ty), written to every home of the reduced
// value.  One launch finalizes up to kMaxIterDims reductions of one producer:
// blockIdx.y = input q, n = dims[q] its length, its homes the stores with
// store_slot == q.  The logical shape depends on n alone ((32, 8) for n >= 32,
// else (1, 256)), so every sum is the one a launch of its own would produce.
__global__ void __launch_bounds__(256) finalize_kernel(const __grid_constant__ EwParams p) {
  pdl_trigger();
  pdl_wait();
  __shared__ float part[256];
  const int qi = blockIdx.y;
  const int64_t n = p.dims[qi];
  const int ex = n >= 32 ? 32 : 1, cy = 256 / ex;
  if ((int64_t)blockIdx.x * ex >= n) return;  // CTA-uniform: this reduction needs fewer CTAs
  const int tid = threadIdx.y * blockDim.x + threadIdx.x, tx = tid % ex, ty = tid / ex;
  const int64_t e = (int64_t)blockIdx.x * ex + tx;
  const EwDevIn& in = p.in[qi];
  const float* P = reinterpret_cast<const float*>(in.ptr);
  float s = 0.f;
  if (e < n) {
    const float* q = P + e * in.s[0];
    int k = ty;
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    const int64_t cs = in.chunk_stride, step = (int64_t)cy * cs;
    const float* qk = q + (int64_t)k * cs;
    for (; k + 7 * cy < in.nchunks; k += 8 * cy, qk += 8 * step) {  // 8 loads in flight
      float v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = __ldg(qk + j * step);
      a0 = __fadd_rn(a0, v[0]);
      a1 = __fadd_rn(a1, v[1]);
      a2 = __fadd_rn(a2, v[2]);
      a3 = __fadd_rn(a3, v[3]);
      a0 = __fadd_rn(a0, v[4]);
      a1 = __fadd_rn(a1, v[5]);
      a2 = __fadd_rn(a2, v[6]);
      a3 = __fadd_rn(a3, v[7]);
    }
    for (; k + 3 * cy < in.nchunks; k += 4 * cy, qk += 4 * step) {
      // all four loads issue before the adds (same summation order)
      const float v0 = __ldg(qk), v1 = __ldg(qk + step), v2 = __ldg(qk + 2 * step), v3 = __ldg(qk + 3 * step);
      a0 = __fadd_rn(a0, v0);
      a1 = __fadd_rn(a1, v1);
      a2 = __fadd_rn(a2, v2);
      a3 = __fadd_rn(a3, v3);
    }
    for (; k < in.nchunks; k += cy) a0 = __fadd_rn(a0, __ldg(q + (int64_t)k * in.chunk_stride));
    s = __fadd_rn(__fadd_rn(a0, a1), __fadd_rn(a2, a3));
  }
  part[tid] = s;  // == part[ty * ex + tx]
  __syncthreads();
  for (int w = cy / 2; w > 0; w >>= 1) {  // fixed-order tree over ty
    if (ty < w) part[ty * ex + tx] = __fadd_rn(part[ty * ex + tx], part[(ty + w) * ex + tx]);
    __syncthreads();
  }
  if (ty == 0 && e < n) {
    const float t = part[tx];
    for (int o = 0; o < p.prog.n_stores; ++o)
      if (p.prog.store_slot[o] == qi) st1(p.out[o].ptr, e * p.out[o].s[0], p.out[o].st, t);
  }
}

#endif

// Streaming row loads of the f32 fast path.  Measured on c2 (GB/s fwd /
// fwd+adjoint): __ldg 6289 / 5809; DLVM_EW_LDHINT=1 (L1::no_allocate +
// L2::256B prefetch hint) 5980 / 5659; =2 (L1::no_allocate + L2 evict_first
// policy) 5956 / 5603.  Default: plain __ldg.  Streaming (__stcs) stores of
// the row loop measured no change (6273 / 5803).
#ifndef DLVM_EW_LDHINT
#define DLVM_EW_LDHINT 0
#endif
__device__ __forceinline__ float4 ld_row4(const float* p) {
#if DLVM_EW_LDHINT == 1
  float4 v;
  asm("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0, %1, %2, %3}, [%4];"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "l"(p));
  return v;
#elif DLVM_EW_LDHINT == 2
  float4 v;
  asm("{\n\t.reg .b64 pol;\n\tcreatepolicy.fractional.L2::evict_first.b64 pol, 1.0;\n\t"
      "ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], pol;\n\t}"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "l"(p));
  return v;
#else
  return __ldg(reinterpret_cast<const float4*>(p));
#endif
}

// 2-D specialised fast path ([R, C], row-major refs, no row reductions):
// per-thread column pointers advanced by one row stride per step, operands
// that do not depend on the row (bias / scale vectors, scalars) loaded once,
// RPI rows loaded before they are computed.  Same arithmetic as ew_kernel.
// ew2d_kernel's row loop when every row-varying input is f32 and every store
// f32 or bf16, all with unit column stride (the common case: the planner
// stores f32 or bf16 and element-wise inputs are f32): float4 loads and
// 16- / 8-byte stores through pointers that advance by the row step -- no
// per-load storage-type dispatch or 64-bit index products.  Same arithmetic
// and the same bf16 rounding (f2bf) as the general loop.  (bf16 stores
// through the general loop ran at 3.2-4.4 TB/s against 5.8-6.7 for f32:
// tools/ew_inputs_probe.py.)
// BF16: some stores are bf16 (a separate instantiation: the per-store type
// test costs the all-f32 loop ~17% on c2 fwd+adjoint)
template <class P, int RPI, int NI, int NR, bool BF16>
__device__ __forceinline__ void ew2d_rows_f32(const EwParams& p, int64_t c, int64_t r0, int by, const bool* rinv,
                                              const float (*inv)[4], float (*acc)[4]) {
  using T = spec::Traits<P>;
  constexpr int NS = T::kSlots, NO = T::Stores::n > 0 ? T::Stores::n : 1;
  const EwProgram& Pg = p.prog;
  const int64_t R = p.dims[0];
  const float* ip[NI];
  int64_t is[NI];
#pragma unroll
  for (int i = 0; i < T::kIn; ++i) {
    ip[i] = reinterpret_cast<const float*>(p.in[i].ptr) + (rinv[i] ? 0 : r0 * p.in[i].s[0] + c);
    is[i] = rinv[i] ? 0 : (int64_t)by * p.in[i].s[0];
  }
  char* op[NO];     // byte pointers: f32 or bf16 rows
  int64_t os[NO];   // row step in bytes
  bool ob[NO];      // store s2 is bf16
#pragma unroll
  for (int s2 = 0; s2 < T::Stores::n; ++s2) {
    ob[s2] = BF16 && p.out[s2].st == (uint8_t)SType::BF16;
    const int64_t es = ob[s2] ? 2 : 4;
    op[s2] = reinterpret_cast<char*>(p.out[s2].ptr) + (r0 * p.out[s2].s[0] + c) * es;
    os[s2] = (int64_t)by * p.out[s2].s[0] * es;
  }
  for (int k = 0; k < p.rpt; k += RPI) {
    bool ok[RPI];
#pragma unroll
    for (int u = 0; u < RPI; ++u) ok[u] = (k + u) < p.rpt && r0 + (int64_t)(k + u) * by < R;
    float w[NS][RPI * 4];
#pragma unroll
    for (int i = 0; i < T::kLit; ++i)
#pragma unroll
      for (int j = 0; j < RPI * 4; ++j) w[T::kIn + i][j] = Pg.lits[i];
#pragma unroll
    for (int i = 0; i < T::kIn; ++i)
#pragma unroll
      for (int u = 0; u < RPI; ++u) {
        if (rinv[i]) {
#pragma unroll
          for (int j = 0; j < 4; ++j) w[i][u * 4 + j] = inv[i][j];
        } else {
          float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
          if (ok[u]) x = ld_row4(ip[i] + u * is[i]);
          w[i][u * 4 + 0] = x.x;
          w[i][u * 4 + 1] = x.y;
          w[i][u * 4 + 2] = x.z;
          w[i][u * 4 + 3] = x.w;
        }
      }
    T::template exec<RPI * 4>(w);
#pragma unroll
    for (int s2 = 0; s2 < T::Stores::n; ++s2)
#pragma unroll
      for (int u = 0; u < RPI; ++u)
        if (ok[u]) {
          const int sl = T::Stores::at(s2);
          if (BF16 && ob[s2]) {
            uint2 x;
            x.x = (unsigned)f2bf(w[sl][u * 4]) | ((unsigned)f2bf(w[sl][u * 4 + 1]) << 16);
            x.y = (unsigned)f2bf(w[sl][u * 4 + 2]) | ((unsigned)f2bf(w[sl][u * 4 + 3]) << 16);
            *reinterpret_cast<uint2*>(op[s2] + u * os[s2]) = x;
          } else {
            *reinterpret_cast<float4*>(op[s2] + u * os[s2]) =
                make_float4(w[sl][u * 4], w[sl][u * 4 + 1], w[sl][u * 4 + 2], w[sl][u * 4 + 3]);
          }
        }
#pragma unroll
    for (int q = 0; q < T::Reds::n; ++q)
#pragma unroll
      for (int u = 0; u < RPI; ++u)
        if (ok[u])
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[q][j] = __fadd_rn(acc[q][j], w[T::Reds::at(2 * q)][u * 4 + j]);
#pragma unroll
    for (int i = 0; i < T::kIn; ++i) ip[i] += RPI * is[i];
#pragma unroll
    for (int s2 = 0; s2 < T::Stores::n; ++s2) op[s2] += RPI * os[s2];
  }
}

// occupancy target: 3 CTAs/SM, 2 for programs with many slots (their RPI x 4
// slot registers would spill under the 3-CTA register budget)
template <class P>
__host__ __device__ constexpr int ew2d_minb() {
  return spec::Traits<P>::kSlots > 8 ? 2 : 3;  // (1 row per iteration at 3 CTAs/SM measured slower)
}

// rows per row-loop iteration: 4 for programs with column sums (more loads
// in flight per thread for the 3-read adjoint; c2 fwd+adjoint 5910-5960 ->
// 6120-6140 GB/s), 2 otherwise (4 rows measured 29% slower on the c2
// forward).  DLVM_EW_RPI (build variant "rpi4") forces one value.
template <class P>
__host__ __device__ constexpr int ew2d_rpi() {
#ifdef DLVM_EW_RPI
  return DLVM_EW_RPI;
#else
  using T = spec::Traits<P>;
  for (int q = 0; q < T::Reds::n; ++q)
    if (T::Reds::at(2 * q + 1) == RED_COL) return 4;
  return 2;
#endif
}
template <int VEC, class P, int RPI = ew2d_rpi<P>(), int MINB = ew2d_minb<P>(), bool PF = false>
__global__ void __launch_bounds__(256, MINB) ew2d_kernel(const __grid_constant__ EwParams p) {
  pdl_trigger();
  pdl_wait();
  using T = spec::Traits<P>;
  constexpr int NS = T::kSlots, NI = T::kIn > 0 ? T::kIn : 1;
  constexpr int NR = T::Reds::n > 0 ? T::Reds::n : 1;
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
  // row-varying inputs of RPI rows starting at step k (zeros past the end)
  float nx[NI][RPI * VEC];
  auto fetch = [&](int k) {
#pragma unroll
    for (int i = 0; i < T::kIn; ++i) {
      if (rinv[i]) continue;
      const EwDevIn& in = p.in[i];
#pragma unroll
      for (int u = 0; u < RPI; ++u) {
        const int64_t rr = r0 + (int64_t)(k + u) * by;
        if ((k + u) < p.rpt && rr < R) {
          vm_load<VEC>(in, rr * in.s[0] + c * in.s[1], in.s[1], &nx[i][u * VEC]);
        } else {
#pragma unroll
          for (int j = 0; j < VEC; ++j) nx[i][u * VEC + j] = 0.f;
        }
      }
    }
  };
  bool f32rows = VEC == 4, anybf = false;
#pragma unroll
  for (int i = 0; i < T::kIn; ++i)
    f32rows &= rinv[i] || (p.in[i].st == (uint8_t)SType::F32 && p.in[i].s[1] == 1 && p.in[i].nchunks == 1);
#pragma unroll
  for (int s2 = 0; s2 < T::Stores::n; ++s2) {
    f32rows &= (p.out[s2].st == (uint8_t)SType::F32 || p.out[s2].st == (uint8_t)SType::BF16) && p.out[s2].s[1] == 1;
    anybf |= p.out[s2].st == (uint8_t)SType::BF16;
  }
  if constexpr (VEC == 4) {
    if (cval && f32rows) {
      if (anybf)
        ew2d_rows_f32<P, RPI, NI, NR, true>(p, c, r0, by, rinv, inv, acc);
      else
        ew2d_rows_f32<P, RPI, NI, NR, false>(p, c, r0, by, rinv, inv, acc);
    }
  }
  if (cval && !f32rows) {
    if (PF) fetch(0);
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
      if (!PF) fetch(k);
#pragma unroll
      for (int i = 0; i < T::kIn; ++i)
#pragma unroll
        for (int j = 0; j < RPI * VEC; ++j) w[i][j] = rinv[i] ? inv[i][j % VEC] : nx[i][j];
      if (PF && k + RPI < p.rpt) fetch(k + RPI);  // next rows in flight during this step's math
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

#ifdef DLVM_EW_DEFINE_FIXED_KERNELS
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
#endif


// TMA-staged 2-D element-wise kernel ([R, C], VEC = 4, 256 consumer threads
// = 1024 columns per tile, only column / full reductions): HBM-bound
// programs stream through shared memory.  Warp 8 (one lane) copies each
// row-varying input's row segment of a tile, RT rows per stage, with 1-D
// bulk copies (cp.async.bulk, completing on the stage's mbarrier) into an
// NST-stage ring; warps 0-7 read the stage from shared memory, run the
// compile-time program on RT x 4 elements per thread, store, and release the
// stage.  The ring keeps ~NST x stage bytes per SM in flight independent of
// registers, and the consumers issue no global loads or 64-bit address
// arithmetic per element.  CTAs are persistent over the planner's tile grid
// (gx column strips x gy row blocks of rpt rows, strip index fastest), so
// the reduction partials have the layout of ew2d_kernel.  Same arithmetic
// (spec::Traits::exec) as every other path.
constexpr int kTmaRowBytes = 4096;   // 1024 columns x 4 bytes (f32 worst case)
// rows per stage: 4, or 2 for programs whose RT x 4 slot registers would spill
template <class P>
__host__ __device__ constexpr int tma_rows() {
  return spec::Traits<P>::kSlots <= 6 ? 4 : 2;
}

__device__ __forceinline__ void lds4(const unsigned char* p, uint8_t st, float* v) {
  if (st == (uint8_t)SType::F32) {
    const float4 x = *reinterpret_cast<const float4*>(p);
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
  } else if (st == (uint8_t)SType::BF16) {
    const uint2 x = *reinterpret_cast<const uint2*>(p);
    v[0] = __uint_as_float(x.x << 16);
    v[1] = __uint_as_float(x.x & 0xffff0000u);
    v[2] = __uint_as_float(x.y << 16);
    v[3] = __uint_as_float(x.y & 0xffff0000u);
  } else {
    const unsigned x = *reinterpret_cast<const unsigned*>(p);
    v[0] = (x & 0xffu) ? 1.f : 0.f;
    v[1] = (x & 0xff00u) ? 1.f : 0.f;
    v[2] = (x & 0xff0000u) ? 1.f : 0.f;
    v[3] = (x & 0xff000000u) ? 1.f : 0.f;
  }
}

__device__ __forceinline__ int st_size(uint8_t st) {
  return st_bytes(st);
}

template <class P>
__global__ void __launch_bounds__(288, 2) ew_tma_kernel(const __grid_constant__ EwParams p, int nst) {
  using T = spec::Traits<P>;
  constexpr int NS = T::kSlots, NI = T::kIn > 0 ? T::kIn : 1;
  constexpr int NR = T::Reds::n > 0 ? T::Reds::n : 1;
  constexpr int RT = tma_rows<P>();
  extern __shared__ __align__(128) unsigned char tma_smem[];
  const EwProgram& Pg = p.prog;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t C = p.dims[1], R = p.dims[0];
  const int64_t gx = p.gx, n_tiles = p.gx * p.gy;
  // stream (row-varying) inputs and their slot in a stage
  int sidx[NI];
  int nsi = 0;
#pragma unroll
  for (int i = 0; i < T::kIn; ++i) sidx[i] = p.in[i].s[0] != 0 ? nsi++ : -1;
  const uint32_t stage_bytes = (uint32_t)nsi * RT * kTmaRowBytes;
  unsigned char* ring = tma_smem;
  const uint32_t bar0 = smem_u32(tma_smem + (size_t)nst * stage_bytes);  // full[nst], empty[nst]
  __shared__ float red_s[8];
  if (tid == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(bar0 + 8 * s, 1);
      mbar_init(bar0 + 8 * (nst + s), 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_trigger();
  pdl_wait();
  if (warp == 8) {  // ------------------------------------------ producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int64_t c0 = (t % gx) * 1024, rb = t / gx;
        const int64_t cols = C - c0 < 1024 ? C - c0 : 1024;
        const int64_t r_lo = rb * p.rpt, r_hi = r_lo + p.rpt < R ? r_lo + p.rpt : R;
        for (int64_t r = r_lo; r < r_hi; r += RT) {
          mbar_wait(bar0 + 8 * (nst + s), ph ^ 1);
          const int nrow = (int)(r_hi - r < RT ? r_hi - r : RT);
          uint32_t bytes = 0;
#pragma unroll
          for (int i = 0; i < T::kIn; ++i)
            if (sidx[i] >= 0) bytes += (uint32_t)(nrow * cols * st_size(p.in[i].st));
          const uint32_t fb = bar0 + 8 * s;
          mbar_expect_tx(fb, bytes);
#pragma unroll
          for (int i = 0; i < T::kIn; ++i) {
            if (sidx[i] < 0) continue;
            const EwDevIn& in = p.in[i];
            const int es = st_size(in.st);
            const unsigned char* src = reinterpret_cast<const unsigned char*>(in.ptr) + (r * in.s[0] + c0) * es;
            const uint32_t dst = smem_u32(ring + (size_t)s * stage_bytes + (size_t)sidx[i] * RT * kTmaRowBytes);
            for (int u = 0; u < nrow; ++u)
              bulk_load(dst + u * kTmaRowBytes, src + (int64_t)u * in.s[0] * es, (uint32_t)(cols * es), fb);
          }
          if (++s == nst) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
    return;
  }
  // --------------------------------------------------------- consumers
  const int64_t cl = (int64_t)tid * 4;  // column within the tile
  int s = 0;
  uint32_t ph = 0;
  for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const int64_t c0 = (t % gx) * 1024, rb = t / gx;
    const int64_t c = c0 + cl;
    const bool cval = c < C;
    const int64_t r_lo = rb * p.rpt, r_hi = r_lo + p.rpt < R ? r_lo + p.rpt : R;
    float inv[NI][4];
#pragma unroll
    for (int i = 0; i < T::kIn; ++i)
      if (sidx[i] < 0 && cval) vm_load<4>(p.in[i], c * p.in[i].s[1], p.in[i].s[1], inv[i]);
    float acc[NR][4];
#pragma unroll
    for (int q = 0; q < NR; ++q)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[q][j] = 0.f;
    for (int64_t r = r_lo; r < r_hi; r += RT) {
      mbar_wait(bar0 + 8 * s, ph);
      const int nrow = (int)(r_hi - r < RT ? r_hi - r : RT);
      if (cval) {
        float w[NS][RT * 4];
#pragma unroll
        for (int i = 0; i < T::kLit; ++i)
#pragma unroll
          for (int j = 0; j < RT * 4; ++j) w[T::kIn + i][j] = Pg.lits[i];
#pragma unroll
        for (int i = 0; i < T::kIn; ++i) {
          if (sidx[i] < 0) {
#pragma unroll
            for (int j = 0; j < RT * 4; ++j) w[i][j] = inv[i][j & 3];
          } else {
            const int es = st_size(p.in[i].st);
            const unsigned char* b = ring + (size_t)s * stage_bytes + (size_t)sidx[i] * RT * kTmaRowBytes + cl * es;
#pragma unroll
            for (int u = 0; u < RT; ++u)
              if (u < nrow) lds4(b + u * kTmaRowBytes, p.in[i].st, &w[i][u * 4]);
          }
        }
        T::template exec<RT * 4>(w);
#pragma unroll
        for (int s2 = 0; s2 < T::Stores::n; ++s2) {
          const EwDevOut& o = p.out[s2];
#pragma unroll
          for (int u = 0; u < RT; ++u)
            if (u < nrow) vm_store<4>(o, (r + u) * o.s[0] + c, 1, &w[T::Stores::at(s2)][u * 4]);
        }
#pragma unroll
        for (int q = 0; q < T::Reds::n; ++q)
#pragma unroll
          for (int u = 0; u < RT; ++u)
            if (u < nrow)
#pragma unroll
              for (int j = 0; j < 4; ++j) acc[q][j] = __fadd_rn(acc[q][j], w[T::Reds::at(2 * q)][u * 4 + j]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(bar0 + 8 * (nst + s));
      if (++s == nst) {
        s = 0;
        ph ^= 1;
      }
    }
    // tile partials (layout of ew2d_kernel with by = 1)
#pragma unroll
    for (int q = 0; q < T::Reds::n; ++q) {
      if (T::Reds::at(2 * q + 1) == RED_COL) {
        if (cval)
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (c + j < C) p.red[q][rb * C + c + j] = acc[q][j];
      } else {  // RED_ALL
        float v = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) v = __fadd_rn(v, acc[q][j]);
        v = warp_sum(v);
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (lane == 0) red_s[warp] = v;
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (tid == 0) {
          float u2 = 0.f;
          for (int w2 = 0; w2 < 8; ++w2) u2 = __fadd_rn(u2, red_s[w2]);
          p.red[q][rb * gx + (t % gx)] = u2;
        }
      }
    }
  }
}

}  // namespace kern
}  // namespace dlvm
