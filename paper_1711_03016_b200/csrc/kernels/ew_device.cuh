// Device side of the element-wise program: op semantics, loads, stores,
// program interpretation.  Shared by the EW kernel and both GEMM epilogues.
//
// Arithmetic follows the IR's op definitions in fp32 (Table 1
// L170-181) with IEEE round-to-nearest: explicit __f*_rn intrinsics
// (the compiler never contracts; the planner emits VM_FMA where it wants one
// rounding for a*b + c, so every program evaluates identically wherever it
// runs), accurate expf/tanhf/logf/powf (no tanh.approx / ex2.approx:
// reading A13), no flush-to-zero.  sech2 is the cancellation-free tanh
// derivative (reading A12).
#pragma once

#include <cuda_bf16.h>

#include "kernels.h"

namespace dlvm {

// sech^2(z) = 4 t / (1 + t)^2 with t = exp(-2|z|) in (0, 1]: no cancellation,
// relative error a few ulp (expf <= 2 ulp, __fdividef <= 2 ulp for the
// denominator range [1, 4] here), far inside the 1e-5 tolerance (reading A12).
__device__ __forceinline__ float vm_sech2(float z) {
  float t = expf(-2.0f * fabsf(z));
  float d = __fadd_rn(1.0f, t);
  return __fdividef(__fmul_rn(4.0f, t), __fmul_rn(d, d));
}

__device__ __forceinline__ float vm_apply(uint8_t op, float a, float b, float c) {
  switch (op) {
    case VM_NEG: return -a;
    case VM_TANH: return tanhf(a);
    case VM_EXP: return expf(a);
    case VM_LOG: return logf(a);
    case VM_SQRT: return __fsqrt_rn(a);
    case VM_ABS: return fabsf(a);
    case VM_SIGN: return a > 0.f ? 1.f : (a < 0.f ? -1.f : (a == 0.f ? 0.f : a));
    case VM_ADD: return __fadd_rn(a, b);
    case VM_SUB: return __fsub_rn(a, b);
    case VM_MUL: return __fmul_rn(a, b);
    case VM_DIV: return __fdiv_rn(a, b);
    case VM_POW: return powf(a, b);
    case VM_LT: return a < b ? 1.f : 0.f;
    case VM_LE: return a <= b ? 1.f : 0.f;
    case VM_GT: return a > b ? 1.f : 0.f;
    case VM_GE: return a >= b ? 1.f : 0.f;
    case VM_EQ: return a == b ? 1.f : 0.f;
    case VM_NE: return a != b ? 1.f : 0.f;
    case VM_SELECT: return a != 0.f ? b : c;
    case VM_TOBOOL: return a != 0.f ? 1.f : 0.f;
    case VM_COPY: return a;
    case VM_SECH2: return vm_sech2(a);
    case VM_FMA: return __fmaf_rn(a, b, c);
    default: return 0.f;
  }
}

__device__ __forceinline__ float ld1(const void* p, int64_t off, uint8_t st) {
  if (st == (uint8_t)SType::F32) return __ldg(reinterpret_cast<const float*>(p) + off);
  if (st == (uint8_t)SType::BF16) {
    unsigned short u = __ldg(reinterpret_cast<const unsigned short*>(p) + off);
    return __uint_as_float(((unsigned)u) << 16);
  }
  return __ldg(reinterpret_cast<const unsigned char*>(p) + off) ? 1.f : 0.f;
}

__device__ __forceinline__ void ld4(const void* p, int64_t off, uint8_t st, float* v) {
  if (st == (uint8_t)SType::F32) {
    float4 x = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p) + off));
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
  } else if (st == (uint8_t)SType::BF16) {
    uint2 x = __ldg(reinterpret_cast<const uint2*>(reinterpret_cast<const unsigned short*>(p) + off));
    v[0] = __uint_as_float(x.x << 16);
    v[1] = __uint_as_float(x.x & 0xffff0000u);
    v[2] = __uint_as_float(x.y << 16);
    v[3] = __uint_as_float(x.y & 0xffff0000u);
  } else {
    unsigned x = __ldg(reinterpret_cast<const unsigned*>(reinterpret_cast<const unsigned char*>(p) + off));
    v[0] = (x & 0xffu) ? 1.f : 0.f;
    v[1] = (x & 0xff00u) ? 1.f : 0.f;
    v[2] = (x & 0xff0000u) ? 1.f : 0.f;
    v[3] = (x & 0xff000000u) ? 1.f : 0.f;
  }
}

__device__ __forceinline__ unsigned short f2bf(float f) {
  __nv_bfloat16 h = __float2bfloat16_rn(f);
  return *reinterpret_cast<unsigned short*>(&h);
}

// 4 consecutive f32 (16-byte aligned) added into global memory in one
// vector reduction (sm_90+ red.global.add.v4.f32), local or peer
__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

__device__ __forceinline__ void st1(void* p, int64_t off, uint8_t st, float v) {
  if (st == (uint8_t)SType::F32)
    reinterpret_cast<float*>(p)[off] = v;
  else if (st == (uint8_t)SType::F32_ADD)  // accumulate (red.global.add; may be peer memory)
    atomicAdd(reinterpret_cast<float*>(p) + off, v);
  else if (st == (uint8_t)SType::BF16)
    reinterpret_cast<unsigned short*>(p)[off] = f2bf(v);
  else
    reinterpret_cast<unsigned char*>(p)[off] = v != 0.f ? 1 : 0;
}

__device__ __forceinline__ void st4(void* p, int64_t off, uint8_t st, const float* v) {
  if (st == (uint8_t)SType::F32) {
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(p) + off) = make_float4(v[0], v[1], v[2], v[3]);
  } else if (st == (uint8_t)SType::F32_ADD) {  // one 16-byte vector reduction
    red_add_v4(reinterpret_cast<float*>(p) + off, v[0], v[1], v[2], v[3]);
  } else if (st == (uint8_t)SType::BF16) {
    uint2 x;
    x.x = (unsigned)f2bf(v[0]) | ((unsigned)f2bf(v[1]) << 16);
    x.y = (unsigned)f2bf(v[2]) | ((unsigned)f2bf(v[3]) << 16);
    *reinterpret_cast<uint2*>(reinterpret_cast<unsigned short*>(p) + off) = x;
  } else {
    unsigned x = (v[0] != 0.f ? 1u : 0u) | (v[1] != 0.f ? 0x100u : 0u) | (v[2] != 0.f ? 0x10000u : 0u) |
                 (v[3] != 0.f ? 0x1000000u : 0u);
    *reinterpret_cast<unsigned*>(reinterpret_cast<unsigned char*>(p) + off) = x;
  }
}

// load input `in` at element offset `off` (column stride cs) into v[0..VEC)
template <int VEC>
__device__ __forceinline__ void vm_load(const EwDevIn& in, int64_t off, int64_t cs, float* v) {
  if (in.nchunks > 1 && in.chunk_op == 0 && VEC == 4 && cs == 1 && in.chunk_stride % 4 == 0) {
    // sum of partials (split-K, reductions), four contiguous columns per
    // load: one 16-byte load per chunk, several chunks in flight, summed in
    // chunk order per column (the same order as the scalar path below)
    float s[4] = {0.f, 0.f, 0.f, 0.f};
    for (int k = 0; k < in.nchunks; k += 4) {
      float x[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (k + u < in.nchunks) ld4(in.ptr, off + (k + u) * in.chunk_stride, in.st, x[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (k + u < in.nchunks)
#pragma unroll
          for (int j = 0; j < 4; ++j) s[j] = __fadd_rn(s[j], x[u][j]);
    }
#pragma unroll
    for (int j = 0; j < VEC; ++j) v[j] = s[j];
    return;
  }
  if (in.nchunks > 1) {
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      float s;
      if (in.chunk_op == 1) {  // product over the reduced axis, in index order
        s = 1.f;
        for (int k = 0; k < in.nchunks; ++k) s = __fmul_rn(s, ld1(in.ptr, off + j * cs + k * in.chunk_stride, in.st));
      } else if (in.chunk_op == 2) {  // maximum over the reduced axis (a NaN wins, like numpy)
        s = ld1(in.ptr, off + j * cs, in.st);
        for (int k = 1; k < in.nchunks; ++k) {
          const float x = ld1(in.ptr, off + j * cs + k * in.chunk_stride, in.st);
          s = (x > s || x != x) ? x : s;
        }
      } else {
        s = 0.f;
        for (int k = 0; k < in.nchunks; ++k) s = __fadd_rn(s, ld1(in.ptr, off + j * cs + k * in.chunk_stride, in.st));
      }
      v[j] = s;
    }
    return;
  }
  if (VEC == 4 && cs == 1) {
    ld4(in.ptr, off, in.st, v);
  } else if (cs == 0) {
    float x = ld1(in.ptr, off, in.st);
#pragma unroll
    for (int j = 0; j < VEC; ++j) v[j] = x;
  } else {
#pragma unroll
    for (int j = 0; j < VEC; ++j) v[j] = ld1(in.ptr, off + j * cs, in.st);
  }
}

template <int VEC>
__device__ __forceinline__ void vm_store(const EwDevOut& o, int64_t off, int64_t cs, const float* v) {
  if (VEC == 4 && cs == 1) {
    st4(o.ptr, off, o.st, v);
  } else {
#pragma unroll
    for (int j = 0; j < VEC; ++j) st1(o.ptr, off + j * cs, o.st, v[j]);
  }
}

// run the instruction list over slots (inputs/literals already in place)
template <int VEC>
__device__ __forceinline__ void vm_exec(const EwProgram& P, float (*v)[VEC]) {
  const int base = P.n_in + P.n_lits;
  for (int k = 0; k < P.n_ins; ++k) {
    const EwIns I = P.ins[k];
#pragma unroll
    for (int j = 0; j < VEC; ++j) v[base + k][j] = vm_apply(I.op, v[I.a][j], v[I.b][j], v[I.c][j]);
  }
}

}  // namespace dlvm
