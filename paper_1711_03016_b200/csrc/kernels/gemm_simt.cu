// SIMT GEMM for `dot` (Table 1) under the fp32 policy (exact fp32
// operands, FFMA accumulation; K6 of SURVEY.md §2.5) and for bf16 dots whose
// shapes/strides the tensor-core path cannot take (tiny or TMA-misaligned).
// `transpose` feeding a dot is absorbed as operand strides (A/B may be row-
// or column-major).  64x64 tile, BK = 16, 256 threads x 4x4 outputs; the
// accumulator then runs the fused element-wise epilogue program (bias,
// activation, activation derivative, reductions).
#include "ew_device.cuh"

namespace dlvm {

namespace {

constexpr int BM = 64, BN = 64, BK = 16;

template <bool BF16>
__device__ __forceinline__ float ldop(const void* p, int64_t off) {
  if (BF16) return __uint_as_float(((unsigned)__ldg(reinterpret_cast<const unsigned short*>(p) + off)) << 16);
  return __ldg(reinterpret_cast<const float*>(p) + off);
}

template <bool BF16>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const __grid_constant__ GemmParams p) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  __shared__ float red_t[BM][BN + 1];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  for (int64_t k0 = 0; k0 < p.K; k0 += BK) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int e = tid + i * 256;
      int kk, mm;
      if (p.a_kmajor) { kk = e % BK; mm = e / BK; } else { mm = e % BM; kk = e / BM; }
      int64_t gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < p.M && gk < p.K) ? ldop<BF16>(p.a, gm * p.a_s0 + gk * p.a_s1) : 0.f;
      int nn;
      if (p.b_kmajor) { kk = e % BK; nn = e / BK; } else { nn = e % BN; kk = e / BN; }
      int64_t gn = n0 + nn;
      gk = k0 + kk;
      Bs[kk][nn] = (gn < p.N && gk < p.K) ? ldop<BF16>(p.b, gk * p.b_s0 + gn * p.b_s1) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  // epilogue program on each accumulator element (slot 0)
  const EwParams& E = p.epi;
  const EwProgram& P = E.prog;
  float v[kMaxSlots][1];
  for (int i = 0; i < P.n_lits; ++i) v[P.n_in + i][0] = P.lits[i];
  float redv[kMaxReduces][4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
      const bool ok = m < p.M && n < p.N;
      for (int q = 0; q < kMaxReduces; ++q) redv[q][i][j] = 0.f;
      if (!ok) continue;
      v[0][0] = acc[i][j];
      for (int s = 1; s < P.n_in; ++s) vm_load<1>(E.in[s], m * E.in[s].s[0] + n * E.in[s].s[1], 0, v[s]);
      vm_exec<1>(P, v);
      for (int s = 0; s < P.n_stores; ++s) st1(E.out[s].ptr, m * E.out[s].s[0] + n * E.out[s].s[1], E.out[s].st, v[P.store_slot[s]][0]);
      for (int q = 0; q < P.n_reduces; ++q) redv[q][i][j] = v[P.reduce_slot[q]][0];
    }
  // epilogue reductions: tile values -> smem -> fixed-order sums
  const int64_t gx = E.gx;
  for (int q = 0; q < P.n_reduces; ++q) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) red_t[ty * 4 + i][tx * 4 + j] = redv[q][i][j];
    __syncthreads();
    const uint8_t kind = P.reduce_kind[q];
    if (tid < 64) {
      float s = 0.f;
      if (kind == RED_ROW) {
        for (int c = 0; c < BN; ++c) s = __fadd_rn(s, red_t[tid][c]);
        if (m0 + tid < p.M) E.red[q][(m0 + tid) * gx + blockIdx.x] = s;
      } else {
        for (int r = 0; r < BM; ++r) s = __fadd_rn(s, red_t[r][tid]);
        if (kind == RED_COL) {
          if (n0 + tid < p.N) E.red[q][blockIdx.y * p.N + n0 + tid] = s;
        } else {
          red_t[0][tid] = s;  // column sums, then one thread sums them in order
        }
      }
    }
    __syncthreads();
    if (kind == RED_ALL && tid == 0) {
      float s = 0.f;
      for (int c = 0; c < BN; ++c) s = __fadd_rn(s, red_t[0][c]);
      E.red[q][blockIdx.y * gx + blockIdx.x] = s;
    }
    __syncthreads();
  }
}

}  // namespace

cudaError_t launch_gemm_simt(const GemmParams& p, cudaStream_t stream) {
  dim3 grid((unsigned)((p.N + BN - 1) / BN), (unsigned)((p.M + BM - 1) / BM));
  if (p.bf16)
    gemm_simt_kernel<true><<<grid, 256, 0, stream>>>(p);
  else
    gemm_simt_kernel<false><<<grid, 256, 0, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace dlvm
