#pragma once
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
// Device code only: compiled ahead of time (gemm_simt.cu) and at create time
// by NVRTC for epilogue programs outside the registry (csrc/jit.cpp).
#include <cooperative_groups.h>

#include "ew_kernels.cuh"

namespace dlvm {
namespace kern {
namespace simt {

namespace cg = cooperative_groups;

constexpr int BN = 64, BK = 16;

template <bool BF16>
__device__ __forceinline__ float ldop(const void* p, int64_t off) {
  if (BF16) return __uint_as_float(((unsigned)__ldg(reinterpret_cast<const unsigned short*>(p) + off)) << 16);
  return __ldg(reinterpret_cast<const float*>(p) + off);
}

struct SimtVm {};  // epilogue program interpreted from GemmParams::epi.prog

// program shape: compile-time for a spec::Prog, from the parameters for SimtVm
template <class PROG>
struct EpiShape {
  using T = spec::Traits<PROG>;
  static constexpr bool kSpec = true;
  static constexpr int kSlots = T::kSlots, kChunk = 0;  // 0: all of a thread's outputs at once
  __device__ static constexpr int n_in(const EwProgram&) { return T::kIn; }
  __device__ static constexpr int n_lits(const EwProgram&) { return T::kLit; }
  __device__ static constexpr int n_stores(const EwProgram&) { return T::Stores::n; }
  __device__ static constexpr int store_slot(const EwProgram&, int k) { return T::Stores::at(k); }
  __device__ static constexpr int n_reduces(const EwProgram&) { return T::Reds::n; }
  __device__ static constexpr int reduce_slot(const EwProgram&, int q) { return T::Reds::at(2 * q); }
  __device__ static constexpr int reduce_kind(const EwProgram&, int q) { return T::Reds::at(2 * q + 1); }
  template <int E>
  __device__ static void exec(const EwProgram&, float (&v)[kSlots][E]) { T::template exec<E>(v); }
};
template <>
struct EpiShape<SimtVm> {
  static constexpr bool kSpec = false;
  static constexpr int kSlots = kMaxSlots, kChunk = 4;
  __device__ static int n_in(const EwProgram& P) { return P.n_in; }
  __device__ static int n_lits(const EwProgram& P) { return P.n_lits; }
  __device__ static int n_stores(const EwProgram& P) { return P.n_stores; }
  __device__ static int store_slot(const EwProgram& P, int k) { return P.store_slot[k]; }
  __device__ static int n_reduces(const EwProgram& P) { return P.n_reduces; }
  __device__ static int reduce_slot(const EwProgram& P, int q) { return P.reduce_slot[q]; }
  __device__ static int reduce_kind(const EwProgram& P, int q) { return P.reduce_kind[q]; }
  template <int E>
  __device__ static void exec(const EwProgram& P, float (&v)[kSlots][E]) { vm_exec<E>(P, v); }
};

// epilogue over E outputs of one thread: rows m[r] (E/4 rows), columns
// n0c..n0c+3 each; slot 0 = accumulator values; reduction values -> rv
template <class S, int E>
__device__ __forceinline__ void simt_epilogue(const GemmParams& p, const int64_t* m, int64_t n0c, const float* acc,
                                              float (*rv)[E]) {
  const EwParams& Ep = p.epi;
  const EwProgram& Pg = Ep.prog;
  constexpr int R = E / 4;
  const bool full4 = n0c + 3 < p.N;
  float v[S::kSlots][E];
#pragma unroll
  for (int e = 0; e < E; ++e) v[0][e] = acc[e];
#pragma unroll
  for (int s = 1; s < (S::kSpec ? S::n_in(Pg) : kMaxIn); ++s) {
    if (!S::kSpec && s >= S::n_in(Pg)) break;
    const EwDevIn& in = Ep.in[s];
    const bool vec_ok = full4 && in.nchunks == 1 && in.s[1] == 1 && (in.s[0] & 3) == 0 &&
                        (reinterpret_cast<uintptr_t>(in.ptr) & 15) == 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (m[r] >= p.M) {
#pragma unroll
        for (int j = 0; j < 4; ++j) v[s][r * 4 + j] = 0.f;
        continue;
      }
      const int64_t off = m[r] * in.s[0] + n0c * in.s[1];
      if (vec_ok) {
        vm_load<4>(in, off, 1, &v[s][r * 4]);
      } else if (in.nchunks > 1) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (n0c + j < p.N) vm_load<1>(in, off + j * in.s[1], 0, &v[s][r * 4 + j]);
          else v[s][r * 4 + j] = 0.f;
      } else if (in.st == (uint8_t)SType::F32) {  // type switch outside the loop:
        const float* q = reinterpret_cast<const float*>(in.ptr) + off;  // independent loads
#pragma unroll
        for (int j = 0; j < 4; ++j) v[s][r * 4 + j] = n0c + j < p.N ? __ldg(q + j * in.s[1]) : 0.f;
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) v[s][r * 4 + j] = n0c + j < p.N ? ld1(in.ptr, off + j * in.s[1], in.st) : 0.f;
      }
    }
  }
  const int nin = S::n_in(Pg);
#pragma unroll
  for (int l = 0; l < (S::kSpec ? S::n_lits(Pg) : kMaxLits); ++l) {
    if (!S::kSpec && l >= S::n_lits(Pg)) break;
#pragma unroll
    for (int e = 0; e < E; ++e) v[nin + l][e] = Pg.lits[l];
  }
  S::template exec<E>(Pg, v);
#pragma unroll
  for (int k = 0; k < (S::kSpec ? S::n_stores(Pg) : kMaxStores); ++k) {
    if (!S::kSpec && k >= S::n_stores(Pg)) break;
    const EwDevOut& o = Ep.out[k];
    const int slot = S::store_slot(Pg, k);
    const bool vec_ok = full4 && o.s[1] == 1 && (o.s[0] & 3) == 0 && (reinterpret_cast<uintptr_t>(o.ptr) & 15) == 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (m[r] >= p.M) continue;
      const int64_t off = m[r] * o.s[0] + n0c * o.s[1];
      if (vec_ok) {
        vm_store<4>(o, off, 1, &v[slot][r * 4]);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (n0c + j < p.N) st1(o.ptr, off + j * o.s[1], o.st, v[slot][r * 4 + j]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < (S::kSpec ? S::n_reduces(Pg) : kMaxReduces); ++q) {
    if (!S::kSpec && q >= S::n_reduces(Pg)) break;
    const int slot = S::reduce_slot(Pg, q);
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int j = 0; j < 4; ++j) rv[q][r * 4 + j] = (m[r] < p.M && n0c + j < p.N) ? v[slot][r * 4 + j] : 0.f;
  }
}

// K per batch staged through registers (one K tile: deeper batches measured
// no faster on c1's latency-bound shapes, tools/simt_probe.py)
constexpr int KB = BK;

template <bool BF16, int BM, class PROG>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const __grid_constant__ GemmParams p, int64_t kchunk) {
  pdl_trigger();
  pdl_wait();
  using S = EpiShape<PROG>;
  constexpr int TM = BM / 16;
  constexpr int NA = BM * KB / 256, NB = KB * BN / 256;
  __shared__ float As[KB][BM + 4];
  __shared__ float Bs[KB][BN + 4];
  __shared__ float red_t[BM][BN + 1];
  __shared__ float part[4][BN];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  float acc[TM][4];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  // K segments (sums of products, one accumulator); a split K (cluster)
  // applies to single-segment GEMMs
  for (int q = 0; q < p.n_seg; ++q) {
    const GemmSegParams& G = p.seg[q];
    const int64_t kb = gridDim.z > 1 ? (int64_t)blockIdx.z * kchunk : 0;
    const int64_t ke = gridDim.z > 1 ? (kb + kchunk < G.K ? kb + kchunk : G.K) : G.K;
    // element e of the A batch (BM x KB) / B batch (KB x BN), in the operand's
    // contiguous order so consecutive threads read consecutive addresses
    auto a_idx = [&](int e, int& kk, int& mm) {
      if (G.a_kmajor) { kk = e % KB; mm = e / KB; } else { mm = e % BM; kk = e / BM; }
    };
    auto b_idx = [&](int e, int& kk, int& nn) {
      if (G.b_kmajor) { kk = e % KB; nn = e / KB; } else { nn = e % BN; kk = e / BN; }
    };
    float ra[NA], rb[NB];
    auto load = [&](int64_t k0) {
#pragma unroll
      for (int i = 0; i < NA; ++i) {
        int kk, mm;
        a_idx(tid + i * 256, kk, mm);
        const int64_t gm = m0 + mm, gk = k0 + kk;
        ra[i] = (gm < p.M && gk < ke) ? ldop<BF16>(G.a, gm * G.a_s0 + gk * G.a_s1) : 0.f;
      }
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        int kk, nn;
        b_idx(tid + i * 256, kk, nn);
        const int64_t gn = n0 + nn, gk = k0 + kk;
        rb[i] = (gn < p.N && gk < ke) ? ldop<BF16>(G.b, gk * G.b_s0 + gn * G.b_s1) : 0.f;
      }
    };
    if (kb < ke) load(kb);
    for (int64_t k0 = kb; k0 < ke; k0 += KB) {
#pragma unroll
      for (int i = 0; i < NA; ++i) {
        int kk, mm;
        a_idx(tid + i * 256, kk, mm);
        As[kk][mm] = ra[i];
      }
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        int kk, nn;
        b_idx(tid + i * 256, kk, nn);
        Bs[kk][nn] = rb[i];
      }
      __syncthreads();
      if (k0 + KB < ke) load(k0 + KB);  // in flight while this tile's FMAs run
      const int kn = ke - k0 < KB ? (int)(ke - k0) : KB;
#pragma unroll 4
      for (int kk = 0; kk < kn; ++kk) {
        float a[TM], b[4];
#pragma unroll
        for (int i = 0; i < TM; ++i) a[i] = As[kk][ty * TM + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      }
      __syncthreads();
    }
  }
  if (gridDim.z > 1) {
    // split K: partial tiles through distributed shared memory, summed by
    // rank 0 in rank order; peers stay resident until rank 0 has read them
    cg::cluster_group cl = cg::this_cluster();
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) red_t[ty * TM + i][tx * 4 + j] = acc[i][j];
    cl.sync();
    const unsigned rank = cl.block_rank();
    if (rank == 0) {
      for (unsigned r = 1; r < gridDim.z; ++r) {
        const float* peer = cl.map_shared_rank(&red_t[0][0], r);
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = __fadd_rn(acc[i][j], peer[(ty * TM + i) * (BN + 1) + tx * 4 + j]);
      }
    }
    cl.sync();
    if (rank != 0) return;
  }
  // epilogue program over the thread's TM x 4 outputs (slot 0 = accumulator)
  const EwParams& E = p.epi;
  const EwProgram& P = E.prog;
  float redv[kMaxReduces][TM * 4];
  const int64_t n0c = n0 + tx * 4;
  if constexpr (S::kSpec) {
    int64_t m[TM];
#pragma unroll
    for (int i = 0; i < TM; ++i) m[i] = m0 + ty * TM + i;
    simt_epilogue<S, TM * 4>(p, m, n0c, &acc[0][0], redv);
  } else {
#pragma unroll 1
    for (int i = 0; i < TM; ++i) {
      int64_t m[1] = {m0 + ty * TM + i};
      float rv[kMaxReduces][4];
      simt_epilogue<S, 4>(p, m, n0c, &acc[i][0], rv);
      for (int q = 0; q < S::n_reduces(P); ++q)
#pragma unroll
        for (int j = 0; j < 4; ++j) redv[q][i * 4 + j] = rv[q][j];
    }
  }
  // epilogue reductions: tile values -> smem -> fixed-order sums
  const int64_t gx = E.gx;
#pragma unroll
  for (int q = 0; q < (S::kSpec ? S::n_reduces(P) : kMaxReduces); ++q) {
    if (!S::kSpec && q >= S::n_reduces(P)) break;
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) red_t[ty * TM + i][tx * 4 + j] = redv[q][i * 4 + j];
    __syncthreads();
    const int kind = S::reduce_kind(P, q);
    // fixed-order sums (deterministic): a warp per row (lane pairs, then a
    // butterfly; lane 0's value is used), or 4 row groups per column added
    // in group order
    const int lane = tid & 31, warp = tid >> 5;
    if (kind == RED_ROW) {
      for (int r = warp; r < BM; r += 8) {
        float s = __fadd_rn(red_t[r][lane], red_t[r][lane + 32]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
        if (lane == 0 && m0 + r < p.M) E.red[q][(m0 + r) * gx + blockIdx.x] = s;
      }
    } else {
      {
        const int c = tid % BN, g = tid / BN;  // 4 groups of BM/4 rows
        float s = 0.f;
#pragma unroll
        for (int r = g * (BM / 4); r < (g + 1) * (BM / 4); ++r) s = __fadd_rn(s, red_t[r][c]);
        part[g][c] = s;
      }
      __syncthreads();
      if (tid < BN) {
        const float s = __fadd_rn(__fadd_rn(part[0][tid], part[1][tid]), __fadd_rn(part[2][tid], part[3][tid]));
        if (kind == RED_COL) {
          if (n0 + tid < p.N) E.red[q][blockIdx.y * p.N + n0 + tid] = s;
        } else {
          part[0][tid] = s;  // column sums of the tile
        }
      }
      if (kind == RED_ALL) {
        __syncthreads();
        if (warp == 0) {
          float s = __fadd_rn(part[0][lane], part[0][lane + 32]);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
          if (lane == 0) E.red[q][blockIdx.y * gx + blockIdx.x] = s;
        }
      }
    }
    __syncthreads();
  }
}

}  // namespace simt
}  // namespace kern
}  // namespace dlvm
