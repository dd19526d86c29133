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
// Device code only: compiled ahead of time (gemm_tc*.cu) and, for epilogue
// programs outside the registry, at create time by NVRTC (csrc/jit.cpp).
#ifdef __CUDACC_RTC__
// the kernel only passes the descriptor's address to TMA
struct alignas(64) CUtensorMap_st {
  unsigned long long opaque[16];
};
typedef CUtensorMap_st CUtensorMap;
#else
#include <cuda.h>
#endif

#include "ew_kernels.cuh"

namespace dlvm {
namespace kern {

constexpr int BM = 128, BK = 64, STAGES = 4, NUM_THREADS = 384;
constexpr int kTraceSlots = 32;  // u64 trace slots per CTA (trace builds)
constexpr int A_STAGE_BYTES = BM * BK * 2;  // 16 KB

// TMA epilogue (set up by make_params when the program is compile-time
// specialised with 16-column chunks and its operands are TMA-legal):
//  * stores: each epilogue warp writes its 32-row x 64-column column group of
//    every stored value (four 16-column chunks) into its shared-memory
//    staging region, swizzled like the TMA box so the row-per-lane writes
//    are conflict-free, and one lane issues cp.async.bulk.tensor stores
//    (bulk groups) of 64-byte or 128-byte rows.  The TMA unit's cost grows
//    with the number of box rows, so wide rows matter (measured: 16-column
//    boxes cost ~2.3 us per stored value per 128x256 tile);
//  * row-contiguous inputs ([M, N] operands such as the saved ReLU mask) and
//    row-vector inputs ([1, N] biases) of a tile are loaded by warp 3 into a
//    per-tile input buffer (TMA boxes of 128 rows x 128 bytes; a 1-D bulk
//    copy for row vectors) while the tile's MMAs run, completing on
//    in_full[b]; the epilogue warps release it on in_empty[b].
// The pipeline then runs with `nst` stages so everything fits in 227 KB.
constexpr int kEpiTmaIn = 4;  // staged row-contiguous epilogue inputs (tensor maps)
struct EpiTma {
  int32_t on;                   // stores through staging + TMA
  int32_t nst;                  // pipeline stages
  int32_t n_in_bufs;            // 0 (no staged inputs), 1 or 2 per-tile input buffers
  int32_t in_buf_bytes;         // one input buffer
  int8_t in_kind[kMaxIn];       // per input slot: 0 direct, 1 staged [M,N] (map in_map), 2 staged [1,N] row vector
  int8_t in_map[kMaxIn];
  int32_t in_off[kMaxIn];       // byte offset of the slot's data in an input buffer
  int32_t in_cols[kMaxIn];      // kind 1: columns per 128-row box (128-byte rows: 128 / element size)
  int32_t st_off[kMaxStores];   // byte offset of store o in a warp's staging region
  int32_t st_slot_bytes;        // one warp's staging region (one 32 x 64 group of every store)
  int32_t split3d;              // store 0 is the split-K partial: 3-D map {N, M, S}
  int32_t red0;                 // store 0 adds into its (zeroed) home: TMA reduce-add, no partials
  int32_t epi_off;              // byte offset of the staging region from the aligned base
  int32_t dbg;                  // DLVM_EPI_DBG & 8 (trace builds): per-section cycles of epilogue warp 4
};

struct TcParams {
  CUtensorMap tma_a[kMaxSeg];  // per K segment (sums of products share one accumulator)
  CUtensorMap tma_b[kMaxSeg];
  CUtensorMap tma_st[kMaxStores];  // TMA epilogue stores
  CUtensorMap tma_in[kEpiTmaIn];   // TMA epilogue staged inputs
  EpiTma et;
  GemmParams g;
  int32_t tiles_m, tiles_n;
  int32_t hint_a, hint_b;      // L2 policy per operand: 0 normal, 1 keep (evict_last), 2 stream (evict_first)
  int32_t group_m;             // tile raster: tile-rows per group (N-fastest inside a group is M-fastest here)
  int* sched;                  // dynamic tile scheduling: zeroed work counter (nullptr: static round robin)
  int32_t mc;                  // CTA pairs in 4-CTA clusters sharing B by multicast (tiles_m counts super tiles)
  int32_t super_items;         // pairs working on super tiles (tiles_m counts them): unit u = items 2u, 2u + 1
  int32_t unit0;               // first static work unit of this launch; < 0: claimed (hybrid_claim, sched = state)
  int32_t dyn_base;            // dynamic scheduling: the counter hands out units dyn_base, ... (0: gridDim / cluster;
                               // unused when unit0 < 0: units 0, 1, ...)
#ifdef DLVM_GEMM_TRACE
  unsigned long long* trace;   // [gridDim.x][8] %globaltimer stamps (trace builds, tools/gemm_trace.py)
#endif
};

// Phase stamps of a trace build (-DDLVM_GEMM_TRACE, build variant "trace"):
// 0 entry, 1 after the PDL wait, 2 first TMA issued, 3 first stage landed
// (MMA issuer), 4 last MMA committed, 5 first accumulator ready (epilogue
// warp 4), 6 last epilogue tile done (warp 4), 7 exit.  No-ops otherwise.
#ifdef DLVM_GEMM_TRACE
#define DLVM_GT(P_, slot)                                                           \
  do {                                                                              \
    unsigned long long t_;                                                          \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                         \
    if ((P_).trace) (P_).trace[(size_t)blockIdx.x * kTraceSlots + (slot)] = t_;               \
  } while (0)
// cycles spent in `stmt` added to `acc` (trace builds; plain `stmt` otherwise)
#define DLVM_WAITC(acc, stmt)          \
  do {                                 \
    const long long w0_ = clock64();   \
    stmt;                              \
    acc += clock64() - w0_;            \
  } while (0)
#define DLVM_SECT(var)                                                  \
  do {                                                                  \
    long long c_ = clock64();                                           \
    var += c_ - sect_t0;                                                \
    sect_t0 = c_;                                                       \
  } while (0)
#else
#define DLVM_WAITC(acc, stmt) \
  do {                        \
    stmt;                     \
  } while (0)
#define DLVM_SECT(var) \
  do {                 \
  } while (0)
#define DLVM_GT(P_, slot) \
  do {                    \
  } while (0)
#endif

// CTA-pair (cta_group::2) primitives: a shared::cluster address of the same
// offset in CTA `rank` of the cluster, remote arrive, cluster barrier
__device__ __forceinline__ uint32_t mapa_rank(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// relaxed: it only has to follow this warp's completed TMEM reads (wait::ld +
// fence::before_thread_sync), not its global stores; a release arrive
// compiles to MEMBAR.ALL.GPU and stalls the epilogue on its own stores
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_arrive_release_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_acq_cluster(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAITC_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void st_cluster_u32(uint32_t cluster_addr, int v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_shared_s32(uint32_t addr) {
  int v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void st_shared_s32(uint32_t addr, int v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// both CTAs of a pair load their half; the bytes complete on the leader's
// barrier.  `pol`: L2 eviction policy (createpolicy) for the tile's lines.
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, uint32_t leader_bar, int32_t c0,
                                                 int32_t c1, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
      "[%1, {%3, %4}], [%2], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1), "l"(pol)
      : "memory");
}
// two CTA pairs of a 4-CTA cluster share a B tile: each CTA loads half of
// its pair-half of B and multicasts it to itself and the CTA at the same
// position in the other pair (`mask`); the bytes landing in each
// destination complete on that destination's pair-leader barrier
__device__ __forceinline__ void tma_load_2d_pair_mc(uint32_t dst, const CUtensorMap* map, uint32_t leader_bar,
                                                    int32_t c0, int32_t c1, uint64_t pol, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      ".L2::cache_hint [%0], [%1, {%4, %5}], [%2], %3, %6;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "h"(mask), "r"(c0), "r"(c1), "l"(pol)
      : "memory");
}
// Hybrid work claims: one 64-bit state per GEMM, low word = super tiles
// claimed from the front (the multicast clusters), high word = pair tiles
// claimed from the back (the pair launch), over n_pair pair tiles (unit u =
// pair tiles 2u, 2u + 1).  A claim only succeeds (compare-and-swap) while
// it overlaps no earlier claim, so every pair tile is taken exactly once; a
// single pair tile left between the two sides goes to the pair launch.
// Returns the claimed unit (front) or pair tile (back), or -1 when none is left.
__device__ __forceinline__ int hybrid_claim(unsigned long long* state, bool front, int n_pair) {
  unsigned long long old = atomicAdd(state, 0ull);
  for (;;) {
    const int f = (int)(old & 0xffffffffull), b = (int)(old >> 32);
    if (front ? 2 * f + 2 > n_pair - b : n_pair - b - 1 < 2 * f) return -1;
    const unsigned long long want = front ? old + 1ull : old + (1ull << 32);
    const unsigned long long got = atomicCAS(state, old, want);
    if (got == old) return front ? f : n_pair - 1 - b;
    old = got;
  }
}

// L2 policies: keep (evict_last) the small operand every tile re-reads,
// stream (evict_first) the large one read once, or normal
__device__ __forceinline__ uint64_t l2_policy(int hint) {
  uint64_t p;
  if (hint == 1)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else if (hint == 2)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int32_t c0,
                                            int32_t c1, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4}], "
      "[%2], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "l"(pol)
      : "memory");
}

// TMA epilogue primitives: smem -> global tensor stores in bulk groups
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, uint32_t src, int32_t c0, int32_t c1,
                                             int32_t c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
// smem -> global element-wise f32 add (performed at L2; the K-split work
// items of a tile add their accumulators into one zeroed output)
__device__ __forceinline__ void tma_red_add_2d(const CUtensorMap* map, uint32_t src, int32_t c0, int32_t c1) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}

// Staged epilogue boxes.  Every box row is 128 bytes (SWIZZLE_128B: the
// 16-byte unit u of row r sits at unit u ^ (r & 7)) or, for byte stores of
// a 64-column group, 64 bytes (SWIZZLE_64B: unit u at u ^ ((r >> 1) & 3)),
// so the row-per-lane 16-byte accesses of a warp hit distinct bank groups.
__device__ __forceinline__ uint32_t sw128(uint32_t base, int r, int u) {
  return base + r * 128 + ((u ^ (r & 7)) << 4);
}
__device__ __forceinline__ uint32_t sw64(uint32_t base, int r, int u) {
  return base + r * 64 + ((u ^ ((r >> 1) & 3)) << 4);
}

// 16 values of row r starting at 16-byte unit u0 of a 128-byte-row staged
// input box (stored type st) -> float
__device__ __forceinline__ void box_read16(uint32_t base, int r, int u0, uint8_t st, float* v) {
  if (st == (uint8_t)SType::F32) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint4 x = lds128(sw128(base, r, u0 + c));
      v[4 * c] = __uint_as_float(x.x); v[4 * c + 1] = __uint_as_float(x.y);
      v[4 * c + 2] = __uint_as_float(x.z); v[4 * c + 3] = __uint_as_float(x.w);
    }
  } else if (st == (uint8_t)SType::BF16) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const uint4 x = lds128(sw128(base, r, u0 + c));
      const unsigned w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        v[8 * c + 2 * k] = __uint_as_float(w[k] << 16);
        v[8 * c + 2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
      }
    }
  } else {
    const uint4 x = lds128(sw128(base, r, u0));
    const unsigned w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[4 * k] = (w[k] & 0xffu) ? 1.f : 0.f;
      v[4 * k + 1] = (w[k] & 0xff00u) ? 1.f : 0.f;
      v[4 * k + 2] = (w[k] & 0xff0000u) ? 1.f : 0.f;
      v[4 * k + 3] = (w[k] & 0xff000000u) ? 1.f : 0.f;
    }
  }
}

__device__ __forceinline__ unsigned pack_bf16x2(float lo, float hi) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);  // one cvt.rn.bf16x2.f32, RNE like f2bf
  return *reinterpret_cast<const unsigned*>(&h);
}
// four values known to be exactly 0.0f / 1.0f -> bytes 0 / 1: byte 3 of 1.0f
// is 0x3f, of 0.0f 0x00, so the low bit of that byte is the value
__device__ __forceinline__ unsigned pack01x4(float a, float b, float c, float d) {
  const unsigned ab = __byte_perm(__float_as_uint(a), __float_as_uint(b), 0x0073);
  const unsigned cd = __byte_perm(__float_as_uint(c), __float_as_uint(d), 0x0073);
  return __byte_perm(ab, cd, 0x5410) & 0x01010101u;
}

// Chunk gi (16 columns) of row r of a warp's staged 32-row x 64-column store
// group, stored as type st: f32 in two 32-column boxes of 128-byte rows
// (4 KB apart), bf16 one box of 128-byte rows, bytes one box of 64-byte
// rows.  `is01`: the values are 0.0f / 1.0f (a compare result), which pack
// to bytes without per-element compares.
__device__ __forceinline__ void grp_write16(uint32_t base, int r, int gi, uint8_t st, const float* v, bool is01) {
  if (st == (uint8_t)SType::F32) {
    const uint32_t b = base + (gi >> 1) * 4096;
#pragma unroll
    for (int c = 0; c < 4; ++c)
      sts128(sw128(b, r, (gi & 1) * 4 + c), __float_as_uint(v[4 * c]), __float_as_uint(v[4 * c + 1]),
             __float_as_uint(v[4 * c + 2]), __float_as_uint(v[4 * c + 3]));
  } else if (st == (uint8_t)SType::BF16) {
    unsigned w[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) w[k] = pack_bf16x2(v[2 * k], v[2 * k + 1]);
    sts128(sw128(base, r, 2 * gi), w[0], w[1], w[2], w[3]);
    sts128(sw128(base, r, 2 * gi + 1), w[4], w[5], w[6], w[7]);
  } else {
    unsigned w[4];
    if (is01) {
#pragma unroll
      for (int k = 0; k < 4; ++k) w[k] = pack01x4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        w[k] = (v[4 * k] != 0.f ? 1u : 0u) | (v[4 * k + 1] != 0.f ? 0x100u : 0u) |
               (v[4 * k + 2] != 0.f ? 0x10000u : 0u) | (v[4 * k + 3] != 0.f ? 0x1000000u : 0u);
    }
    sts128(sw64(base, r, gi), w[0], w[1], w[2], w[3]);
  }
}

// UMMA shared-memory matrix descriptor, SWIZZLE_128B (layout type 2), version 1
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// instruction descriptor for kind::f16: bf16 x bf16 -> f32, M=m (128, or 256
// for a CTA pair), N=n
__host__ __device__ constexpr uint32_t umma_idesc(int n, bool a_mn, bool b_mn, int m = BM) {
  return (1u << 4)                       // D format f32
         | (1u << 7)                     // A format bf16
         | (1u << 10)                    // B format bf16
         | ((a_mn ? 1u : 0u) << 15)      // A major (0 = K)
         | ((b_mn ? 1u : 0u) << 16)      // B major (0 = K)
         | ((uint32_t)(n >> 3) << 17)    // N >> 3
         | ((uint32_t)(m >> 4) << 24);   // M >> 4
}

__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
// CTA pair: issued by the leader; one MMA spans both CTAs' smem and TMEM
__device__ __forceinline__ void umma_bf16_pair(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// arrive on the barrier at this offset in every CTA of `mask` (the pair,
// or all four CTAs of a multicast cluster)
__device__ __forceinline__ void umma_commit_pair(uint32_t bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// RV consecutive rows m0.. of column n of an epilogue operand: one storage-
// type branch and one 64-bit offset per batch; rows >= nrow are skipped.
template <int RV>
__device__ __forceinline__ void epi_load(const EwDevIn& in, int64_t m0, int64_t n, int nrow, float* v) {
  const int64_t base = m0 * in.s[0] + n * in.s[1];
  const int64_t rs = in.s[0];
  if (in.st == (uint8_t)SType::F32) {
    const float* p = reinterpret_cast<const float*>(in.ptr) + base;
#pragma unroll
    for (int j = 0; j < RV; ++j) v[j] = j < nrow ? __ldg(p + j * rs) : 0.f;
  } else if (in.st == (uint8_t)SType::BF16) {
    const unsigned short* p = reinterpret_cast<const unsigned short*>(in.ptr) + base;
#pragma unroll
    for (int j = 0; j < RV; ++j) v[j] = j < nrow ? __uint_as_float(((unsigned)__ldg(p + j * rs)) << 16) : 0.f;
  } else {
    const unsigned char* p = reinterpret_cast<const unsigned char*>(in.ptr) + base;
#pragma unroll
    for (int j = 0; j < RV; ++j) v[j] = (j < nrow && __ldg(p + j * rs)) ? 1.f : 0.f;
  }
}

template <int RV>
__device__ __forceinline__ void epi_store(const EwDevOut& o, int64_t m0, int64_t n, int nrow, const float* v) {
  const int64_t base = m0 * o.s[0] + n * o.s[1];
  const int64_t rs = o.s[0];
  if (o.st == (uint8_t)SType::F32) {
    float* p = reinterpret_cast<float*>(o.ptr) + base;
#pragma unroll
    for (int j = 0; j < RV; ++j)
      if (j < nrow) p[j * rs] = v[j];
  } else if (o.st == (uint8_t)SType::F32_ADD) {
    float* p = reinterpret_cast<float*>(o.ptr) + base;
#pragma unroll
    for (int j = 0; j < RV; ++j)
      if (j < nrow) atomicAdd(p + j * rs, v[j]);
  } else if (o.st == (uint8_t)SType::BF16) {
    unsigned short* p = reinterpret_cast<unsigned short*>(o.ptr) + base;
#pragma unroll
    for (int j = 0; j < RV; ++j)
      if (j < nrow) p[j * rs] = f2bf(v[j]);
  } else {
    unsigned char* p = reinterpret_cast<unsigned char*>(o.ptr) + base;
#pragma unroll
    for (int j = 0; j < RV; ++j)
      if (j < nrow) p[j * rs] = v[j] != 0.f ? 1 : 0;
  }
}


template <int CW>
__device__ __forceinline__ void tmem_ldn(uint32_t taddr, float* v) {
  if constexpr (CW == 16) {
    tmem_ld16(taddr, v);
  } else if constexpr (CW == 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
  } else {
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(r[i]);
  }
}

// CW consecutive columns n0.. of row m of an epilogue operand.  `full`: the
// whole segment is in bounds and 16-byte vector accesses are legal.
template <int CW>
__device__ __forceinline__ void epi_row_load(const EwDevIn& in, int64_t m, int64_t n0, int ncol, bool full,
                                             float* v) {
  const int64_t off = m * in.s[0] + n0 * in.s[1];
  if (in.s[1] == 0) {  // constant along the row (column vector / scalar)
    const float x = ncol > 0 ? ld1(in.ptr, off, in.st) : 0.f;
#pragma unroll
    for (int j = 0; j < CW; ++j) v[j] = x;
    return;
  }
  if (full && in.s[1] == 1) {
    if (in.st == (uint8_t)SType::F32) {
      const float4* p = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(in.ptr) + off);
#pragma unroll
      for (int k = 0; k < CW / 4; ++k) {
        const float4 x = __ldg(p + k);
        v[4 * k] = x.x; v[4 * k + 1] = x.y; v[4 * k + 2] = x.z; v[4 * k + 3] = x.w;
      }
      return;
    }
    if (in.st == (uint8_t)SType::BF16) {
      unsigned w[CW / 2];
      const unsigned short* p = reinterpret_cast<const unsigned short*>(in.ptr) + off;
      if constexpr (CW >= 8) {
#pragma unroll
        for (int k = 0; k < CW / 8; ++k) {
          const uint4 x = __ldg(reinterpret_cast<const uint4*>(p + 8 * k));
          w[4 * k] = x.x; w[4 * k + 1] = x.y; w[4 * k + 2] = x.z; w[4 * k + 3] = x.w;
        }
      } else {
        const uint2 x = __ldg(reinterpret_cast<const uint2*>(p));
        w[0] = x.x; w[1] = x.y;
      }
#pragma unroll
      for (int k = 0; k < CW / 2; ++k) {
        v[2 * k] = __uint_as_float(w[k] << 16);
        v[2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
      }
      return;
    }
    unsigned w[CW / 4];
    const unsigned char* p = reinterpret_cast<const unsigned char*>(in.ptr) + off;
    if constexpr (CW == 16) {
      const uint4 x = __ldg(reinterpret_cast<const uint4*>(p));
      w[0] = x.x; w[1] = x.y; w[2] = x.z; w[3] = x.w;
    } else if constexpr (CW == 8) {
      const uint2 x = __ldg(reinterpret_cast<const uint2*>(p));
      w[0] = x.x; w[1] = x.y;
    } else {
      w[0] = __ldg(reinterpret_cast<const unsigned*>(p));
    }
#pragma unroll
    for (int k = 0; k < CW / 4; ++k) {
      v[4 * k] = (w[k] & 0xffu) ? 1.f : 0.f;
      v[4 * k + 1] = (w[k] & 0xff00u) ? 1.f : 0.f;
      v[4 * k + 2] = (w[k] & 0xff0000u) ? 1.f : 0.f;
      v[4 * k + 3] = (w[k] & 0xff000000u) ? 1.f : 0.f;
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < CW; ++j) v[j] = j < ncol ? ld1(in.ptr, off + j * in.s[1], in.st) : 0.f;
}

// optional streamed epilogue stores (st.global.cs, evict-first in L2):
// measured no change of z1's DRAM reads (1.33 -> 1.31 GB) or the c4 step,
// so off (DLVM_EPI_STREAM_STORES=1 at build time enables)
#ifndef DLVM_EPI_STREAM_STORES
#define DLVM_EPI_STREAM_STORES 0
#endif
template <class V>
__device__ __forceinline__ void epi_st(V* p, V x) {
#if DLVM_EPI_STREAM_STORES
  __stcs(p, x);
#else
  *p = x;
#endif
}

template <int CW>
__device__ __forceinline__ void epi_row_store(const EwDevOut& o, int64_t m, int64_t n0, int ncol, bool full,
                                              const float* v) {
  const int64_t off = m * o.s[0] + n0 * o.s[1];
  if (full && o.s[1] == 1) {  // widest aligned stores of the row segment
    if (o.st == (uint8_t)SType::F32) {
      float* p = reinterpret_cast<float*>(o.ptr) + off;
#pragma unroll
      for (int k = 0; k < CW / 4; ++k)
        epi_st(reinterpret_cast<float4*>(p + 4 * k), make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]));
    } else if (o.st == (uint8_t)SType::F32_ADD) {  // accumulate into (possibly peer) memory
      float* p = reinterpret_cast<float*>(o.ptr) + off;
#pragma unroll
      for (int k = 0; k < CW / 4; ++k) red_add_v4(p + 4 * k, v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
    } else if (o.st == (uint8_t)SType::BF16) {
      unsigned w[CW / 2];
#pragma unroll
      for (int k = 0; k < CW / 2; ++k) w[k] = (unsigned)f2bf(v[2 * k]) | ((unsigned)f2bf(v[2 * k + 1]) << 16);
      unsigned short* p = reinterpret_cast<unsigned short*>(o.ptr) + off;
      if constexpr (CW >= 8) {
#pragma unroll
        for (int k = 0; k < CW / 8; ++k)
          epi_st(reinterpret_cast<uint4*>(p + 8 * k), make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]));
      } else {
        epi_st(reinterpret_cast<uint2*>(p), make_uint2(w[0], w[1]));
      }
    } else {
      unsigned w[CW / 4];
#pragma unroll
      for (int k = 0; k < CW / 4; ++k)
        w[k] = (v[4 * k] != 0.f ? 1u : 0u) | (v[4 * k + 1] != 0.f ? 0x100u : 0u) |
               (v[4 * k + 2] != 0.f ? 0x10000u : 0u) | (v[4 * k + 3] != 0.f ? 0x1000000u : 0u);
      unsigned char* p = reinterpret_cast<unsigned char*>(o.ptr) + off;
      if constexpr (CW == 16) {
        epi_st(reinterpret_cast<uint4*>(p), make_uint4(w[0], w[1], w[2], w[3]));
      } else if constexpr (CW == 8) {
        epi_st(reinterpret_cast<uint2*>(p), make_uint2(w[0], w[1]));
      } else {
        epi_st(reinterpret_cast<unsigned*>(p), w[0]);
      }
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < CW; ++j)
    if (j < ncol) st1(o.ptr, off + j * o.s[1], o.st, v[j]);
}


// Raw 16-byte words of a row segment (prefetched one chunk ahead, decoded
// when the chunk is computed).  Sized for f32 (CW/4 uint4).
template <int CW>
struct RawSeg {
  uint4 w[CW / 4];
};

// an operand whose CW-column row segment is one contiguous vector access
__device__ __forceinline__ bool seg_vector(const EwDevIn& in) { return in.s[1] == 1 && in.s[0] != 0; }

#ifndef DLVM_EPI_L1_PREFETCH
#define DLVM_EPI_L1_PREFETCH 0  // measured no gain on the mask + bf16 epilogue (tools/gemm_store_probe.py)
#endif
constexpr bool kEpiL1Prefetch = DLVM_EPI_L1_PREFETCH != 0;

__device__ __forceinline__ void epi_row_prefetch_l1(const EwDevIn& in, int64_t m, int64_t n0) {
  const int es = st_bytes(in.st);
  const char* a = reinterpret_cast<const char*>(in.ptr) + (m * in.s[0] + n0) * es;
  asm volatile("prefetch.global.L1 [%0];" ::"l"(a));
}

template <int CW>
__device__ __forceinline__ void epi_row_fetch(const EwDevIn& in, int64_t m, int64_t n0, RawSeg<CW>& r) {
  const int64_t off = m * in.s[0] + n0;
  if (in.st == (uint8_t)SType::F32) {
    const uint4* p = reinterpret_cast<const uint4*>(reinterpret_cast<const float*>(in.ptr) + off);
#pragma unroll
    for (int k = 0; k < CW / 4; ++k) r.w[k] = __ldg(p + k);
  } else if (in.st == (uint8_t)SType::BF16) {
    const unsigned short* p = reinterpret_cast<const unsigned short*>(in.ptr) + off;
    if constexpr (CW >= 8) {
#pragma unroll
      for (int k = 0; k < CW / 8; ++k) r.w[k] = __ldg(reinterpret_cast<const uint4*>(p + 8 * k));
    } else {
      const uint2 x = __ldg(reinterpret_cast<const uint2*>(p));
      r.w[0] = make_uint4(x.x, x.y, 0, 0);
    }
  } else {
    const unsigned char* p = reinterpret_cast<const unsigned char*>(in.ptr) + off;
    if constexpr (CW == 16) {
      r.w[0] = __ldg(reinterpret_cast<const uint4*>(p));
    } else if constexpr (CW == 8) {
      const uint2 x = __ldg(reinterpret_cast<const uint2*>(p));
      r.w[0] = make_uint4(x.x, x.y, 0, 0);
    } else {
      r.w[0] = make_uint4(__ldg(reinterpret_cast<const unsigned*>(p)), 0, 0, 0);
    }
  }
}

template <int CW>
__device__ __forceinline__ void epi_row_decode(const EwDevIn& in, const RawSeg<CW>& r, float* v) {
  const unsigned* w = reinterpret_cast<const unsigned*>(r.w);
  if (in.st == (uint8_t)SType::F32) {
#pragma unroll
    for (int j = 0; j < CW; ++j) v[j] = __uint_as_float(w[j]);
  } else if (in.st == (uint8_t)SType::BF16) {
#pragma unroll
    for (int k = 0; k < CW / 2; ++k) {
      v[2 * k] = __uint_as_float(w[k] << 16);
      v[2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
    }
  } else {
#pragma unroll
    for (int k = 0; k < CW / 4; ++k) {
      v[4 * k] = (w[k] & 0xffu) ? 1.f : 0.f;
      v[4 * k + 1] = (w[k] & 0xff00u) ? 1.f : 0.f;
      v[4 * k + 2] = (w[k] & 0xff0000u) ? 1.f : 0.f;
      v[4 * k + 3] = (w[k] & 0xff000000u) ? 1.f : 0.f;
    }
  }
}

// Column sums over the 32 lanes of CW values per lane (fixed butterfly
// order): returns the sum for column *col; lanes < CW hold distinct columns.
template <int CW>
__device__ __forceinline__ float col_butterfly(float (&x)[CW], int lane, int* col) {
  int base = 0;
#pragma unroll
  for (int k = 0, w = CW / 2; w >= 1; ++k, w /= 2) {
    const bool up = (lane >> k) & 1;
#pragma unroll
    for (int i = 0; i < w; ++i) {
      const float send = up ? x[i] : x[i + w];
      const float keep = up ? x[i + w] : x[i];
      x[i] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 1 << k));
    }
    if (up) base += w;
  }
#pragma unroll
  for (int s = CW; s < 32; s *= 2) x[0] = __fadd_rn(x[0], __shfl_xor_sync(0xffffffffu, x[0], s));
  *col = base;
  return x[0];
}

// Tile raster: groups of GROUP_M tile-rows, N fastest inside a group, so the
// ~148 tiles in flight share a few A row-panels and all of B through L2
// (a plain M-fastest order re-reads A once per N tile).
constexpr int GROUP_M = 8;  // default group height (TcParams.group_m, DLVM_GEMM_GROUP_M)
__device__ __forceinline__ void tile_coords(int t, int tiles_m, int tiles_n, int* tm, int* tn, int group_m = GROUP_M) {
  const int per_group = group_m * tiles_n;
  const int grp = t / per_group;
  const int first = grp * group_m;
  const int gsz = min(group_m, tiles_m - first);
  const int r = t - grp * per_group;
  *tm = first + r % gsz;
  *tn = r / gsz;
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }


// 32 lanes x 32 columns -> lane l holds the sum over lanes of column l
__device__ __forceinline__ float transpose_reduce32(float* v, int lane) {
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
#pragma unroll
    for (int i = 0; i < w; ++i) {
      const bool upper = (lane & w) != 0;
      float send = upper ? v[i] : v[i + w];
      float keep = upper ? v[i + w] : v[i];
      float recv = __shfl_xor_sync(0xffffffffu, send, w);
      v[i] = __fadd_rn(keep, recv);
    }
  }
  return v[0];
}

constexpr int kEpiReds = 2;  // reductions per GEMM epilogue (smem budget); more -> not fused

template <bool B>
struct bool_c {
  static constexpr bool value = B;
};
template <class T, bool S>
__host__ __device__ constexpr int epi_num_stores() {
  if constexpr (S) return T::Stores::n; else return 0;
}
template <class T, bool S>
__host__ __device__ constexpr int epi_num_reds() {
  if constexpr (S) return T::Reds::n; else return kEpiReds;
}

// Interpreted epilogue programs, instantiated per column-chunk width CW (the
// same width a specialised program of the same size uses, so both sum their
// reductions in the same order and stay bit-identical).
template <int CW>
struct VmEpi {};
struct VmEpiTraits {
  static constexpr int kSlots = kMaxSlots;
  static constexpr int kIn = 0, kLit = 0;
};
template <class P>
struct vm_cw {
  static constexpr int value = 0;
};
template <int CW>
struct vm_cw<VmEpi<CW>> {
  static constexpr int value = CW;
};
__host__ __device__ constexpr int epi_chunk_width(int slots) { return slots <= 6 ? 16 : (slots <= 12 ? 8 : 4); }

// CTAS = 1: one CTA per 128 x BN tile.  CTAS = 2: a CTA pair (cluster of 2
// on one TPC) per 256 x BN tile: each CTA stages its 128 rows of A and half
// of B's columns, the leader issues cta_group::2 MMAs over both CTAs' smem
// into both CTAs' TMEM (per-SM smem traffic per MMA drops by a third), and
// each CTA runs the epilogue of its own 128 rows.
#ifndef DLVM_GEMM_STAGES_PAIR
#define DLVM_GEMM_STAGES_PAIR 6
#endif
template <int CTAS, int BN>
__host__ __device__ constexpr int num_stages() {
  return CTAS == 2 ? DLVM_GEMM_STAGES_PAIR : STAGES;
}
__host__ __device__ constexpr int num_stages_rt(int ctas) { return ctas == 2 ? DLVM_GEMM_STAGES_PAIR : STAGES; }

template <int BN, class PROG, int CTAS = 1>
__global__ void __launch_bounds__(NUM_THREADS, 1) gemm_tc_kernel(const __grid_constant__ TcParams P) {
  constexpr int VMCW = vm_cw<PROG>::value;
  constexpr bool SPEC = VMCW == 0;
  using T = cond_t<SPEC, spec::Traits<cond_t<SPEC, PROG, spec::Prog<0, 0, spec::St<>, spec::Rd<>>>>,
                               VmEpiTraits>;
  constexpr int NS = T::kSlots;
  constexpr int NRS = epi_num_reds<T, SPEC>();
  constexpr int NST = num_stages<CTAS, BN>();
  constexpr int BNC = BN / CTAS;                     // B columns staged per CTA
  constexpr int B_STAGE_BYTES = BNC * BK * 2;
  constexpr uint32_t STAGE_TX = A_STAGE_BYTES + B_STAGE_BYTES;  // per CTA
  constexpr int TMEM_COLS = 2 * BN;  // 256 or 512
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const EpiTma& xt = P.et;
  const int nst = xt.on ? xt.nst : NST;  // pipeline stages (fewer when the TMA epilogue stages)
  const uint32_t sA = base;
  const uint32_t sB = base + nst * A_STAGE_BYTES;
  // barriers: full[<=6] @0, empty[<=6] @48, tfull[2] @96, tempty[2] @112,
  // in_full[2] @128, in_empty[2] @144, tile queue tq_full[4] @160 and
  // tq_empty[4] @192; TMEM address @224; tile ids tileq[4] @240; reductions @256
  const uint32_t sBar = sB + nst * B_STAGE_BYTES;
  const uint32_t full_bar = sBar, empty_bar = sBar + 48, tfull_bar = sBar + 96, tempty_bar = sBar + 112,
                 in_full_bar = sBar + 128, in_empty_bar = sBar + 144, tq_full_bar = sBar + 160,
                 tq_empty_bar = sBar + 192, tileq = sBar + 240;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(gbase + (sBar - base) + 224);
  // reduction scratch sized by the program's reduction count (NRS; the
  // interpreter reserves kEpiReds), so programs without reductions leave
  // that space to the pipeline / TMA epilogue (host: tail_bytes)
  float* colred = reinterpret_cast<float*>(gbase + (sBar - base) + 256);  // [NRS][4][BN]
  float* rowred = colred + NRS * 4 * BN;                                               // [NRS][2][BM]
  float* allred = rowred + NRS * 2 * BM;                                               // [NRS][8]

  const GemmParams& g = P.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) DLVM_GT(P, 0);
  const int base_tiles = P.tiles_m * P.tiles_n;  // tiles of CTAS*BM rows
  const int nsplit = g.ksplit > 1 ? g.ksplit : 1;
  const int n_tiles = base_tiles * nsplit;       // work units (tile, K split)
  const uint32_t rank = CTAS == 2 ? cluster_rank() : 0;
  // multicast clusters (P.mc): 4 CTAs = two pairs; a work item is a super
  // tile of two pair tiles stacked in M (pair `pidx` takes tile row
  // 2 * tm + pidx) that share their B tile.  `prank`: rank in the pair,
  // `pbase`: the pair leader's cluster rank
  const bool mc = CTAS == 2 && P.mc;
  const uint32_t prank = rank & 1u, pbase = rank & 2u;
  const int pidx = (int)(rank >> 1);
  const int cl = mc ? 4 : CTAS;
  // Hybrid launches (gemm_tc.cuh launch_hybrid): a multicast-cluster launch
  // claims super tiles (units u: pair tiles 2u, 2u + 1) from the front of
  // the work list and a pair launch on the SMs the 4-CTA packing leaves
  // over claims single pair tiles (items p: unit p / 2, half p % 2,
  // P.super_items) from the back (hybrid_claim)
  const bool sup = CTAS == 2 && P.super_items;
  const int tile0 = (sup ? 2 : 1) * (P.unit0 + (int)blockIdx.x / cl), tile_step = gridDim.x / cl;
  // item -> the pair's tile row and column; returns the K split
  auto decode = [&](int item, int* tm, int* tn) -> int {
    const int u = sup ? item >> 1 : item;
    tile_coords(u % base_tiles, P.tiles_m, P.tiles_n, tm, tn, P.group_m);
    *tm = sup ? 2 * *tm + (item & 1) : mc ? 2 * *tm + pidx : *tm;
    return u / base_tiles;
  };
  auto split_of = [&](int item) { return (sup ? item >> 1 : item) / base_tiles; };
  const int n_items = sup ? 2 * n_tiles : n_tiles;
  // Dynamic scheduling (P.sched != nullptr): the first tile of every CTA
  // (pair) is its static one; later ones come from an atomic counter
  // (tile_step + counter), fetched by the leader's producer lane one tile
  // ahead and published through the shared tile queue to every other role
  // of the pair (the peer through distributed shared memory), so a grid
  // running beside another kernel takes over tiles as SMs free up.
  const bool dyn = P.sched != nullptr;
  auto tq_publish = [&](int k, int t) {  // leader, warp 0, lane 0
    const int slot = k & 3;
    mbar_wait(tq_empty_bar + 8 * slot, ((k >> 2) & 1) ^ 1);
    st_shared_s32(tileq + 4 * slot, t);
    if constexpr (CTAS == 2) {
      for (int r = 1; r < cl; ++r) {
        st_cluster_u32(mapa_rank(tileq + 4 * slot, r), t);
        mbar_arrive_release_cluster(mapa_rank(tq_full_bar + 8 * slot, r));
      }
    }
    mbar_arrive(tq_full_bar + 8 * slot);
  };
  auto tq_take = [&](int k) -> int {  // one lane of a consumer role
    const int slot = k & 3;
    mbar_wait_acq_cluster(tq_full_bar + 8 * slot, (k >> 2) & 1);
    const int t = ld_shared_s32(tileq + 4 * slot);
    if constexpr (CTAS == 2) {
      if (rank != 0) {
        mbar_arrive_cluster(mapa_rank(tq_empty_bar + 8 * slot, 0));
        return t;
      }
    }
    mbar_arrive(tq_empty_bar + 8 * slot);
    return t;
  };
  // tile of iteration k for a consumer warp (lane 0 takes, the warp shares)
  auto warp_tile = [&](int k) -> int {
    if (!dyn) return tile0 + k * tile_step;
    int t = 0;
    if (lane == 0) t = tq_take(k);
    return __shfl_sync(0xffffffffu, t, 0);
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(full_bar + 8 * s, 1);
      mbar_init(empty_bar + 8 * s, mc ? 2 : 1);  // multicast: both pairs' MMAs release the slot
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(tfull_bar + 8 * s, 1);
      mbar_init(tempty_bar + 8 * s, 8 * CTAS);  // one arrival per epilogue warp of the pair
      mbar_init(in_full_bar + 8 * s, 1);        // the loader's arrive + the staged bytes
      mbar_init(in_empty_bar + 8 * s, 8);       // one arrival per epilogue warp of this CTA
    }
    // tile queue (dynamic scheduling): one publish per slot use; released by
    // every consumer of the pair: the peer's producer, the MMA issuer, the
    // epilogue warps and the input loaders
    // (per pair: the peer's producer, the leader's MMA issuer; a multicast
    // cluster counts both pairs)
    const int n_cons = (cl - 1) + (CTAS == 2 ? cl / 2 : 1) + 8 * cl + (xt.on && xt.n_in_bufs > 0 ? cl : 0);
    for (int s = 0; s < 4; ++s) {
      mbar_init(tq_full_bar + 8 * s, 1);
      mbar_init(tq_empty_bar + 8 * s, n_cons);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int q = 0; q < g.n_seg; ++q) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&P.tma_a[q])) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&P.tma_b[q])) : "memory");
    }
  }
  if (warp == 2) {
    if constexpr (CTAS == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                   "n"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                   "n"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CTAS == 2) cluster_sync_all();  // peer barriers initialised before any remote signal
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  // prologue done: let the next kernel start its own, then wait for the
  // previous kernel's results (PDL, launch.cuh)
  pdl_trigger_gemm();
  pdl_wait();
  if (threadIdx.x == 0) DLVM_GT(P, 1);

  if (warp == 0) {  // ---------------- TMA producer (lane 0) + L2 prefetch of epilogue inputs (all lanes)
    int s = 0;
    uint32_t ph = 0;
    int t_next = tile0;  // leader lane 0 (dynamic): the item published for the next iteration
    // plain dynamic scheduling: counter value c hands out unit dyn_base + c,
    // after every CTA's (pair's) static first unit
    const int dyn_base = P.dyn_base ? P.dyn_base : tile_step;
    // hybrid launches (P.unit0 < 0): every item is claimed, the first one
    // included, so a cluster that becomes resident late finds the work taken
    // instead of holding a static unit for the tail
    auto next_item = [&]() -> int {
      if (P.unit0 < 0) {
        const int c = hybrid_claim(reinterpret_cast<unsigned long long*>(P.sched), !sup, 2 * n_tiles);
        return c < 0 ? n_items : c;
      }
      return dyn_base + atomicAdd(P.sched, 1);
    };
    if (dyn && rank == 0 && lane == 0) {
      if (P.unit0 < 0) t_next = next_item();
      tq_publish(0, t_next);
    }
    for (int pit = 0;; ++pit) {
      int t;
      if (!dyn) {
        t = tile0 + pit * tile_step;
      } else {
        int tl = 0;
        if (lane == 0) {
          if (rank == 0) {
            tl = t_next;
            if (tl < n_items) {  // fetch and publish the next one ahead of need
              t_next = next_item();
              tq_publish(pit + 1, t_next);
            }
          } else {
            tl = tq_take(pit);
          }
        }
        t = __shfl_sync(0xffffffffu, tl, 0);
      }
      if (t >= n_items) break;
      int tm, tn;
      const int split = decode(t, &tm, &tn);
      const int m0 = (tm * CTAS + (int)prank) * BM, n0 = tn * BN;
      for (int i = 0; i < g.n_pf; ++i) {
        const int64_t cols = min((int64_t)BN, g.N - n0);
        const uint32_t bytes = (uint32_t)((cols * g.pf_esize[i] + 15) & ~15);
        for (int r = lane; r < BM && m0 + r < g.M; r += 32) {
          const char* a = reinterpret_cast<const char*>(g.pf_ptr[i]) + (int64_t)(m0 + r) * g.pf_row_bytes[i] +
                          (int64_t)n0 * g.pf_esize[i];
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(bytes) : "memory");
        }
      }
      if (lane == 0) {
        const uint64_t pol_a = l2_policy(P.hint_a), pol_b = l2_policy(P.hint_b);
        for (int q = 0; q < g.n_seg; ++q) {
          const GemmSegParams& G = g.seg[q];
          const CUtensorMap* ma = &P.tma_a[q];
          const CUtensorMap* mb = &P.tma_b[q];
          const int num_kb = (int)((G.K + BK - 1) / BK);
          const int kbs = (num_kb + nsplit - 1) / nsplit;
          const int kb_lo = split * kbs, kb_hi = kb_lo + kbs < num_kb ? kb_lo + kbs : num_kb;
          for (int kb = kb_lo; kb < kb_hi; ++kb) {
            mbar_wait(empty_bar + 8 * s, ph ^ 1);
            if (t == tile0 && q == 0 && kb == kb_lo) DLVM_GT(P, 2);
            const uint32_t fb = full_bar + 8 * s;
            const uint32_t a_dst = sA + s * A_STAGE_BYTES, b_dst = sB + s * B_STAGE_BYTES;
            const int k0 = kb * BK;
            const int nb = n0 + (int)prank * BNC;  // this CTA's half of B
            if constexpr (CTAS == 2) {
              // both halves complete on the leader's barrier, armed with both CTAs' bytes
              const uint32_t lb = mapa_rank(fb, pbase);
#ifdef DLVM_PROBE_SKIP_B
              // measurement probe (wrong results): B loaded on even k-blocks
              // only, 25% fewer operand bytes from L2
              const bool skipb = kb & 1;
              if (prank == 0) mbar_expect_tx(fb, 2 * (skipb ? A_STAGE_BYTES : STAGE_TX));
#else
              constexpr bool skipb = false;
              if (prank == 0) mbar_expect_tx(fb, 2 * STAGE_TX);
#endif
              if (G.a_kmajor) {
                tma_load_2d_pair(a_dst, ma, lb, k0, m0, pol_a);
              } else {
                tma_load_2d_pair(a_dst, ma, lb, m0, k0, pol_a);
                tma_load_2d_pair(a_dst + 8192, ma, lb, m0 + 64, k0, pol_a);
              }
              if (skipb) {
              } else if (mc) {
                // half of this CTA's B half (64 of its BNC = 128 columns), to
                // both pairs
                const uint16_t mask = (uint16_t)((1u << prank) | (1u << (prank + 2)));
                if (G.b_kmajor)
                  tma_load_2d_pair_mc(b_dst + pidx * 8192, mb, lb, k0, nb + 64 * pidx, pol_b, mask);
                else
                  tma_load_2d_pair_mc(b_dst + pidx * 8192, mb, lb, nb + 64 * pidx, k0, pol_b, mask);
              } else if (G.b_kmajor) {
                tma_load_2d_pair(b_dst, mb, lb, k0, nb, pol_b);
              } else {
#pragma unroll
                for (int c = 0; c < BNC / 64; ++c) tma_load_2d_pair(b_dst + c * 8192, mb, lb, nb + 64 * c, k0, pol_b);
              }
            } else {
              mbar_expect_tx(fb, STAGE_TX);
              if (G.a_kmajor) {
                tma_load_2d(a_dst, ma, fb, k0, m0, pol_a);
              } else {
                tma_load_2d(a_dst, ma, fb, m0, k0, pol_a);
                tma_load_2d(a_dst + 8192, ma, fb, m0 + 64, k0, pol_a);
              }
              if (G.b_kmajor) {
                tma_load_2d(b_dst, mb, fb, k0, nb, pol_b);
              } else {
#pragma unroll
                for (int c = 0; c < BNC / 64; ++c) tma_load_2d(b_dst + c * 8192, mb, fb, nb + 64 * c, k0, pol_b);
              }
            }
            if (++s == nst) {
              s = 0;
              ph ^= 1;
            }
          }
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    if (lane == 0 && prank == 0) {  // ---------------- MMA issuer (the pair's leader)
      int s = 0;
      uint32_t ph = 0;
      long long w_acc = 0, w_stage = 0, c_loop = clock64();  // trace builds: wait cycles
      int n_it = 0;
      for (int it = 0;; ++it) {
        const int t = dyn ? tq_take(it) : tile0 + it * tile_step;
        if (t >= n_items) break;
        ++n_it;
        const int split = split_of(t);
        const int as = it & 1;
        const uint32_t aph = (it >> 1) & 1;
        DLVM_WAITC(w_acc, mbar_wait(tempty_bar + 8 * as, aph ^ 1));
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + as * BN;
        uint32_t accum = 0;  // the tile's first MMA overwrites the accumulator
        for (int q = 0; q < g.n_seg; ++q) {
          const GemmSegParams& G = g.seg[q];
          const uint32_t idesc = umma_idesc(BN, !G.a_kmajor, !G.b_kmajor, BM * CTAS);
          const int num_kb = (int)((G.K + BK - 1) / BK);
          const int kbs = (num_kb + nsplit - 1) / nsplit;
          const int kb_lo = split * kbs, kb_hi = kb_lo + kbs < num_kb ? kb_lo + kbs : num_kb;
          for (int kb = kb_lo; kb < kb_hi; ++kb) {
            DLVM_WAITC(w_stage, mbar_wait(full_bar + 8 * s, ph));
            tc_fence_after();
            if (t == tile0 && q == 0 && kb == kb_lo) DLVM_GT(P, 3);
            const uint32_t a0 = sA + s * A_STAGE_BYTES, b0 = sB + s * B_STAGE_BYTES;
            // a K tail (c4 d11: K = 1000 = 15 x 64 + 40): only the 16-wide
            // steps that hold data; the rest of the zero-filled box would
            // add exact zeros
            const int nk16 = kb == num_kb - 1 ? (int)((G.K - (int64_t)kb * BK + 15) / 16) : BK / 16;
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              if (k >= nk16) break;
              const uint64_t ad = G.a_kmajor ? umma_desc(a0 + 32 * k, 16, 1024) : umma_desc(a0 + 2048 * k, 8192, 1024);
              const uint64_t bd = G.b_kmajor ? umma_desc(b0 + 32 * k, 16, 1024) : umma_desc(b0 + 2048 * k, 8192, 1024);
              if constexpr (CTAS == 2)
                umma_bf16_pair(d_tmem, ad, bd, idesc, accum);
              else
                umma_bf16(d_tmem, ad, bd, idesc, accum);
              accum = 1;
            }
            if constexpr (CTAS == 2)
              umma_commit_pair(empty_bar + 8 * s, mc ? 0xF : 3);  // the slot is free in every CTA it feeds
            else
              umma_commit(empty_bar + 8 * s);
            if (++s == nst) {
              s = 0;
              ph ^= 1;
            }
          }
        }
        if constexpr (CTAS == 2)
          umma_commit_pair(tfull_bar + 8 * as, (uint16_t)(3u << pbase));
        else
          umma_commit(tfull_bar + 8 * as);
      }
      DLVM_GT(P, 4);
#ifdef DLVM_GEMM_TRACE
      // slots 16..19: MMA issuer cycles waiting for an empty accumulator
      // (epilogue-bound), for a full operand stage (load-bound), its whole
      // loop, and its tile count
      if (P.trace) {
        P.trace[(size_t)blockIdx.x * kTraceSlots + 16] = (unsigned long long)w_acc;
        P.trace[(size_t)blockIdx.x * kTraceSlots + 17] = (unsigned long long)w_stage;
        P.trace[(size_t)blockIdx.x * kTraceSlots + 18] = (unsigned long long)(clock64() - c_loop);
        P.trace[(size_t)blockIdx.x * kTraceSlots + 19] = (unsigned long long)n_it;
      }
#else
      (void)w_acc;
      (void)w_stage;
      (void)c_loop;
      (void)n_it;
#endif
    }
  } else if (warp == 3) {  // ---------------- epilogue input loader (TMA epilogue)
    if (xt.on && xt.n_in_bufs > 0 && lane == 0) {
      const uint32_t in_base = base + (uint32_t)xt.epi_off;
      const EwParams& E = g.epi;
      for (int it = 0;; ++it) {
        const int t = dyn ? tq_take(it) : tile0 + it * tile_step;
        if (t >= n_items) break;
        int tm, tn;
        decode(t, &tm, &tn);
        const int m0 = (tm * CTAS + (int)prank) * BM, n0 = tn * BN;
        const int b = xt.n_in_bufs == 2 ? (it & 1) : 0;
        const uint32_t ph = xt.n_in_bufs == 2 ? ((it >> 1) & 1) : (it & 1);
        mbar_wait(in_empty_bar + 8 * b, ph ^ 1);
        const uint32_t fb = in_full_bar + 8 * b;
        const uint32_t buf = in_base + (uint32_t)(b * xt.in_buf_bytes);
        const int cols = (int)min((int64_t)BN, g.N - n0);
        uint32_t tx = 0;
        for (int s2 = 1; s2 < kMaxIn; ++s2) {
          if (xt.in_kind[s2] == 1) tx += (uint32_t)(BN / xt.in_cols[s2]) * (uint32_t)(BM * 128);
          else if (xt.in_kind[s2] == 2) tx += (uint32_t)((cols * 4 + 15) & ~15);
        }
        mbar_expect_tx(fb, tx);
        for (int s2 = 1; s2 < kMaxIn; ++s2) {
          if (xt.in_kind[s2] == 1) {
            const CUtensorMap* mp = &P.tma_in[xt.in_map[s2]];
            const int ic = xt.in_cols[s2];
#pragma unroll 1
            for (int c = 0; c < BN / ic; ++c)
              tma_load_2d(buf + xt.in_off[s2] + c * (BM * 128), mp, fb, n0 + ic * c, m0, l2_policy(0));
          } else if (xt.in_kind[s2] == 2) {
            const float* src = reinterpret_cast<const float*>(E.in[s2].ptr) + n0;
            bulk_load(buf + xt.in_off[s2], src, (uint32_t)((cols * 4 + 15) & ~15), fb);
          }
        }
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue
    // 8 warps: warp (q, h) owns TMEM lanes 32q..32q+31 (lane = tile row, the
    // native tcgen05.ld 32x32b layout) and the CW-column chunks ch = h, h+2, ...
    // Each lane loads / stores its row segment of CW consecutive elements
    // with vector accesses; column sums use a shuffle butterfly.
    const int ew = warp - 4;
    const int q = ew & 3, h = ew >> 2;
    const int et = threadIdx.x - 128;  // 0..255
    const EwParams& E = g.epi;
    const EwProgram& Pg = E.prog;
    constexpr int CW = SPEC ? epi_chunk_width(NS) : VMCW;
    constexpr int NSV = SPEC ? NS : (CW == 16 ? 6 : (CW == 8 ? 12 : kMaxSlots));  // interpreter slots
    float v[NSV][CW];
    if constexpr (SPEC) {
#pragma unroll
      for (int i = 0; i < T::kLit; ++i)
#pragma unroll
        for (int j = 0; j < CW; ++j) v[T::kIn + i][j] = Pg.lits[i];
    } else {
      for (int i = 0; i < Pg.n_lits; ++i)
#pragma unroll
        for (int j = 0; j < CW; ++j) v[Pg.n_in + i][j] = Pg.lits[i];
    }
    auto red_slot = [&](int r) -> int {
      if constexpr (SPEC) return T::Reds::at(2 * r); else return Pg.reduce_slot[r];
    };
    auto red_kind = [&](int r) -> int {
      if constexpr (SPEC) return T::Reds::at(2 * r + 1); else return Pg.reduce_kind[r];
    };
    const int nred = SPEC ? NRS : Pg.n_reduces;
    bool has_col = false, has_row = false, has_all = false;
#pragma unroll
    for (int r = 0; r < NRS; ++r)
      if (r < nred) {
        has_col |= red_kind(r) == RED_COL;
        has_row |= red_kind(r) == RED_ROW;
        has_all |= red_kind(r) == RED_ALL;
      }
    const bool vec_ok = E.vec == 4;
    // TMA epilogue (compile-time specialised programs with 16-column chunks)
    constexpr bool TMA_EPI = SPEC && CW == 16;
    const bool tma_on = TMA_EPI && xt.on;
    const bool staged_in = tma_on && xt.n_in_bufs > 0;
    const uint32_t in_base = base + (uint32_t)xt.epi_off;
    const uint32_t st_base = in_base + (uint32_t)(xt.n_in_bufs * xt.in_buf_bytes) +
                             (uint32_t)(ew * xt.st_slot_bytes);  // this warp's staging region
    // per-slot descriptors of the TMA epilogue, read from the parameter
    // space once: input kind / storage type / buffer offset / box width
    // (log2 of its columns), store type and staging offset
    constexpr int NIK = SPEC && T::kIn > 0 ? T::kIn : 1;
    constexpr int NSK = epi_num_stores<T, SPEC>() > 0 ? epi_num_stores<T, SPEC>() : 1;
    int in_kind[NIK], in_off[NIK], in_lgc[NIK];
    uint8_t in_st[NIK], out_st[NSK];
    uint32_t out_off[NSK];
    if constexpr (TMA_EPI) {
#pragma unroll
      for (int s2 = 0; s2 < NIK; ++s2) {
        in_kind[s2] = s2 > 0 && staged_in ? xt.in_kind[s2] : 0;
        in_off[s2] = xt.in_off[s2];
        in_st[s2] = E.in[s2].st;
        in_lgc[s2] = in_st[s2] == (uint8_t)SType::U8 ? 7 : in_st[s2] == (uint8_t)SType::BF16 ? 6 : 5;
      }
#pragma unroll
      for (int s2 = 0; s2 < NSK; ++s2) {
        out_st[s2] = E.out[s2].st;
        out_off[s2] = st_base + (uint32_t)xt.st_off[s2];
      }
    }
#ifdef DLVM_GEMM_TRACE
    long long sect[7] = {0, 0, 0, 0, 0, 0, 0}, sect_t0 = clock64();
#endif
    long long w_full = 0, c_epi = clock64();  // trace builds: accumulator waits, loop cycles
    for (int it = 0;; ++it) {
      const int t = warp_tile(it);
      if (t >= n_items) break;
      int tm, tn;
      const int split = decode(t, &tm, &tn);
      tm = tm * CTAS + (int)prank;  // this CTA's 128-row block (partials layout)
      // split K: this work item's raw accumulator goes to its split's slice
      EwDevOut out0 = E.out[0];
      out0.ptr = static_cast<char*>(out0.ptr) + (int64_t)split * g.split_bytes;
      const bool block_live = (int64_t)tm * BM < g.M;
      const bool tile_full = (int64_t)tm * BM + BM <= g.M && (int64_t)tn * BN + BN <= g.N;
      const int64_t m = (int64_t)tm * BM + 32 * q + lane;
      const bool mval = m < g.M;
      // this row's segments take the vector path only if every row-contiguous
      // operand's row starts on its vector width (min(16, CW * element bytes))
      bool row_vec = vec_ok;
      if (row_vec) {
        auto al = [&](const void* p, int64_t s0, uint8_t st) {
          const int es = st_bytes(st);
          const int w = CW * es < 16 ? CW * es : 16;
          return ((reinterpret_cast<uintptr_t>(p) + (uintptr_t)(m * s0 * es)) & (uintptr_t)(w - 1)) == 0;
        };
        int nin, nst;
        if constexpr (SPEC) {
          nin = T::kIn;
          nst = T::Stores::n;
        } else {
          nin = Pg.n_in;
          nst = Pg.n_stores;
        }
        for (int s2 = 1; s2 < nin; ++s2)
          if (E.in[s2].s[1] == 1) row_vec &= al(E.in[s2].ptr, E.in[s2].s[0], E.in[s2].st);
        for (int s2 = 0; s2 < nst; ++s2) row_vec &= al(s2 == 0 ? out0.ptr : E.out[s2].ptr, E.out[s2].s[0], E.out[s2].st);
      }
      const int as = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      DLVM_WAITC(w_full, mbar_wait(tfull_bar + 8 * as, aph));
      tc_fence_after();
      if (it == 0 && ew == 0 && lane == 0) DLVM_GT(P, 5);
      const int ib = xt.n_in_bufs == 2 ? (it & 1) : 0;
      const uint32_t in_buf = in_base + (uint32_t)(ib * xt.in_buf_bytes);
      if (staged_in) mbar_wait(in_full_bar + 8 * ib, xt.n_in_bufs == 2 ? ((it >> 1) & 1) : (it & 1));
      float rowacc[NRS > 0 ? NRS : 1], allacc[NRS > 0 ? NRS : 1];
#pragma unroll
      for (int r = 0; r < (NRS > 0 ? NRS : 1); ++r) rowacc[r] = allacc[r] = 0.f;
      constexpr int NPF = SPEC && T::kIn > 1 ? T::kIn - 1 : 1;
      RawSeg<CW> pf[NPF];  // next chunk's row segments of the vector operands
      auto seg_full = [&](int ch) {
        const int64_t n0 = (int64_t)tn * BN + ch * CW;
        return mval && row_vec && n0 + CW <= g.N;
      };
      // warp h takes every other 64-column block (its GCH chunks of CW
      // columns in order), so which warp sums which columns -- and with
      // element-by-element row/full sums the whole summation order -- does
      // not depend on the chunk width: a kept loss computed by the gradient's
      // epilogue equals the primal's bit for bit (reading A20) even when the
      // two programs get different chunk widths
      constexpr int GCH = 64 / CW;                 // chunks per 64-column group
      constexpr int NIT = BN / CW / 2;             // chunks per warp per tile
      auto chunk_of = [&](int i) { return (h + 2 * (i / GCH)) * GCH + i % GCH; };
      auto staged = [&](int s2) {
        if constexpr (TMA_EPI) return in_kind[s2] != 0; else return false;
      };
      // fast TMA tile: every input is staged or constant along the row
      // (column vector / scalar: loaded once per tile) -- no per-chunk
      // global loads, prefetch registers or bounds checks
      bool fast = false;
      float rowc[SPEC && T::kIn > 1 ? T::kIn : 1];
      if constexpr (TMA_EPI) {
        fast = tma_on;
#pragma unroll
        for (int s2 = 1; s2 < T::kIn; ++s2) {
          const bool st_ = staged(s2);
          fast = fast && (st_ || E.in[s2].s[1] == 0);
          rowc[s2] = (!st_ && E.in[s2].s[1] == 0 && mval) ? ld1(E.in[s2].ptr, m * E.in[s2].s[0], E.in[s2].st) : 0.f;
        }
      }
      if constexpr (SPEC) {
        if (!fast && seg_full(chunk_of(0)))
#pragma unroll
          for (int s2 = 1; s2 < T::kIn; ++s2)
            if (seg_vector(E.in[s2]) && !staged(s2))
              epi_row_fetch<CW>(E.in[s2], m, (int64_t)tn * BN + chunk_of(0) * CW, pf[s2 - 1]);
      }
      // the chunk loop, compiled twice: the fast TMA tile (FAST) and the
      // general one, so the hot loop of a fast tile is a compact body
      // (instruction-cache footprint) without the direct-path variants
      auto chunk_loop = [&](auto fast_c) {
      constexpr bool FAST = decltype(fast_c)::value;
      for (int it = 0; it < NIT; ++it) {
        const int ch = chunk_of(it);
        const int64_t n0 = (int64_t)tn * BN + ch * CW;
        const int ncol = tile_full ? CW : (int)min((int64_t)CW, max((int64_t)0, g.N - n0));  // valid columns
        const bool full = mval && ncol == CW && row_vec;
        RawSeg<CW> cur[NPF];
        if constexpr (SPEC && !FAST) {
#pragma unroll
          for (int s2 = 0; s2 < NPF; ++s2) cur[s2] = pf[s2];
          const int nx = it + 1 < NIT ? chunk_of(it + 1) : 0;
          if (it + 1 < NIT && seg_full(nx))
#pragma unroll
            for (int s2 = 1; s2 < T::kIn; ++s2)
              if (seg_vector(E.in[s2]) && !staged(s2))
                epi_row_fetch<CW>(E.in[s2], m, (int64_t)tn * BN + nx * CW, pf[s2 - 1]);
          // row segments three chunks further on into L1 (no registers)
          const int nx3 = it + 3 < NIT ? chunk_of(it + 3) : 0;
          if (kEpiL1Prefetch && it + 3 < NIT && seg_full(nx3))
#pragma unroll
            for (int s2 = 1; s2 < T::kIn; ++s2)
              if (seg_vector(E.in[s2])) epi_row_prefetch_l1(E.in[s2], m, (int64_t)tn * BN + nx3 * CW);
        }
        DLVM_SECT(sect[0]);  // prefetch / loop overhead
        tmem_ldn<CW>(tmem_base + ((uint32_t)(32 * q) << 16) + as * BN + ch * CW, v[0]);
        DLVM_SECT(sect[1]);  // TMEM load
        if constexpr (SPEC) {
#pragma unroll
          for (int s2 = 1; s2 < T::kIn; ++s2) {
            if constexpr (TMA_EPI) {
              if (FAST && !staged(s2)) {
#pragma unroll
                for (int j = 0; j < CW; ++j) v[s2][j] = rowc[s2];
                continue;
              }
              if (staged(s2)) {
                if (in_kind[s2] == 1) {  // [M, N]: row 32q+lane, columns ch*16.. of the tile
                  const int col = ch * CW, lg = in_lgc[s2];  // boxes of 2^lg columns (128-byte rows)
                  box_read16(in_buf + in_off[s2] + (col >> lg) * (BM * 128), 32 * q + lane,
                             ((col & ((1 << lg) - 1)) << (7 - lg)) >> 4, in_st[s2], reinterpret_cast<float*>(v[s2]));
                } else {  // [1, N] row vector: the chunk's 16 values, same for every lane
                  const uint32_t a0 = in_buf + in_off[s2] + ch * 64;
#pragma unroll
                  for (int c = 0; c < 4; ++c) {
                    const uint4 x = lds128(a0 + 16 * c);
                    v[s2][4 * c] = __uint_as_float(x.x); v[s2][4 * c + 1] = __uint_as_float(x.y);
                    v[s2][4 * c + 2] = __uint_as_float(x.z); v[s2][4 * c + 3] = __uint_as_float(x.w);
                  }
                }
                continue;
              }
            }
            if constexpr (!FAST) {
              if (full && seg_vector(E.in[s2]))
                epi_row_decode<CW>(E.in[s2], cur[s2 - 1], v[s2]);
              else
                epi_row_load<CW>(E.in[s2], m, n0, mval ? ncol : 0, full, v[s2]);
            }
          }
          DLVM_SECT(sect[2]);  // inputs
          T::template exec<CW>(v);
          DLVM_SECT(sect[3]);  // program
          if (FAST || tma_on) {
            if constexpr (TMA_EPI) {
              // stage this chunk into the warp's 32 x 64 group boxes; the
              // group's first chunk waits until the TMA has read the
              // previous group, its last one hands the boxes to TMA
              const int gi = it % GCH;
              if (gi == 0) {
                DLVM_SECT(sect[4]);
                if (lane == 0) bulk_wait_read<0>();
                __syncwarp();
                DLVM_SECT(sect[6]);  // waiting for the staging to be read
              }
#pragma unroll
              for (int s2 = 0; s2 < T::Stores::n; ++s2)
                grp_write16(out_off[s2], lane, gi, out_st[s2], reinterpret_cast<const float*>(v[T::Stores::at(s2)]),
                            T::is01(T::Stores::at(s2)));
              if (gi == GCH - 1) {
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                  const int32_t r0 = tm * BM + 32 * q;
                  const int32_t c0 = (int32_t)((int64_t)tn * BN + (ch - gi) * CW);  // the group's first column
#pragma unroll
                  for (int s2 = 0; s2 < T::Stores::n; ++s2) {
                    const uint32_t b = out_off[s2];
                    const bool f32 = out_st[s2] == (uint8_t)SType::F32;
                    if (s2 == 0 && xt.split3d) {
                      tma_store_3d(&P.tma_st[0], b, c0, r0, split);
                      tma_store_3d(&P.tma_st[0], b + 4096, c0 + 32, r0, split);
                    } else if (s2 == 0 && xt.red0) {
                      tma_red_add_2d(&P.tma_st[0], b, c0, r0);
                      tma_red_add_2d(&P.tma_st[0], b + 4096, c0 + 32, r0);
                    } else {
                      tma_store_2d(&P.tma_st[s2], b, c0, r0);
                      if (f32) tma_store_2d(&P.tma_st[s2], b + 4096, c0 + 32, r0);
                    }
                  }
                  bulk_commit();
                }
              }
            }
          } else if constexpr (!FAST) {
#pragma unroll
            for (int s2 = 0; s2 < T::Stores::n; ++s2)
              epi_row_store<CW>(s2 == 0 ? out0 : E.out[s2], m, n0, mval ? ncol : 0, full, v[T::Stores::at(s2)]);
          }
        } else {
          for (int s2 = 1; s2 < Pg.n_in; ++s2) epi_row_load<CW>(E.in[s2], m, n0, mval ? ncol : 0, full, v[s2]);
          vm_exec<CW>(Pg, v);
          for (int s2 = 0; s2 < Pg.n_stores; ++s2)
            epi_row_store<CW>(s2 == 0 ? out0 : E.out[s2], m, n0, mval ? ncol : 0, full, v[Pg.store_slot[s2]]);
        }
        DLVM_SECT(sect[4]);  // stores
#pragma unroll
        for (int r = 0; r < NRS; ++r) {
          if (r >= nred) break;
          const int kind = red_kind(r);
          float x[CW];
          if (tile_full) {  // interior tile: every row and column is in range
#pragma unroll
            for (int j = 0; j < CW; ++j) x[j] = v[red_slot(r)][j];
          } else {
#pragma unroll
            for (int j = 0; j < CW; ++j) x[j] = (mval && j < ncol) ? v[red_slot(r)][j] : 0.f;
          }
          if (kind == RED_COL) {
            int col;
            const float cs = col_butterfly<CW>(x, lane, &col);
            if (lane < CW) colred[(r * 4 + q) * BN + ch * CW + col] = cs;
          } else if (kind == RED_ROW) {  // element by element (chunk-width independent)
#pragma unroll
            for (int j = 0; j < CW; ++j) rowacc[r] = __fadd_rn(rowacc[r], x[j]);
          } else {
#pragma unroll
            for (int j = 0; j < CW; ++j) allacc[r] = __fadd_rn(allacc[r], x[j]);
          }
        }
        DLVM_SECT(sect[5]);  // reductions
      }
      };
      if (fast) chunk_loop(bool_c<true>{}); else chunk_loop(bool_c<false>{});
      // this warp is done with the tile's staged inputs
      if (staged_in) {
        __syncwarp();
        if (lane == 0) mbar_arrive(in_empty_bar + 8 * ib);
      }
      // accumulator buffer free for the next tile's MMAs (one arrival per warp,
      // on the leader's barrier for a pair)
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CTAS == 2)
          mbar_arrive_cluster(mapa_rank(tempty_bar + 8 * as, pbase));
        else
          mbar_arrive(tempty_bar + 8 * as);
      }
      if (has_row || has_all) {
#pragma unroll
        for (int r = 0; r < NRS; ++r) {
          if (r >= nred) break;
          if (red_kind(r) == RED_ROW) rowred[(r * 2 + h) * BM + 32 * q + lane] = rowacc[r];
          if (red_kind(r) == RED_ALL) {
            const float s3 = warp_sum(allacc[r]);
            if (lane == 0) allred[r * 8 + ew] = s3;
          }
        }
      }
      if ((has_col || has_row || has_all) && block_live) {
        epi_bar();
#pragma unroll
        for (int r = 0; r < NRS; ++r) {
          if (r >= nred) break;
          const int kind = red_kind(r);
          if (kind == RED_COL) {
            for (int c = et; c < BN; c += 256) {
              const int64_t n = (int64_t)tn * BN + c;
              if (n >= g.N) continue;
              float s3 = 0.f;
              for (int w2 = 0; w2 < 4; ++w2) s3 = __fadd_rn(s3, colred[(r * 4 + w2) * BN + c]);
              E.red[r][(int64_t)tm * g.N + n] = s3;
            }
          } else if (kind == RED_ROW) {
            if (et < BM) {
              const int64_t mm = (int64_t)tm * BM + et;
              if (mm < g.M)
                E.red[r][mm * E.gx + tn] = __fadd_rn(rowred[(r * 2) * BM + et], rowred[(r * 2 + 1) * BM + et]);
            }
          } else if (et == 0) {
            float s3 = 0.f;
            for (int w2 = 0; w2 < 8; ++w2) s3 = __fadd_rn(s3, allred[r * 8 + w2]);
            E.red[r][(int64_t)tm * E.gx + tn] = s3;
          }
        }
        epi_bar();
      }
    }
    if (tma_on && lane == 0) bulk_wait_all();  // this warp's TMA stores are complete
    if (ew == 0 && lane == 0) DLVM_GT(P, 6);
#ifdef DLVM_GEMM_TRACE
    // slots 20, 21: epilogue warp 4's cycles waiting for a full accumulator
    // (MMA-bound) and its whole tile loop
    if (ew == 0 && lane == 0 && P.trace) {
      P.trace[(size_t)blockIdx.x * kTraceSlots + 20] = (unsigned long long)w_full;
      P.trace[(size_t)blockIdx.x * kTraceSlots + 21] = (unsigned long long)(clock64() - c_epi);
    }
#else
    (void)w_full;
    (void)c_epi;
#endif
#ifdef DLVM_GEMM_TRACE
    // epilogue section cycles of warp 4 (DLVM_EPI_DBG & 8): slots 8..14 =
    // loop overhead, TMEM loads, inputs, program, stores, reductions, staging waits
    if ((xt.dbg & 8) && ew == 0 && lane == 0 && P.trace) {
      long long c_ = clock64();
      (void)c_;
      for (int k = 0; k < 7; ++k) P.trace[(size_t)blockIdx.x * kTraceSlots + 8 + k] = (unsigned long long)sect[k];
    }
#endif
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CTAS == 2) cluster_sync_all();  // the pair's MMAs and epilogues are done
  if (warp == 2) {
    tc_fence_after();
    if constexpr (CTAS == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(TMEM_COLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(TMEM_COLS));
  }
  if (threadIdx.x == 0) DLVM_GT(P, 7);
}

}  // namespace kern
}  // namespace dlvm
