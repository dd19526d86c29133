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
#include <cstdio>
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

constexpr int kMaxDynSmem = 227 * 1024;
__host__ __device__ constexpr int stage_bytes(int bn, int ctas) { return A_STAGE_BYTES + (bn / ctas) * BK * 2; }
// bytes after the stages: barriers (256) + the epilogue reduction scratch
__host__ __device__ constexpr int tail_bytes(int bn, int nred = kEpiReds) {
  return 256 + (nred * 4 * bn + nred * 2 * BM + nred * 8) * 4;
}
constexpr int round_up(int x, int a) { return (x + a - 1) / a * a; }

template <int BN, int CTAS = 1>
constexpr int smem_bytes() {
  return 1024 + num_stages<CTAS, BN>() * stage_bytes(BN, CTAS) + tail_bytes(BN);
}
static_assert(smem_bytes<256, 2>() <= kMaxDynSmem, "CTA-pair stages exceed shared memory");

// dynamic shared memory of a launch: the default pipeline, or with the TMA
// epilogue its stage count plus the staging region
int launch_smem(const TcParams& tp, int bn, int ctas) {
  if (!tp.et.on) return 1024 + num_stages_rt(ctas) * stage_bytes(bn, ctas) + tail_bytes(bn);
  return 1024 + tp.et.epi_off + tp.et.n_in_bufs * tp.et.in_buf_bytes + 8 * tp.et.st_slot_bytes;
}

int es_of(uint8_t st) { return st_bytes(st); }

// 2-D (or, with `splits`, 3-D {cols, rows, splits}) tensor map of an
// epilogue operand with box {box_cols, box_rows}; box rows of 128 bytes use
// SWIZZLE_128B, of 64 bytes SWIZZLE_64B (the layouts sw128 / sw64 read and
// write)
bool encode_epi(CUtensorMap* map, const void* ptr, uint8_t st, int64_t cols, int64_t rows, int64_t pitch_bytes,
                int box_cols, int box_rows, int64_t splits = 0, int64_t split_bytes = 0) {
  auto fn = get_encode();
  if (!fn) return false;
  const int es = es_of(st);
  const int row_bytes = box_cols * es;
  if (reinterpret_cast<uintptr_t>(ptr) % 16 || pitch_bytes % 16 || pitch_bytes <= 0 || rows < 1 || cols < 1)
    return false;
  if (splits > 1 && split_bytes % 16) return false;
  if (row_bytes != 128 && row_bytes != 64) return false;
  const CUtensorMapDataType dt = es == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                 : es == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_UINT8;
  const CUtensorMapSwizzle sw = row_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)(splits > 1 ? splits : 1)};
  cuuint64_t strides[2] = {(cuuint64_t)pitch_bytes, (cuuint64_t)split_bytes};
  cuuint32_t box[3] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows, 1u};
  cuuint32_t esd[3] = {1u, 1u, 1u};
  const cuuint32_t rank = splits > 1 ? 3 : 2;
  CUresult r = fn(map, dt, rank, const_cast<void*>(ptr), dims, strides, box, esd, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

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

// 4-CTA clusters that can be resident at once with one CTA per SM (GPCs
// whose SM count is not a multiple of 4 leave SMs over); 0 if unknown
__global__ void mc_probe_kernel() {}
int max_clusters4() {
  static const int n = [] {
    if (cudaFuncSetAttribute(mc_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem) !=
        cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(4 * 64, 1, 1);
    cfg.blockDim = dim3(NUM_THREADS, 1, 1);
    cfg.dynamicSmemBytes = kMaxDynSmem;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = 4;
    a[0].val.clusterDim.y = 1;
    a[0].val.clusterDim.z = 1;
    cfg.attrs = a;
    cfg.numAttrs = 1;
    int c = 0;
    if (cudaOccupancyMaxActiveClusters(&c, (const void*)mc_probe_kernel, &cfg) != cudaSuccess) {
      cudaGetLastError();
      c = 0;
    }
    return c;
  }();
  return n;
}

// TMA epilogue set-up (see EpiTma): stores, staged inputs, stage count.
// `spec_prog`: the kernel runs a compile-time program (ahead-of-time or
// NVRTC), whose chunk width follows from its slot count.
void setup_tma_epilogue_impl(const GemmParams& p, TcParams* tp, int ctas, bool spec_prog);
// DLVM_EPI_VERBOSE=1: one stderr line per launch set-up (TMA epilogue on/off, stages, buffers)
void setup_tma_epilogue(const GemmParams& p, TcParams* tp, int ctas, bool spec_prog) {
  setup_tma_epilogue_impl(p, tp, ctas, spec_prog);
  static const bool verbose = [] {
    const char* e = std::getenv("DLVM_EPI_VERBOSE");
    return e && e[0] == '1';
  }();
  if (verbose) {
    const EpiTma& et = tp->et;
    fprintf(stderr, "dlvm gemm M=%lld N=%lld bn=%d ctas=%d mc=%d sup=%d spec=%d slots=%d stores=%d: tma_epi=%d "
            "nst=%d in_bufs=%d in_buf=%d st_region=%d clusters4=%d\n", (long long)p.M, (long long)p.N, p.bn, ctas,
            tp->mc, tp->super_items, (int)spec_prog,
            p.epi.prog.n_in + p.epi.prog.n_lits + p.epi.prog.n_ins, p.epi.prog.n_stores, et.on, et.nst,
            et.n_in_bufs, et.in_buf_bytes, et.st_slot_bytes, max_clusters4());
  }
}

void setup_tma_epilogue_impl(const GemmParams& p, TcParams* tp, int ctas, bool spec_prog) {
  EpiTma& et = tp->et;
  et.on = 0;
  static const bool enabled = [] {
    const char* e = std::getenv("DLVM_GEMM_TMA_EPI");
    return !(e && e[0] == '0');
  }();
  const EwParams& E = p.epi;
  const EwProgram& Pg = E.prog;
  if (!enabled || !spec_prog || epi_chunk_width(Pg.n_in + Pg.n_lits + Pg.n_ins) != 16 || Pg.n_stores < 1) return;
  const int BN = p.bn;
  // stores: every one TMA-legal, else the direct path for all.  A warp's
  // staging region holds one 32-row x 64-column group of every store: f32 as
  // two 32-column boxes (4 KB each), bf16 one box of 128-byte rows (4 KB),
  // bytes one box of 64-byte rows (2 KB)
  int off = 0;
  for (int o = 0; o < Pg.n_stores; ++o) {
    const EwDevOut& r = E.out[o];
    const int es = es_of(r.st);
    if (r.s[1] != 1 || r.st == (uint8_t)SType::F32_ADD) return;  // accumulated outputs: direct red path
    const bool split = o == 0 && p.ksplit > 1 && !p.split_red;
    if (!encode_epi(&tp->tma_st[o], r.ptr, r.st, p.N, p.M, r.s[0] * es, es == 4 ? 32 : 64, 32,
                    split ? p.ksplit : 0, split ? p.split_bytes : 0))
      return;
    off = round_up(off, es == 1 ? 512 : 1024);
    et.st_off[o] = off;
    off += es == 4 ? 8192 : es == 2 ? 4096 : 2048;
  }
  et.split3d = p.ksplit > 1 && !p.split_red;
  et.red0 = p.split_red && p.ksplit > 1;
  et.st_slot_bytes = round_up(off, 1024);
  // staged inputs: [M, N] rows (kind 1: boxes of 128 rows x 128 bytes) and
  // [1, N] f32 row vectors (kind 2)
  int nmap = 0, in_bytes = 0, in1_bytes = 0;
  int8_t kind[kMaxIn] = {0};
  for (int s2 = 1; s2 < Pg.n_in; ++s2) {
    const EwDevIn& in = E.in[s2];
    if (in.nchunks != 1 || in.chunk_op) continue;
    const int es = es_of(in.st);
    if (in.s[1] == 1 && in.s[0] != 0 && nmap < kEpiTmaIn && BN % (128 / es) == 0 &&
        encode_epi(&tp->tma_in[nmap], in.ptr, in.st, p.N, p.M, in.s[0] * es, 128 / es, BM)) {
      kind[s2] = 1;
      et.in_map[s2] = (int8_t)nmap++;
      et.in_cols[s2] = 128 / es;
      in_bytes = round_up(in_bytes, 1024);
      et.in_off[s2] = in_bytes;
      in_bytes += BN * es * BM;
      in1_bytes += BN * es * BM;
    } else if (in.s[0] == 0 && in.s[1] == 1 && in.st == (uint8_t)SType::F32 && p.N % 4 == 0 &&
               reinterpret_cast<uintptr_t>(in.ptr) % 16 == 0) {
      kind[s2] = 2;
      in_bytes = round_up(in_bytes, 16);
      et.in_off[s2] = in_bytes;
      in_bytes += BN * 4;
    }
  }
  const int stage = stage_bytes(BN, ctas), tail = tail_bytes(BN, Pg.n_reduces);  // compile-time programs: NRS
  const int nst_max = num_stages_rt(ctas), nst_min = ctas == 2 ? 4 : 3;
  auto total = [&](int nst, int nbufs, int ibytes) {
    return 1024 + round_up(nst * stage + tail, 1024) + nbufs * round_up(ibytes, 1024) + 8 * et.st_slot_bytes;
  };
  // prefer more pipeline stages, then two input buffers; drop the [M, N]
  // inputs back to direct loads if even one buffer does not fit
  for (int pass = 0; pass < 2; ++pass) {
    const int ib = pass == 0 ? in_bytes : in_bytes - in1_bytes;  // pass 1: row vectors only
    if (pass == 1) {
      int o2 = 0;
      for (int s2 = 1; s2 < kMaxIn; ++s2) {
        if (kind[s2] == 1) kind[s2] = 0;
        if (kind[s2] == 2) {
          et.in_off[s2] = o2;
          o2 += BN * 4;
        }
      }
    }
    for (int nst = nst_max; nst >= nst_min; --nst)
      for (int nb = ib > 0 ? 2 : 0; nb >= (ib > 0 ? 1 : 0); --nb)
        if (total(nst, nb, ib) <= kMaxDynSmem) {
          for (int s2 = 0; s2 < kMaxIn; ++s2) et.in_kind[s2] = kind[s2];
          et.nst = nst;
          et.n_in_bufs = nb;
          et.in_buf_bytes = round_up(ib, 1024);
          et.epi_off = round_up(nst * stage + tail, 1024);
          et.on = 1;
          static const int dbg = [] {
            const char* e = std::getenv("DLVM_EPI_DBG");
            return e ? std::atoi(e) : 0;
          }();
          et.dbg = dbg;
          return;
        }
  }
}

// Multicast clusters (DLVM_GEMM_MC: 0 off (default), 1 hybrid, 2 alone):
// two CTA pairs in a 4-CTA cluster share their B tile through TMA
// multicast, so each pair reads 24 instead of 32 KB of operands from L2 per
// k-block.  The 4-CTA packing leaves SMs over (B200: 33 clusters = 132
// SMs); mode 1 runs a multicast launch beside a pair launch on the rest
// (launch_hybrid), both claiming tiles through one zeroed 8-byte state
// (GemmParams::hyb).  Both need an even number of pair tile rows.
// Measured (c4 GEMMs, one B200): multicast alone on 132 SMs takes the same
// time as plain pairs on 148, and the hybrid is no faster than plain pairs
// (z-type 1.646 vs 1.643 ms; the c4 step slower): the mainloop is bound by
// the bytes each SM receives (multicast delivers the same bytes to both
// pairs), not by L2 reads, so only a larger tile per CTA lowers it.
int mc_mode() {
  static const int mode = [] {
    const char* e = std::getenv("DLVM_GEMM_MC");
    return e ? std::atoi(e) : 0;  // off: measured no gain (below)
  }();
  return mode;
}
bool mc_shape_ok(const GemmParams& p, int ctas) {
  const int64_t pair_rows = (p.M + 2 * BM - 1) / (2 * BM);
  return ctas == 2 && !p.sched && pair_rows % 2 == 0 && max_clusters4() > 0;
}
// a multicast launch alone: forced, or when the packing leaves at most 8 SMs
bool use_mc(const GemmParams& p, int ctas) {
  const int mode = mc_mode();
  return mode != 0 && mc_shape_ok(p, ctas) && (mode == 2 || 4 * max_clusters4() >= num_sms() - 8);
}

// launch roles: plain (CTA or pair tiles), multicast clusters, pairs on
// super tiles (the hybrid's second launch)
enum { kRolePlain = 0, kRoleMc = 1, kRoleSuper = 2 };

// CTAs per cluster and grid size of a launch of `tp`
void grid_of(const TcParams& tp, int ctas, int* cluster, int* grid) {
  const int items = tp.tiles_m * tp.tiles_n * std::max(tp.g.ksplit, 1);  // work units (tile x K split)
  *cluster = tp.mc ? 4 : ctas;
  const int slots = tp.mc ? max_clusters4() : num_sms() / ctas;  // persistent: one cluster per slot
  *grid = *cluster * std::min(items, slots);
}

bool make_params(const GemmParams& p, TcParams* tp, int ctas = 1, bool spec_prog = false, int role = -1) {
  memset(tp, 0, sizeof(*tp));
  tp->g = p;
  tp->sched = p.sched;
  if (role < 0) role = use_mc(p, ctas) ? kRoleMc : kRolePlain;
  tp->mc = role == kRoleMc;
  tp->super_items = role == kRoleSuper;
#ifdef DLVM_GEMM_TRACE
  // launch k of the traced run writes slice k % slots of [slots][148][kTraceSlots]
  tp->trace = g_gemm_trace_ptr ? g_gemm_trace_ptr + (size_t)(g_gemm_trace_next++ % g_gemm_trace_slots) * 148 * kTraceSlots
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
    if (G.b_kmajor)  // B stored [N][K]: map {K, N}, box {64, BN / ctas} (a CTA's share; half of it multicast)
      ok = encode(&tp->tma_b[q], G.b, G.K, p.N, G.b_s1, BN / ctas / (tp->mc ? 2 : 1));
    else  // B stored [K][N]: map {N, K}, box {64, 64}
      ok = encode(&tp->tma_b[q], G.b, p.N, G.K, G.b_s0, 64);
    if (!ok) return false;
  }
  static const int group_env = [] {
    const char* e = std::getenv("DLVM_GEMM_GROUP_M");
    return e ? std::atoi(e) : 0;
  }();
  tp->tiles_m = (int)((p.M + BM * ctas - 1) / (BM * ctas));
  if (role != kRolePlain) tp->tiles_m = (tp->tiles_m + 1) / 2;  // super tiles of two pair tiles

  tp->tiles_n = (int)((p.N + BN - 1) / BN);
  // tile raster: tall GEMMs (many more tile rows than columns: the forward
  // and activation-gradient GEMMs, A streamed once) walk groups of 2 tile
  // rows, so the few A row panels in flight stay in L2 while every column
  // tile reads them (c4 z1: DRAM reads 1.44 -> 0.89 GB, 1641 -> 1611 us,
  // ncu); square weight-gradient GEMMs keep groups of 8 (d20: 1496 vs 1518 us)
  tp->group_m = group_env > 0 ? group_env : (tp->tiles_m >= 4 * tp->tiles_n ? 2 : GROUP_M);
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
  setup_tma_epilogue(p, tp, ctas, spec_prog);
  if (p.split_red && p.ksplit > 1) {
    if (p.epi.prog.n_stores != 1 || p.epi.out[0].st != (uint8_t)SType::F32) return false;
    tp->g.split_bytes = 0;  // every split addresses the one output
    if (!tp->et.on) tp->g.epi.out[0].st = (uint8_t)SType::F32_ADD;  // direct stores: red.global.add
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

// the hybrid's second stream and fork / join events: per host thread and
// device (concurrent callers never share an event), created outside stream
// capture
struct HybridAux {
  cudaStream_t aux = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
HybridAux* hybrid_aux(cudaStream_t stream) {
  thread_local HybridAux per_dev[16];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return nullptr;
  HybridAux& x = per_dev[dev];
  if (!x.aux) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return nullptr;
    if (cudaStreamCreateWithFlags(&x.aux, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      x.aux = nullptr;
      return nullptr;
    }
  }
  return &x;
}

// the hybrid runs when a zeroed counter is given, the shape suits multicast
// and there are at least two super tiles per cluster
bool use_hybrid(const GemmParams& p, int ctas) {
  if (mc_mode() != 1 || !p.hyb || !mc_shape_ok(p, ctas) || 4 * max_clusters4() >= num_sms() - 8) return false;
  const int64_t units = ((p.M + 4 * BM - 1) / (4 * BM)) * ((p.N + p.bn - 1) / p.bn) * std::max(p.ksplit, 1);
  return units >= 2 * max_clusters4() && num_sms() - 4 * max_clusters4() >= 2;
}

// (one static per kernel instantiation: the attribute is per function)
template <int BN, class PROG, int CTAS>
cudaError_t set_max_smem() {
  auto kern = gemm_tc_kernel<BN, PROG, CTAS>;
  // the max-dynamic-smem attribute is per device: one bit per device ordinal
  static std::atomic<uint64_t> configured{0};
  int dev = 0;
  cudaError_t e0 = cudaGetDevice(&dev);
  if (e0 != cudaSuccess) return e0;
  const uint64_t bit = 1ull << (dev & 63);
  if (!(configured.load(std::memory_order_relaxed) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem);
    if (e != cudaSuccess) return e;
    configured.fetch_or(bit);
  }
  return cudaSuccess;
}

// Hybrid: clusters of 4 on `stream` claim super tiles from the front of the
// work list, pairs on the auxiliary stream claim pair tiles from its back
// (hybrid_claim).  The pair launch waits for
// everything before the GEMM on `stream`, and `stream` waits for it after.
template <int BN, class PROG>
cudaError_t launch_hybrid(const GemmParams& p, cudaStream_t stream, HybridAux* x) {
  auto kern = gemm_tc_kernel<BN, PROG, 2>;
  cudaError_t e = set_max_smem<BN, PROG, 2>();
  if (e != cudaSuccess) return e;
  const bool spec = vm_cw<PROG>::value == 0;
  GemmParams q = p;
  q.sched = nullptr;
  TcParams ta, tb;
  if (!make_params(q, &ta, 2, spec, kRoleMc) || !make_params(q, &tb, 2, spec, kRoleSuper))
    return cudaErrorInvalidValue;
  const int units = ta.tiles_m * ta.tiles_n * std::max(p.ksplit, 1);
  const int nA = std::min(units, max_clusters4());
  const int nB = std::min(units - nA, (num_sms() - 4 * max_clusters4()) / 2);
  ta.sched = tb.sched = p.hyb;  // the 8-byte claim state (hybrid_claim)
  ta.unit0 = tb.unit0 = -1;     // every unit claimed, the first ones included
  if (nB > 0) {
    if ((e = cudaEventRecord(x->fork, stream)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(x->aux, x->fork, 0)) != cudaSuccess) return e;
  }
  LaunchCfg La(dim3((unsigned)(4 * nA), 1, 1), dim3(NUM_THREADS, 1, 1), launch_smem(ta, BN, 2), stream, 4, 1);
  if ((e = cudaLaunchKernelEx(&La.cfg, kern, ta)) != cudaSuccess) return e;
  if (nB > 0) {
    LaunchCfg Lb(dim3((unsigned)(2 * nB), 1, 1), dim3(NUM_THREADS, 1, 1), launch_smem(tb, BN, 2), x->aux, 2, 1,
                 /*pdl=*/false);
    if ((e = cudaLaunchKernelEx(&Lb.cfg, kern, tb)) != cudaSuccess) return e;
    if ((e = cudaEventRecord(x->join, x->aux)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(stream, x->join, 0)) != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

template <int BN, class PROG, int CTAS>
cudaError_t launch_ctas(const GemmParams& p, cudaStream_t stream) {
  auto kern = gemm_tc_kernel<BN, PROG, CTAS>;
  cudaError_t e0 = set_max_smem<BN, PROG, CTAS>();  // the attribute allows every launch's size
  if (e0 != cudaSuccess) return e0;
  if constexpr (CTAS == 2) {
    if (use_hybrid(p, CTAS))
      if (HybridAux* x = hybrid_aux(stream)) return launch_hybrid<BN, PROG>(p, stream, x);
  }
  TcParams tp;
  if (!make_params(p, &tp, CTAS, vm_cw<PROG>::value == 0)) return cudaErrorInvalidValue;
  // persistent: one CTA (pair, multicast cluster) per SM (pair, 4 SMs), up
  // to one per work item (tile x K split)
  int cluster = 1, grid = 1;
  grid_of(tp, CTAS, &cluster, &grid);
  LaunchCfg L(dim3((unsigned)grid, 1, 1), dim3(NUM_THREADS, 1, 1), launch_smem(tp, BN, CTAS), stream,
              (unsigned)cluster, 1);
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
