// Host-visible kernel parameter blocks and launchers (sm_100a).
#pragma once

#ifndef __CUDACC_RTC__
#include <cuda_runtime.h>
#endif

#include "ew_program.h"

namespace dlvm {

// one program input: element (i_0..i_{n-1}) at ptr + sum_d i_d * s[d]
// (+ k * chunk_stride summed over k < nchunks for reduction partials;
// multiplied in k order instead when chunk_op == 1: `reduce ... by multiply`;
// their maximum when chunk_op == 2: `reduce ... by max`, reading A26)
struct EwDevIn {
  const void* ptr;
  int64_t s[kMaxIterDims];
  int64_t chunk_stride;
  int32_t nchunks;
  uint8_t st;  // SType
  uint8_t chunk_op;
};

struct EwDevOut {
  void* ptr;
  int64_t s[kMaxIterDims];
  uint8_t st;
};

struct EwParams {
  int32_t ndims;
  int32_t ncols;   // trailing dims forming the column index (1, or more when they do not collapse)
  int32_t vec;     // 1 or 4 elements per thread along the column dim
  int32_t rpt;     // rows per thread (EW kernel)
  int64_t dims[kMaxIterDims];
  int64_t gx, gy;  // grid (column tiles, row tiles)
  EwProgram prog;
  EwDevIn in[kMaxIn];
  EwDevOut out[kMaxStores];
  float* red[kMaxReduces];  // partial buffers
};

#ifndef __CUDACC_RTC__
// element-wise program kernel over an [R, C] iteration space
cudaError_t launch_ew(const EwParams& p, int bx, int by, cudaStream_t stream);
#endif

constexpr int kMaxSeg = 8;

// one K segment: sum_k A[m,k] B[k,n] over k < K
struct GemmSegParams {
  const void* a;  // bf16 or f32
  const void* b;
  int64_t K;
  int64_t a_s0, a_s1;  // A[m,k] at a + m*a_s0 + k*a_s1 (elements)
  int64_t b_s0, b_s1;  // B[k,n] at b + k*b_s0 + n*b_s1
  int32_t a_kmajor, b_kmajor;
};

// C[M,N] = sum over segments of A_s . B_s, then the epilogue program
struct GemmParams {
  int64_t M, N;
  int32_t n_seg;
  GemmSegParams seg[kMaxSeg];
  int32_t bf16;        // operand element type: 1 bf16, 0 f32
  int32_t bm, bn;      // tile; defines the epilogue partial layout
  EwParams epi;        // ndims 2, dims {M, N}; slot 0 = accumulator
  // epilogue inputs with contiguous rows (e.g. the saved ReLU mask): the TMA
  // producer prefetches each tile's rows into L2 while the tile's MMAs run
  // split K (single segment): work item t covers tile t % tiles, K range
  // split t / tiles of ksplit, and stores its raw accumulator to the single
  // output at + split * split_bytes (a following EW step sums the splits)
  int32_t ksplit;
  int64_t split_bytes;
  // split_red: instead, every work item adds its accumulator into out[0] (f32,
  // zeroed by the caller; program: store of the accumulator only), by TMA
  // reduce-add, else by red.global.add (SType::F32_ADD); split_bytes unused
  int32_t split_red;
  int* sched;                // tcgen05: zeroed work counter (dynamic tile scheduling) or nullptr
  int* hyb;                  // tcgen05: zeroed 8-byte claim state of a hybrid multicast + pair launch, or nullptr
  int32_t n_pf;
  const void* pf_ptr[4];
  int64_t pf_row_bytes[4];  // row stride in bytes
  int32_t pf_esize[4];      // element size in bytes
};

#ifndef __CUDACC_RTC__
cudaError_t launch_gemm_simt(const GemmParams& p, cudaStream_t stream);

// kernels compiled at create time (csrc/jit.cpp): same launch geometry as the
// ahead-of-time launchers, the CUfunction passed as `fn`
cudaError_t launch_ew_fn(void* fn, const EwParams& p, int bx, int by, cudaStream_t stream);
cudaError_t launch_gemm_tc_fn(void* fn, int ctas, const GemmParams& p, cudaStream_t stream);
cudaError_t launch_gemm_simt_fn(void* fn, const GemmParams& p, cudaStream_t stream);
int gemm_tc_ctas(int64_t M, int bn);  // 2: the launcher runs CTA pairs for this shape
bool gemm_hybrid_enabled();           // DLVM_GEMM_MC=1: large pair GEMMs may run as hybrid launches
cudaError_t launch_gemm_tc(const GemmParams& p, cudaStream_t stream);
bool gemm_tc_available();

// sum of reduction partials (p.in[0] with nchunks > 1) into p.out[*]
cudaError_t launch_finalize(const EwParams& p, cudaStream_t stream);

cudaError_t launch_cast_bf16(const float* src, void* dst, int64_t n, cudaStream_t stream);

// [rows, cols] f32 or bf16 (src_f32) -> bf16 rows of `ld` elements (ld >= cols)
cudaError_t launch_pack_bf16(const void* src, bool src_f32, int64_t rows, int64_t cols, void* dst, int64_t ld,
                             cudaStream_t stream);

#endif

}  // namespace dlvm
