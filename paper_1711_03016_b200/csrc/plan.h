// Launch planner: partitions a typed straight-line function into fused
// sm_100a launch groups (the B200 replacement of the paper's "Compute
// Generation" / "Compute Scheduling" stages, Fig. 2, and of
// "fuse compatible element-wise operators to a single kernel to minimize
// the latency between kernel launches"; "linear algebra fusion ...
// Wx + b").
//
// Two kernel families execute every plan:
//   * EW   -- an element-wise program over a strided iteration space with
//             broadcasting loads, stores and row/column/full reductions
//             (partials, finalised deterministically by their consumer);
//   * GEMM -- `dot` (operand major-ness absorbs `transpose`) whose
//             accumulator feeds the same element-wise program as epilogue
//             (bias, activation, activation derivative, column sums).
// The program format (EwProgram) is shared by both, and by the host.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "ir.h"
#include "kernels/ew_program.h"

namespace dlvm {

enum class Policy { F32 = 0, BF16 = 1 };

// A device buffer the plan refers to.  Pointers are bound at run time.
struct BufferSlot {
  enum Kind { Input, Output, Seed, Work } kind = Work;
  int index = -1;      // input / output index
  size_t offset = 0;   // Work: byte offset into the workspace
  size_t bytes = 0;
  SType st = SType::F32;
  int cast_of = -1;    // Work buffer holding a bf16 cast of Input `cast_of` (see CastStep)
  int64_t cast_ld = 0; // ... with rows padded to this many elements (0: dense)
};

// Strided view of a buffer: element (i_0..i_{r-1}) of the value lives at
// offset + sum_j i_j * strides[j] (elements); if nchunks > 1 the value is
// the sum over k < nchunks of the element at + k * chunk_stride (partials).
struct TensorRef {
  int buf = -1;
  int64_t offset = 0;
  std::vector<int64_t> shape, strides;
  int nchunks = 1;
  int64_t chunk_stride = 0;
  SType st = SType::F32;
  bool contiguous() const;
};

constexpr int kPlanDims = 8;  // iteration rank while planning (collapsed to kMaxIterDims)

// An iteration-space operand of a kernel (input load or output store).
struct IterRef {
  int buf = -1;                  // -2: the GEMM accumulator (epilogue slot 0)
  int64_t offset = 0;
  int64_t strides[kPlanDims] = {0, 0, 0, 0, 0, 0, 0, 0};  // per iteration dim
  int nchunks = 1;
  int64_t chunk_stride = 0;
  uint8_t chunk_op = 0;          // chunks summed (0), multiplied in order (1, `reduce ... by multiply`) or maxed (2, `by max`)
  SType st = SType::F32;
  // reductions with a single partial: the value's f32 home, which the
  // producer writes directly when that buffer is bound as f32 at run time
  int direct_buf = -1;
};

struct EwGroup {
  // iteration space, row-major: dims[0..ndims-2] are "row" dims, dims[ndims-1]
  // is the column dim (ndims <= kMaxIterDims).
  int ndims = 1;
  int ncols = 1;                 // trailing dims forming the column index (1, or more when they do not collapse)
  int64_t dims[kMaxIterDims] = {1, 1, 1, 1, 1, 1};
  static_assert(kMaxIterDims == 6, "initialise every dim to 1");
  // launch shape (fixed at plan time: it determines the partials layout)
  int vec = 1, bx = 32, by = 8, rpt = 1;
  int64_t gx = 1, gy = 1;
  EwProgram prog;
  std::vector<IterRef> inputs;   // prog input slots 0..n_in-1 (GEMM: slot 0 is the accumulator)
  std::vector<IterRef> stores;   // prog.stores[k] -> stores[k]
  std::vector<IterRef> reduces;  // prog.reduces[k] -> partial buffer (contiguous)
  std::string desc;
  std::string sig;               // program_signature(prog): key of compile-time specialisations
  bool finalize = false;         // sum of reduction partials (dedicated kernel)
  int direct_buf = -1;           // finalize: skipped when this buffer is bound as f32 (producer wrote it)
};

constexpr int kPlanMaxSeg = 8;  // == kMaxSeg of kernels.h (checked in capi.cpp)

// one K segment of a GEMM: the product a . b accumulated with the others
struct GemmSeg {
  TensorRef a, b;                // a: [M,K], b: [K,N]; one unit stride each
  int64_t K = 0;
  bool a_kmajor = true, b_kmajor = false;
};

struct GemmStep {
  int64_t M = 0, N = 0, K = 0;   // K: total over the segments
  // sum of products (linear algebra fusion: W x + U h + b
  // is one GEMM whose K loop walks both products into one accumulator)
  std::vector<GemmSeg> seg;
  bool tensor_core = false;      // tcgen05 (bf16) vs SIMT (f32/bf16 operands)
  int ksplit = 1;                // > 1: K split into raw partial tiles, summed by the next EW step
  int64_t split_bytes = 0;       // byte stride between the partial tiles
  // ksplit == 2 and the next EW step only stores the sum of the partials
  // into a home with unit column stride: when that home is bound as f32 at
  // run time, the executor zeroes it and the GEMM adds both splits into it
  // (GemmParams::split_red), skipping the partials and the EW step.
  // 0 + a + b rounds once per add in either order: fl(a + b), bit-identical
  // to the EW step's partial0 + partial1 (DLVM_GEMM_SPLITRED=0 disables)
  bool split_red_ok = false;
  int bm = 128, bn = 128;        // tile shape (partials layout of epilogue reductions)
  EwGroup epi;                   // iteration space [M, N]; input slot 0 = accumulator
  int sched_index = -1;          // tcgen05: this GEMM's work counter in Plan::sched_buf (dynamic scheduling)
};

struct CastStep {                // bf16 copy of an input (cast from f32 and/or rows padded to ld)
  int input = -1;
  int dst_buf = -1;
  int64_t numel = 0;
  int64_t cols = 0, ld = 0;      // ld > 0: destination rows padded to ld elements (always runs)
};

struct Step {
  enum Kind { EW, GEMM, CAST, EVENT } kind = EW;
  EwGroup ew;
  GemmStep gemm;
  CastStep cast;
  int event_index = -1;          // EVENT: gradient index whose value is final
  std::string desc;
  // a kernel launch counted by num_launches / launch events (conditional
  // finalizes of single-partial reductions are not: they run only when the
  // reduced output is bound as bf16)
  bool counted_launch() const {
    if (kind == EW) return !(ew.finalize && ew.direct_buf >= 0);
    return kind == GEMM || (kind == CAST && cast.ld);
  }
};

struct Plan {
  std::vector<BufferSlot> bufs;
  std::vector<Step> steps;
  size_t workspace_bytes = 0;
  int n_inputs = 0, n_outputs = 0;
  bool seed_is_input = false;    // gradient plans: last parameter is the seed
  std::vector<int> input_bf16_ok;  // per input: 1 if it may be passed as bf16 (see make_plan)
  std::vector<int> input_u8_ok;    // per input: 1 if it may be passed as bool bytes (0/1 values; not a dot operand)
  int sched_buf = -1, n_sched = 0;  // work counters of the tcgen05 GEMMs (zeroed at the start of a run)
  bool hybrid_counters = false;     // some GEMM may run as a hybrid launch: zero the counters every run
  int launches() const;
  std::string str() const;
  std::string detail() const;  // str() + buffers and every step's operand refs
};

struct PlanOptions {
  Policy policy = Policy::F32;
  bool no_fusion = false;
  bool specialize = true;
  int n_grads = 0;               // gradient plans: outputs [0, n_grads) get ready events
};

Plan make_plan(const Function& f, const PlanOptions& opt);

// "i<n_in>l<n_lits>|op,a,b,c;...|s<slot>,...|r<slot>:<kind>,..." -- everything
// about a program that is fixed at compile time in a specialisation
// (pointers, strides, sizes, storage types and literal values are not).
std::string program_signature(const EwProgram& p);

}  // namespace dlvm
