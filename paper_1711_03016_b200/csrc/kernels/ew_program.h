// Element-wise program format shared by the host planner and the device
// kernels (EW kernel body, GEMM epilogues).
//
// A program evaluates, per element of an iteration space, a DAG of the IR's
// element-wise instructions (unary `tanh`, `negate`, ...;
// binary `add`, `power`, ... with broadcasting; compare/select) in
// registers.  Slots: [0, n_in) are loads of the group inputs (for a GEMM
// epilogue slot 0 is the fp32 accumulator), [n_in, n_in + n_lits) literals,
// then one slot per instruction (SSA: instruction k writes slot
// n_in + n_lits + k).  Booleans are 0.0f / 1.0f in registers and one byte in
// memory.  Results leave the program through stores (same iteration space)
// and reductions (sum over rows / columns / everything, written as
// per-CTA partials and summed in a fixed order by a finalize step, so every
// run is bit-reproducible; reading A14).
#pragma once

#include "rtc_compat.h"

namespace dlvm {

constexpr int kMaxIterDims = 6;  // rank <= 5 with any broadcast pattern (+ a unit column)
constexpr int kMaxIn = 12;
constexpr int kMaxLits = 12;
constexpr int kMaxIns = 40;
constexpr int kMaxStores = 6;
constexpr int kMaxReduces = 4;
constexpr int kMaxSlots = kMaxIn + kMaxLits + kMaxIns;

// F32_ADD: an f32 output the kernels ACCUMULATE into (red.global.add) instead
// of storing -- possibly another GPU's memory over NVLink (dlvm.h DLVM_F32_ADD)
enum class SType : uint8_t { F32 = 0, BF16 = 1, U8 = 2, F32_ADD = 3 };

#if defined(__CUDACC__) || defined(__CUDACC_RTC__)
#define DLVM_HD __host__ __device__
#else
#define DLVM_HD
#endif
DLVM_HD constexpr int st_bytes(uint8_t st) {
  return st == (uint8_t)SType::F32 || st == (uint8_t)SType::F32_ADD ? 4 : st == (uint8_t)SType::BF16 ? 2 : 1;
}

enum VmOp : uint8_t {
  VM_NEG = 0, VM_TANH, VM_EXP, VM_LOG, VM_SQRT, VM_ABS, VM_SIGN,
  VM_ADD, VM_SUB, VM_MUL, VM_DIV, VM_POW,
  VM_LT, VM_LE, VM_GT, VM_GE, VM_EQ, VM_NE,
  VM_SELECT,
  VM_TOBOOL,   // dataTypeCast float -> bool: x != 0
  VM_COPY,     // dataTypeCast bool -> float (values already 0/1), identity
  // planner peepholes (reading A12: derivative closed forms evaluated from
  // the pre-activation, cancellation-free in fp32)
  VM_SECH2,    // subtract(1, multiply(tanh z, tanh z)) == sech^2(z), operand z
  VM_FMA,      // add(multiply(a, b), c) with one rounding (FMA contraction, reading A13)
  VM_NUM_OPS
};

enum RedKind : uint8_t {
  RED_COL = 0,  // sum over all row dims: partials [grid_rows, C]
  RED_ROW = 1,  // sum over the column dim: partials [R, grid_cols]
  RED_ALL = 2   // sum over everything: partials [grid_rows * grid_cols]
};

struct EwIns {
  uint8_t op, a, b, c;
};

struct EwProgram {
  uint8_t n_in = 0, n_lits = 0, n_ins = 0, n_stores = 0, n_reduces = 0;
  EwIns ins[kMaxIns];
  float lits[kMaxLits];
  uint8_t store_slot[kMaxStores];
  uint8_t reduce_slot[kMaxReduces];
  uint8_t reduce_kind[kMaxReduces];
};

inline int vm_arity(uint8_t op) {
  if (op <= VM_SIGN || op == VM_TOBOOL || op == VM_COPY || op == VM_SECH2) return 1;
  if (op == VM_SELECT || op == VM_FMA) return 3;
  return 2;
}

}  // namespace dlvm
