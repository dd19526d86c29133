// DLVM IR core (C++17, host only).
//
// In-memory form of the straight-line DLVM IR: module -> function -> one
// basic block -> instructions (§3.1.1, "module, function,
// basic block, and instruction"; Table 1).  Only single-block
// functions are represented: the hot path is straight-line
// MLP code, and the paper gives no reverse-mode algorithm over CFGs.
//
// This is an independent implementation from oracle/ (which is Python); the
// two share no code.
#pragma once

#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace dlvm {

enum class DType : uint8_t { Bool, I8, I16, I32, I64, F16, F32, F64 };
const char* dtype_name(DType d);
bool dtype_from_name(const std::string& s, DType* out);
inline bool is_float(DType d) { return d == DType::F16 || d == DType::F32 || d == DType::F64; }

struct Type {
  std::vector<int64_t> shape;  // empty = rank-0 scalar
  DType dtype = DType::F32;
  int rank() const { return (int)shape.size(); }
  int64_t numel() const {
    int64_t n = 1;
    for (auto d : shape) n *= d;
    return n;
  }
  bool operator==(const Type& o) const { return shape == o.shape && dtype == o.dtype; }
  bool operator!=(const Type& o) const { return !(*this == o); }
  std::string str() const;
};

enum class Op : uint8_t {
  // element-wise unary (Table 1)
  Negate, Tanh, Exp, Log, Sqrt, Abs, Sign,
  // element-wise binary with broadcasting (Table 1)
  Add, Subtract, Multiply, Divide, Power,
  // compare -> bool (Table 1)
  Lt, Le, Gt, Ge, Eq, Ne,
  Select,
  Dot,          // Table 1
  Reduce,       // Table 1
  Transpose,    // Table 1
  ShapeCast,    // Table 1
  DataTypeCast, // Table 1
  Slice,        // Table 1
  Sech2,        // planner-internal: subtract(1, multiply(tanh z, tanh z)) == sech^2(z) (reading A12)
  DotSum,       // planner-internal: dot(A1,B1) + ... + dot(As,Bs), one GEMM with s K segments
};
const char* op_name(Op op);
bool op_from_name(const std::string& s, Op* out);
inline bool is_unary(Op o) { return o <= Op::Sign; }
inline bool is_binary(Op o) { return o >= Op::Add && o <= Op::Power; }
inline bool is_compare(Op o) { return o >= Op::Lt && o <= Op::Ne; }
inline bool is_elementwise(Op o) { return o <= Op::Select; }

// An operand: an SSA value (function argument or instruction result) or a
// literal (`2: f32`, reading A8; a literal with a tensor type is a splat).
struct Operand {
  int value = -1;  // SSA id, or -1 for a literal
  double lit = 0;
  std::string vname;  // value name as written (resolved by the verifier)
  Type type;       // annotated type (== the value's type after verification)
  int line = 0, col = 0;
  bool is_lit() const { return value < 0; }
};

struct Inst {
  Op op = Op::Add;
  std::vector<Operand> ops;
  int result = -1;
  std::string rname;          // result name as written
  // attributes
  int axis = 0;               // reduce
  bool reduce_mul = false;    // reduce by multiply (else add)
  bool reduce_max = false;    // reduce by max (extension, reading A26)
  std::vector<int64_t> shape; // shapeCast target
  DType cast_to = DType::F32; // dataTypeCast target
  int64_t from = 0, upto = 0; // slice
  int line = 0, col = 0;
};

struct GradConfig {
  std::string source;
  bool has_wrt = false;
  std::vector<int> wrt;      // zero-based argument indices (default all)
  std::vector<int> keeping;  // zero-based output indices
  bool has_from = false;
  int from = 0;
  bool seedable = false;
  int line = 0, col = 0;
};

struct Function {
  std::string name;
  std::vector<Type> params, results;
  bool result_tuple = false;
  bool has_body = false;
  std::string label;
  // SSA value table: ids 0..params.size()-1 are the entry block arguments.
  std::vector<std::string> names;
  std::vector<Type> types;
  std::vector<std::pair<int, int>> arg_locs;  // (line, col) of entry block arguments
  std::vector<Type> arg_types;                // as written in the entry block
  std::vector<Inst> insts;
  std::vector<Operand> ret;
  int ret_line = 0;
  std::optional<GradConfig> grad;
  int line = 0, col = 0;

  int add_value(const std::string& n, const Type& t) {
    names.push_back(n);
    types.push_back(t);
    return (int)names.size() - 1;
  }
  int num_args() const { return (int)params.size(); }
};

struct Module {
  std::string name;
  std::string stage;
  std::vector<Function> fns;
  Function* find(const std::string& n) {
    for (auto& f : fns)
      if (f.name == n) return &f;
    return nullptr;
  }
};

// Errors carry the C-ABI status class (dlvm.h): 2 parse, 1 verify, 6 unsupported.
struct Error : std::runtime_error {
  int status;
  int line, col;
  Error(int st, int ln, int cl, const std::string& msg)
      : std::runtime_error(std::to_string(ln) + ":" + std::to_string(cl) + ": error: " + msg),
        status(st), line(ln), col(cl) {}
};
constexpr int kStatusVerify = 1, kStatusParse = 2, kStatusUsage = 3, kStatusRuntime = 4,
              kStatusCuda = 5, kStatusUnsupported = 6;

// parser.cpp
Module parse_module(const std::string& text);
// infer.cpp
bool broadcast_shapes(const std::vector<int64_t>& a, const std::vector<int64_t>& b,
                      std::vector<int64_t>* out);
Type infer_inst(const Inst& in, const std::vector<Type>& tys);
void verify_module(Module& m);  // types every function; checks gradient declarations
void expected_gradient_type(const Function& src, const GradConfig& cfg, std::vector<Type>* params,
                            std::vector<Type>* results);
// ad.cpp
Function differentiate(const Function& src, const GradConfig& cfg, const std::string& name);
// The function `name` with a body: as written, or its gradient declaration
// canonicalised by `differentiate` (recursively: a declaration of a
// declaration is a higher-order gradient).  Throws a
// verify error for cycles and unknown sources.
Function canonical_function(const Module& m, const std::string& name);
void dead_code_elim(Function& f);
// create-time optimiser (opt.cpp): algebra simplification, CSE, matrix-chain
// reordering, DCE -- value-preserving in exact arithmetic
void optimize_function(Function& f);
// printer.cpp
std::string print_function(const Function& f);

}  // namespace dlvm
