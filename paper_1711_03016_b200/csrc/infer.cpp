// Type / shape inference and verification (Fig. 2,
// "Analyses & Verification: ... Type Checking, Differentiability").
//
// One rule per opcode (Table 1):
//   unary            same type
//   binary/compare   broadcast shape ("All element-wise binary
//                    operators support broadcasting"; reading A1: right
//                    aligned, each dim pair equal or one of them 1, missing
//                    leading dims are 1); compare -> bool (Table 1)
//   select           broadcast of cond/a/b; cond bool
//   dot              rank 2, [m,k].[k,n] -> [m,n]  (Table 1; A19)
//   reduce along d   axis d removed                (Table 1; A2)
//   transpose        axes reversed                 (Table 1; A3)
//   shapeCast        element count preserved       (Table 1)
//   dataTypeCast     shape preserved               (Table 1)
//   slice a upto b   axis 0, half-open             (Table 1)
// Gradient declarations (§3.1.3; Fig. 3; reading A7):
//   params  = source params (+ seed of output `from`'s type, last, if seedable)
//   results = wrt argument types (wrt order) ++ kept output types.
#include <algorithm>
#include <map>
#include <set>

#include "ir.h"

namespace dlvm {

static const char* kDtypeNames[] = {"bool", "i8", "i16", "i32", "i64", "f16", "f32", "f64"};
static const char* kOpNames[] = {"negate", "tanh", "exp", "log", "sqrt", "abs", "sign",
                                 "add", "subtract", "multiply", "divide", "power",
                                 "lt", "le", "gt", "ge", "eq", "ne", "select", "dot", "reduce",
                                 "transpose", "shapeCast", "dataTypeCast", "slice", "sech2"};

const char* dtype_name(DType d) { return kDtypeNames[(int)d]; }
bool dtype_from_name(const std::string& s, DType* out) {
  for (int i = 0; i < 8; ++i)
    if (s == kDtypeNames[i]) {
      *out = (DType)i;
      return true;
    }
  return false;
}
const char* op_name(Op op) { return kOpNames[(int)op]; }
bool op_from_name(const std::string& s, Op* out) {
  for (int i = 0; i < (int)Op::Sech2; ++i)  // sech2 is planner-internal, not parseable
    if (s == kOpNames[i]) {
      *out = (Op)i;
      return true;
    }
  return false;
}

std::string Type::str() const {
  if (shape.empty()) return dtype_name(dtype);
  std::string s = "<";
  for (auto d : shape) s += std::to_string(d) + " x ";
  return s + dtype_name(dtype) + ">";
}

bool broadcast_shapes(const std::vector<int64_t>& a, const std::vector<int64_t>& b,
                      std::vector<int64_t>* out) {
  size_t n = std::max(a.size(), b.size());
  std::vector<int64_t> r(n);
  for (size_t i = 0; i < n; ++i) {
    int64_t x = i < n - a.size() ? 1 : a[i - (n - a.size())];
    int64_t y = i < n - b.size() ? 1 : b[i - (n - b.size())];
    if (x == y || y == 1)
      r[i] = x;
    else if (x == 1)
      r[i] = y;
    else
      return false;
  }
  *out = r;
  return true;
}

static std::string shape_str(const std::vector<int64_t>& s) {
  std::string r = "(";
  for (size_t i = 0; i < s.size(); ++i) r += (i ? ", " : "") + std::to_string(s[i]);
  return r + (s.size() == 1 ? ",)" : ")");
}

Type infer_inst(const Inst& in, const std::vector<Type>& t) {
  auto fail = [&](const std::string& m) -> void {
    throw Error(kStatusVerify, in.line, in.col, std::string("'") + op_name(in.op) + "': " + m);
  };
  auto bc = [&](const std::vector<int64_t>& a, const std::vector<int64_t>& b) {
    std::vector<int64_t> r;
    if (!broadcast_shapes(a, b, &r)) fail("shapes " + shape_str(a) + " and " + shape_str(b) + " are not broadcast-compatible");
    return r;
  };
  Op op = in.op;
  if (is_unary(op) || op == Op::Sech2) {
    if (t[0].dtype == DType::Bool) fail("operand must be numeric");
    if ((op == Op::Tanh || op == Op::Exp || op == Op::Log || op == Op::Sqrt) && !is_float(t[0].dtype))
      fail("operand must have a floating-point type");
    return t[0];
  }
  if (is_binary(op)) {
    if (t[0].dtype != t[1].dtype) fail("operand data types differ");
    if (t[0].dtype == DType::Bool) fail("operands must be numeric");
    if (op == Op::Power && !is_float(t[0].dtype)) fail("operands must have a floating-point type");
    return Type{bc(t[0].shape, t[1].shape), t[0].dtype};
  }
  if (is_compare(op)) {
    if (t[0].dtype != t[1].dtype) fail("operand data types differ");
    return Type{bc(t[0].shape, t[1].shape), DType::Bool};
  }
  switch (op) {
    case Op::Select: {
      if (t[0].dtype != DType::Bool) fail("condition must have type bool");
      if (t[1].dtype != t[2].dtype) fail("branch data types differ");
      return Type{bc(bc(t[0].shape, t[1].shape), t[2].shape), t[1].dtype};
    }
    case Op::Dot: {
      if (t[0].rank() != 2 || t[1].rank() != 2) fail("operands must be rank 2");
      if (t[0].shape[1] != t[1].shape[0]) fail("inner dimensions differ");
      if (t[0].dtype != t[1].dtype) fail("operand data types differ");
      if (t[0].dtype == DType::Bool) fail("operands must be numeric");
      return Type{{t[0].shape[0], t[1].shape[1]}, t[0].dtype};
    }
    case Op::Reduce: {
      int d = in.axis;
      if (t[0].rank() == 0 || d < 0 || d >= t[0].rank()) fail("axis out of range");
      if (t[0].dtype == DType::Bool) fail("operand must be numeric");
      Type r = t[0];
      r.shape.erase(r.shape.begin() + d);
      return r;
    }
    case Op::Transpose: {
      Type r = t[0];
      std::reverse(r.shape.begin(), r.shape.end());
      return r;
    }
    case Op::ShapeCast: {
      Type r{in.shape, t[0].dtype};
      if (r.numel() != t[0].numel()) fail("element count differs");
      return r;
    }
    case Op::DataTypeCast:
      return Type{t[0].shape, in.cast_to};
    case Op::Slice: {
      if (t[0].rank() == 0 || !(0 <= in.from && in.from < in.upto && in.upto <= t[0].shape[0]))
        fail("bounds out of range");
      Type r = t[0];
      r.shape[0] = in.upto - in.from;
      return r;
    }
    default:
      break;
  }
  fail("unknown opcode");
  return Type{};
}

static void infer_function(Function& f) {
  if (!f.has_body) return;
  if (f.arg_types.size() != f.params.size())
    throw Error(kStatusVerify, f.line, f.col, "entry block argument count does not match the function type");
  std::map<std::string, int> ids;
  std::vector<std::string> arg_names(f.names.begin(), f.names.begin() + f.arg_types.size());
  f.names.clear();
  f.types.clear();
  for (size_t i = 0; i < arg_names.size(); ++i) {
    auto [ln, cl] = f.arg_locs[i];
    if (f.arg_types[i] != f.params[i])
      throw Error(kStatusVerify, ln, cl, "argument %" + arg_names[i] + " has type " + f.arg_types[i].str() +
                                             ", function type says " + f.params[i].str());
    if (ids.count(arg_names[i])) throw Error(kStatusVerify, ln, cl, "redefinition of %" + arg_names[i]);
    ids[arg_names[i]] = f.add_value(arg_names[i], f.arg_types[i]);
  }
  auto resolve = [&](Operand& o) -> Type {
    if (o.vname.empty()) {
      o.value = -1;
      return o.type;
    }
    auto it = ids.find(o.vname);
    if (it == ids.end()) throw Error(kStatusVerify, o.line, o.col, "use of undefined value %" + o.vname);
    if (f.types[it->second] != o.type)
      throw Error(kStatusVerify, o.line, o.col,
                  "%" + o.vname + " has type " + f.types[it->second].str() + ", annotated " + o.type.str());
    o.value = it->second;
    return o.type;
  };
  for (auto& in : f.insts) {
    std::vector<Type> tys;
    for (auto& o : in.ops) tys.push_back(resolve(o));
    Type rt = infer_inst(in, tys);
    if (ids.count(in.rname)) throw Error(kStatusVerify, in.line, in.col, "redefinition of %" + in.rname);
    in.result = f.add_value(in.rname, rt);
    ids[in.rname] = in.result;
  }
  std::vector<Type> rts;
  for (auto& o : f.ret) rts.push_back(resolve(o));
  if (rts != f.results) throw Error(kStatusVerify, f.ret_line, 1, "return type does not match function type");
}

void expected_gradient_type(const Function& src, const GradConfig& c, std::vector<Type>* params,
                            std::vector<Type>* results) {
  auto fail = [&](const std::string& m) { throw Error(kStatusVerify, c.line, c.col, m); };
  int n_in = (int)src.params.size(), n_out = (int)src.results.size();
  std::vector<int> wrt = c.wrt;
  if (!c.has_wrt)
    for (int i = 0; i < n_in; ++i) wrt.push_back(i);
  if (std::set<int>(wrt.begin(), wrt.end()).size() != wrt.size()) fail("duplicate index in 'wrt'");
  if (std::set<int>(c.keeping.begin(), c.keeping.end()).size() != c.keeping.size())
    fail("duplicate index in 'keeping'");
  for (int i : wrt) {
    if (i < 0 || i >= n_in) fail("'wrt' index " + std::to_string(i) + " out of range");
    if (!is_float(src.params[i].dtype)) fail("argument " + std::to_string(i) + " has a non-differentiable type");
  }
  for (int j : c.keeping)
    if (j < 0 || j >= n_out) fail("'keeping' index " + std::to_string(j) + " out of range");
  int frm = c.has_from ? c.from : 0;
  if (frm < 0 || frm >= n_out) fail("'from' index out of range");
  if (!is_float(src.results[frm].dtype)) fail("selected output has a non-differentiable type");
  *params = src.params;
  if (c.seedable) params->push_back(src.results[frm]);
  results->clear();
  for (int i : wrt) results->push_back(src.params[i]);
  for (int j : c.keeping) results->push_back(src.results[j]);
}

// Active instructions (float result depending on a wrt argument) need an
// adjoint rule; reduce-by-multiply has none.
static void check_differentiable(const Function& src, const GradConfig& c) {
  std::vector<char> active(src.types.size(), 0);
  if (c.has_wrt) {
    for (int i : c.wrt) active[i] = 1;
  } else {
    for (int i = 0; i < src.num_args(); ++i) active[i] = 1;
  }
  for (auto& in : src.insts) {
    if (!is_float(src.types[in.result].dtype)) continue;
    bool act = false;
    for (auto& o : in.ops)
      if (!o.is_lit() && active[o.value]) act = true;
    if (!act) continue;
    if (in.op == Op::Reduce && in.reduce_mul)
      throw Error(kStatusVerify, in.line, in.col, "'reduce by multiply' is not differentiable");
    if (in.op == Op::DataTypeCast && !is_float(in.ops[0].type.dtype)) continue;
    active[in.result] = 1;
  }
}

void verify_module(Module& m) {
  for (auto& f : m.fns) {
    if (!f.grad && !f.has_body)
      throw Error(kStatusVerify, f.line, f.col, "function @" + f.name + " has no body and no gradient attribute");
    infer_function(f);
  }
  for (auto& f : m.fns) {
    if (!f.grad) continue;
    const GradConfig& c = *f.grad;
    if (f.has_body) throw Error(kStatusVerify, f.line, f.col, "a gradient declaration has no body");
    Function* src = m.find(c.source);
    if (!src) throw Error(kStatusVerify, c.line, c.col, "unknown function @" + c.source);
    std::vector<Type> p, r;
    expected_gradient_type(*src, c, &p, &r);
    if (p != f.params || r != f.results)
      throw Error(kStatusVerify, f.line, f.col,
                  "declared type of @" + f.name + " does not match the expected gradient type");
    if (src->has_body) {
      check_differentiable(*src, c);
    } else {
      // higher order: the source is itself a gradient
      // declaration; its canonical body (ad.cpp) must be differentiable too
      const Function body = canonical_function(m, c.source);
      check_differentiable(body, c);
    }
  }
}

}  // namespace dlvm
