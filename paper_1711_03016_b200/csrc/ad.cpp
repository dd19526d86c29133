// Reverse-mode AD by adjoint code generation (§3.1.3).
//
// "The canonicalization process first copies basic blocks and instructions
// from the original function to the new function body, and then applies
// adjoint code generation to the function" (L296).  `differentiate` does
// exactly that for a single-block function: copy the primal, then walk it
// in reverse program order emitting, per instruction, the IR of its adjoint
// rule (rule table), accumulating multi-use adjoints with `add` and
// unbroadcasting every element-wise contribution (reduce-add over the
// broadcast axes, then shapeCast).  Configurable AD (L308-309):
// `wrt` picks the arguments, `keeping` appends original outputs, `from`
// picks the differentiated output, `seedable` adds the seed as the last
// parameter (else the seed is an all-ones splat, reading A6).
//
// Forward activity (only values depending on a `wrt` argument receive
// adjoints) plus `dead_code_elim` (§3.1.4, "aggressive dead code
// elimination"; L304-305) remove e.g. the layer-1 input gradient of an MLP.
#include <cmath>
#include <cstdio>
#include <map>
#include <set>

#include "ir.h"

namespace dlvm {

namespace {

struct Builder {
  Function& g;
  int counter = 0;
  std::set<std::string> used;
  explicit Builder(Function& f) : g(f) {
    for (auto& n : f.names) used.insert(n);
  }
  std::string fresh(const char* stem) {
    for (;;) {
      std::string n = std::string(stem) + std::to_string(counter++);
      if (!used.count(n)) {
        used.insert(n);
        return n;
      }
    }
  }
  Operand V(int id) {
    Operand o;
    o.value = id;
    o.vname = g.names[id];
    o.type = g.types[id];
    return o;
  }
  static Operand L(double v, const Type& t) {
    Operand o;
    o.value = -1;
    o.lit = v;
    o.type = t;
    return o;
  }
  static Type scalar(DType d) { return Type{{}, d}; }
  Operand emit(Inst in) {
    std::vector<Type> tys;
    for (auto& o : in.ops) tys.push_back(o.type);
    Type rt = infer_inst(in, tys);
    in.rname = fresh("d");
    in.result = g.add_value(in.rname, rt);
    in.line = in.col = 0;
    g.insts.push_back(in);
    return V(in.result);
  }
  Operand op1(Op op, Operand a) {
    if (a.is_lit() && op == Op::Negate) return L(-a.lit, a.type);
    Inst in;
    in.op = op;
    in.ops = {a};
    return emit(in);
  }
  Operand op2(Op op, Operand a, Operand b) {
    Inst in;
    in.op = op;
    in.ops = {a, b};
    return emit(in);
  }
  Operand select(Operand c, Operand a, Operand b) {
    Inst in;
    in.op = Op::Select;
    in.ops = {c, a, b};
    return emit(in);
  }
  Operand reduce_add(Operand a, int axis) {
    Inst in;
    in.op = Op::Reduce;
    in.ops = {a};
    in.axis = axis;
    return emit(in);
  }
  Operand shape_cast(Operand a, const std::vector<int64_t>& s) {
    if (a.type.shape == s) return a;
    if (a.is_lit()) return L(a.lit, Type{s, a.type.dtype});
    if (s.empty()) {  // the text form has no rank-0 shapeCast: sum the unit axes away
      while (a.type.rank() > 0) a = reduce_add(a, a.type.rank() - 1);
      return a;
    }
    Inst in;
    in.op = Op::ShapeCast;
    in.ops = {a};
    in.shape = s;
    return emit(in);
  }
  Operand transpose(Operand a) {
    Inst in;
    in.op = Op::Transpose;
    in.ops = {a};
    return emit(in);
  }
  Operand dtype_cast(Operand a, DType d) {
    if (a.type.dtype == d) return a;
    Inst in;
    in.op = Op::DataTypeCast;
    in.ops = {a};
    in.cast_to = d;
    return emit(in);
  }
  // Sum a contribution over the axes broadcasting expanded.
  Operand unbroadcast(Operand c, const Type& t) {
    if (c.type.shape == t.shape) return c;
    int extra = c.type.rank() - t.rank();
    std::vector<int> axes;
    for (int i = 0; i < extra; ++i) axes.push_back(i);
    for (int i = 0; i < t.rank(); ++i)
      if (t.shape[i] == 1 && c.type.shape[i + extra] != 1) axes.push_back(i + extra);
    if (c.is_lit()) {  // a splat literal sums to a splat literal
      double k = 1;
      for (int a : axes) k *= (double)c.type.shape[a];
      return L(c.lit * k, t);
    }
    for (int k = (int)axes.size() - 1; k >= 0; --k) c = reduce_add(c, axes[k]);
    return shape_cast(c, t.shape);
  }
};

}  // namespace

Function differentiate(const Function& src, const GradConfig& cfg, const std::string& name) {
  Function g;
  g.name = name;
  g.has_body = true;
  g.label = "entry";
  expected_gradient_type(src, cfg, &g.params, &g.results);
  g.result_tuple = g.results.size() > 1;
  g.grad = cfg;
  const int n_in = src.num_args();
  std::vector<int> map(src.types.size(), -1);
  for (int i = 0; i < n_in; ++i) map[i] = g.add_value(src.names[i], src.types[i]);
  const int frm = cfg.has_from ? cfg.from : 0;
  int seed_id = -1;
  if (cfg.seedable) {
    std::string n = "seed";
    for (int k = 0;; ++k) {
      bool clash = false;
      for (auto& s : src.names) clash |= (s == n);
      if (!clash) break;
      n = "seed" + std::to_string(k);
    }
    seed_id = g.add_value(n, src.results[frm]);
  }
  for (int i = 0; i < (int)g.params.size(); ++i) g.arg_types.push_back(g.params[i]);
  // 1. copy the primal body (L296)
  auto remap = [&](Operand o) {
    if (!o.is_lit()) {
      o.value = map[o.value];
      o.vname = g.names[o.value];
    }
    return o;
  };
  for (const Inst& in : src.insts) {
    Inst c = in;
    for (auto& o : c.ops) o = remap(o);
    c.result = g.add_value(src.names[in.result], src.types[in.result]);
    map[in.result] = c.result;
    g.insts.push_back(c);
  }
  const size_t n_primal = g.insts.size();
  Builder b(g);

  // forward activity: which values depend on a wrt argument
  std::vector<int> wrt = cfg.wrt;
  if (!cfg.has_wrt)
    for (int i = 0; i < n_in; ++i) wrt.push_back(i);
  std::vector<char> active(g.types.size() + 1, 0);
  for (int i : wrt) active[map[i]] = 1;
  for (size_t k = 0; k < n_primal; ++k) {
    const Inst& in = g.insts[k];
    if (!is_float(g.types[in.result].dtype)) continue;
    for (auto& o : in.ops)
      if (!o.is_lit() && active[o.value]) active[in.result] = 1;
  }

  // 2. adjoint code generation, reverse program order
  std::map<int, Operand> adj;
  auto acc = [&](const Operand& target, Operand c) {
    if (target.is_lit() || !active[target.value] || !is_float(target.type.dtype)) return;
    c = b.unbroadcast(c, g.types[target.value]);
    auto it = adj.find(target.value);
    if (it == adj.end())
      adj.emplace(target.value, c);
    else if (it->second.is_lit() && c.is_lit())
      it->second = Builder::L(it->second.lit + c.lit, c.type);
    else
      it->second = b.op2(Op::Add, it->second, c);
  };
  const Operand out = remap(src.ret[frm]);
  if (!out.is_lit()) {
    Operand seed = cfg.seedable ? b.V(seed_id) : Builder::L(1.0, out.type);
    acc(out, seed);
  }
  for (size_t k = n_primal; k-- > 0;) {
    const Inst in = g.insts[k];  // copy: emission may reallocate the vector
    auto it = adj.find(in.result);
    if (it == adj.end()) continue;
    const Operand gr = it->second;
    const Operand y = b.V(in.result);
    const DType dt = y.type.dtype;
    auto lit = [&](double v) { return Builder::L(v, Builder::scalar(dt)); };
    const Operand a = in.ops.empty() ? Operand{} : in.ops[0];
    auto is_act = [&](const Operand& o) { return !o.is_lit() && active[o.value] && is_float(o.type.dtype); };
    switch (in.op) {
      case Op::Add:
        acc(in.ops[0], gr);
        acc(in.ops[1], gr);
        break;
      case Op::Subtract:
        acc(in.ops[0], gr);
        if (is_act(in.ops[1])) acc(in.ops[1], b.op1(Op::Negate, gr));
        break;
      case Op::Multiply:
        if (is_act(in.ops[0])) acc(in.ops[0], b.op2(Op::Multiply, gr, in.ops[1]));
        if (is_act(in.ops[1])) acc(in.ops[1], b.op2(Op::Multiply, gr, in.ops[0]));
        break;
      case Op::Divide:
        if (is_act(in.ops[0])) acc(in.ops[0], b.op2(Op::Divide, gr, in.ops[1]));
        if (is_act(in.ops[1])) {
          Operand num = b.op2(Op::Multiply, gr, in.ops[0]);
          Operand den = b.op2(Op::Multiply, in.ops[1], in.ops[1]);
          acc(in.ops[1], b.op1(Op::Negate, b.op2(Op::Divide, num, den)));
        }
        break;
      case Op::Power: {
        const Operand n = in.ops[1];
        if (is_act(a)) {
          Operand nm1 = n.is_lit() ? Builder::L(n.lit - 1.0, n.type) : b.op2(Op::Subtract, n, lit(1.0));
          Operand p = b.op2(Op::Power, a, nm1);
          acc(a, b.op2(Op::Multiply, gr, b.op2(Op::Multiply, n, p)));
        }
        if (is_act(n)) acc(n, b.op2(Op::Multiply, gr, b.op2(Op::Multiply, y, b.op1(Op::Log, a))));
        break;
      }
      case Op::Negate:
        acc(a, b.op1(Op::Negate, gr));
        break;
      case Op::Tanh:  // g * (1 - y*y)
        acc(a, b.op2(Op::Multiply, gr, b.op2(Op::Subtract, lit(1.0), b.op2(Op::Multiply, y, y))));
        break;
      case Op::Exp:
        acc(a, b.op2(Op::Multiply, gr, y));
        break;
      case Op::Log:
        acc(a, b.op2(Op::Divide, gr, a));
        break;
      case Op::Sqrt:
        acc(a, b.op2(Op::Divide, gr, b.op2(Op::Multiply, lit(2.0), y)));
        break;
      case Op::Abs:
        acc(a, b.op2(Op::Multiply, gr, b.op1(Op::Sign, a)));
        break;
      case Op::Sign:
        break;  // zero derivative
      case Op::Select: {
        const Operand& c = in.ops[0];
        if (is_act(in.ops[1])) acc(in.ops[1], b.select(c, gr, lit(0.0)));
        if (is_act(in.ops[2])) acc(in.ops[2], b.select(c, lit(0.0), gr));
        break;
      }
      case Op::Dot:  // (g . b^T, a^T . g)
        if (is_act(in.ops[0])) acc(in.ops[0], b.op2(Op::Dot, gr, b.transpose(in.ops[1])));
        if (is_act(in.ops[1])) acc(in.ops[1], b.op2(Op::Dot, b.transpose(in.ops[0]), gr));
        break;
      case Op::Transpose:
        acc(a, b.transpose(gr));
        break;
      case Op::Reduce: {  // broadcast g back along the reduced axis
        std::vector<int64_t> s = a.type.shape;
        s[in.axis] = 1;
        if (in.reduce_max) {
          // reading A26: g / k at the k positions equal to the max, else 0
          Operand at = b.op2(Op::Eq, a, b.shape_cast(b.V(in.result), s));
          Operand cnt = b.reduce_add(b.dtype_cast(at, a.type.dtype), in.axis);
          Operand q = b.op2(Op::Divide, b.shape_cast(gr, s), b.shape_cast(cnt, s));
          acc(a, b.select(at, q, Builder::L(0.0, Builder::scalar(a.type.dtype))));
          break;
        }
        Operand e = b.shape_cast(gr, s);
        acc(a, b.op2(Op::Multiply, e, Builder::L(1.0, a.type)));
        break;
      }
      case Op::ShapeCast:
        acc(a, b.shape_cast(gr, a.type.shape));
        break;
      case Op::DataTypeCast:
        if (is_float(a.type.dtype)) acc(a, b.dtype_cast(gr, a.type.dtype));
        break;
      case Op::Slice:
        throw Error(kStatusUnsupported, in.line, in.col, "differentiating 'slice' is not supported");
      default:  // compare: no adjoint
        break;
    }
  }
  // 3. results: grads in wrt order, then kept outputs (reading A7)
  for (int i : wrt) {
    auto it = adj.find(map[i]);
    g.ret.push_back(it != adj.end() ? it->second : Builder::L(0.0, src.params[i]));
  }
  for (int j : cfg.keeping) g.ret.push_back(remap(src.ret[j]));
  dead_code_elim(g);
  return g;
}

namespace {
Function canonical_rec(const Module& m, const std::string& name, std::vector<std::string>& stack) {
  const Function* f = nullptr;
  for (auto& g : m.fns)
    if (g.name == name) f = &g;
  if (!f) throw Error(kStatusVerify, 0, 0, "unknown function @" + name);
  if (f->has_body) return *f;
  if (!f->grad) throw Error(kStatusVerify, f->line, f->col, "function @" + name + " has no body and no gradient attribute");
  for (auto& s : stack)
    if (s == name) throw Error(kStatusVerify, f->grad->line, f->grad->col, "cyclic gradient declaration @" + name);
  stack.push_back(name);
  Function src = canonical_rec(m, f->grad->source, stack);
  stack.pop_back();
  return differentiate(src, *f->grad, f->name);
}
}  // namespace

Function canonical_function(const Module& m, const std::string& name) {
  std::vector<std::string> stack;
  return canonical_rec(m, name, stack);
}

// Remove instructions that do not (transitively) contribute to the result.
void dead_code_elim(Function& f) {
  std::vector<char> live(f.types.size(), 0);
  for (auto& o : f.ret)
    if (!o.is_lit()) live[o.value] = 1;
  for (size_t k = f.insts.size(); k-- > 0;) {
    if (!live[f.insts[k].result]) continue;
    for (auto& o : f.insts[k].ops)
      if (!o.is_lit()) live[o.value] = 1;
  }
  std::vector<Inst> keep;
  for (auto& in : f.insts)
    if (live[in.result]) keep.push_back(in);
  f.insts.swap(keep);
}

// Textual form (Fig. 3 syntax), used by dlvm_fn_print and the golden tests.
static std::string lit_str(double v) {
  char buf[64];
  if (std::isfinite(v) && v == std::floor(v) && std::fabs(v) < 1e15)
    std::snprintf(buf, sizeof buf, "%.0f", v);
  else
    std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

static std::string opnd(const Function& f, const Operand& o) {
  if (o.is_lit()) {
    std::string v = o.type.dtype == DType::Bool ? (o.lit != 0 ? "true" : "false") : lit_str(o.lit);
    return v + ": " + o.type.str();
  }
  return "%" + f.names[o.value] + ": " + f.types[o.value].str();
}

std::string print_function(const Function& f) {
  std::string s = "func @" + f.name + ": (";
  for (size_t i = 0; i < f.params.size(); ++i) s += (i ? ", " : "") + f.params[i].str();
  s += ") -> ";
  if (f.result_tuple) s += "(";
  for (size_t i = 0; i < f.results.size(); ++i) s += (i ? ", " : "") + f.results[i].str();
  if (f.result_tuple) s += ")";
  if (!f.has_body) return s + "\n";
  s += " {\n'" + f.label + "(";
  for (size_t i = 0; i < f.params.size(); ++i)
    s += (i ? ", %" : "%") + f.names[i] + ": " + f.params[i].str();
  s += "):\n";
  for (auto& in : f.insts) {
    s += "    %" + f.names[in.result] + " = " + op_name(in.op) + " ";
    for (size_t k = 0; k < in.ops.size(); ++k) s += (k ? ", " : "") + opnd(f, in.ops[k]);
    if (in.op == Op::Reduce)
      s += std::string(" by ") + (in.reduce_mul ? "multiply" : in.reduce_max ? "max" : "add") + " along " +
           std::to_string(in.axis);
    if (in.op == Op::ShapeCast) {
      s += " to ";
      for (size_t k = 0; k < in.shape.size(); ++k) s += (k ? " x " : "") + std::to_string(in.shape[k]);
    }
    if (in.op == Op::DataTypeCast) s += std::string(" to ") + dtype_name(in.cast_to);
    if (in.op == Op::Slice) s += " from " + std::to_string(in.from) + " upto " + std::to_string(in.upto);
    s += "\n";
  }
  s += "    return ";
  if (f.ret.size() > 1) s += "(";
  for (size_t k = 0; k < f.ret.size(); ++k) s += (k ? ", " : "") + opnd(f, f.ret[k]);
  if (f.ret.size() > 1) s += ")";
  return s + "\n}\n";
}

}  // namespace dlvm
