// Create-time IR optimisation (§3.1.2, "domain-specific
// optimizations, such as algebra simplification, linear algebra fusion,
// matrix multiplication reordering, ... and traditional compiler
// optimizations"; §3.1.4 L318 CSE).  Runs on the primal and on the generated
// gradient function before planning (AD is a source transformation, so the
// gradient is optimised separately, L300-301).  Every rewrite preserves the
// value a function computes in exact arithmetic; it only ever replaces a
// value by an operand of identical type (no shape change through
// broadcasting).
//
//  * algebra simplification (L227-229): x^2 -> x*x, x^0 -> 1, x^1 -> x,
//    x^-1 -> 1/x, x*1 -> x, x+0 / x-0 -> x, x/1 -> x, -(-x) -> x,
//    transpose(transpose(x)) -> x; splat literals fold through arithmetic,
//    views and sums (the planner expects view/reduce operands to be values);
//  * common subexpression elimination (identical opcode, operands and
//    attributes; straight-line SSA, so the earlier value dominates);
//  * matrix-chain reordering (L230): (A.B).C <-> A.(B.C) when the inner
//    product is used once and the other association needs fewer
//    multiply-adds, repeated to a fixpoint (each rotation lowers the cost);
//  * dead-code elimination.
// Linear algebra fusion itself is a planner decision (plan.cpp: epilogues,
// DotSum).
#include <map>
#include <sstream>

#include "ir.h"

namespace dlvm {

namespace {

struct Optimizer {
  Function& f;
  int counter = 0;

  explicit Optimizer(Function& fn) : f(fn) {}

  Operand V(int id) const {
    Operand o;
    o.value = id;
    o.vname = f.names[id];
    o.type = f.types[id];
    return o;
  }
  static Operand L(double v, const Type& t) {
    Operand o;
    o.value = -1;
    o.lit = v;
    o.type = t;
    return o;
  }
  std::string fresh() {
    for (;;) {
      std::string n = "opt" + std::to_string(counter++);
      bool clash = false;
      for (auto& s : f.names) clash |= s == n;
      if (!clash) return n;
    }
  }
  std::vector<int> defs() const {
    std::vector<int> d(f.types.size(), -1);
    for (size_t k = 0; k < f.insts.size(); ++k) d[f.insts[k].result] = (int)k;
    return d;
  }
  std::vector<int> uses() const {
    std::vector<int> u(f.types.size(), 0);
    for (auto& in : f.insts)
      for (auto& o : in.ops)
        if (!o.is_lit()) ++u[o.value];
    for (auto& o : f.ret)
      if (!o.is_lit()) u[o.value] += 1000;  // returned: never "single use"
    return u;
  }
  // replace every use of value v by operand r (same type)
  void rauw(int v, const Operand& r) {
    auto sub = [&](Operand& o) {
      if (o.is_lit() || o.value != v) return;
      const int line = o.line, col = o.col;
      o = r;
      o.line = line;
      o.col = col;
    };
    for (auto& in : f.insts)
      for (auto& o : in.ops) sub(o);
    for (auto& o : f.ret) sub(o);
  }

  static bool lit_is(const Operand& o, double v) { return o.is_lit() && o.lit == v; }

  bool simplify() {
    bool changed = false;
    std::vector<int> d = defs();
    for (auto& in : f.insts) {
      const Type rt = f.types[in.result];
      if (!is_float(rt.dtype)) continue;
      auto same = [&](const Operand& o) { return o.type == rt; };
      const int r = in.result;
      if ((in.op == Op::Add || in.op == Op::Subtract || in.op == Op::Multiply || in.op == Op::Divide) &&
          in.ops[0].is_lit() && in.ops[1].is_lit()) {  // splat (op) splat
        const double a = in.ops[0].lit, b = in.ops[1].lit;
        const double v = in.op == Op::Add ? a + b : in.op == Op::Subtract ? a - b : in.op == Op::Multiply ? a * b : a / b;
        rauw(r, L(v, rt));
        changed = true;
        continue;
      }
      switch (in.op) {
        case Op::Power: {
          const Operand a = in.ops[0], n = in.ops[1];
          if (lit_is(n, 1.0) && same(a)) {
            rauw(r, a);
            changed = true;
          } else if (lit_is(n, 0.0)) {  // IEEE pow(x, 0) == 1 for every x, NaN included
            rauw(r, L(1.0, rt));
            changed = true;
          } else if (lit_is(n, 2.0) && !a.is_lit() && same(a)) {
            in.op = Op::Multiply;
            in.ops = {a, a};
            changed = true;
          } else if (lit_is(n, -1.0) && !a.is_lit() && same(a)) {
            in.op = Op::Divide;
            in.ops = {L(1.0, Type{{}, rt.dtype}), a};
            changed = true;
          }
          break;
        }
        case Op::Multiply:
          if (lit_is(in.ops[1], 1.0) && same(in.ops[0])) {
            rauw(r, in.ops[0]);
            changed = true;
          } else if (lit_is(in.ops[0], 1.0) && same(in.ops[1])) {
            rauw(r, in.ops[1]);
            changed = true;
          }
          break;
        case Op::Add:
          if (lit_is(in.ops[1], 0.0) && same(in.ops[0])) {
            rauw(r, in.ops[0]);
            changed = true;
          } else if (lit_is(in.ops[0], 0.0) && same(in.ops[1])) {
            rauw(r, in.ops[1]);
            changed = true;
          }
          break;
        case Op::Subtract:
        case Op::Divide:
          if (lit_is(in.ops[1], in.op == Op::Subtract ? 0.0 : 1.0) && same(in.ops[0])) {
            rauw(r, in.ops[0]);
            changed = true;
          }
          break;
        case Op::ShapeCast:
          // views of a splat literal are that literal at the view's type
          // (a simplified operand may have become a literal; the planner
          // expects view and reduce operands to be values)
          if (in.ops[0].is_lit()) {
            rauw(r, L(in.ops[0].lit, rt));
            changed = true;
          }
          break;
        case Op::Reduce:
          if (in.ops[0].is_lit()) {  // sum / product / max of n copies
            const int64_t n = in.ops[0].type.shape[in.axis];
            double x = in.reduce_mul ? 1.0 : in.reduce_max ? in.ops[0].lit : in.ops[0].lit * (double)n;
            if (in.reduce_mul)
              for (int64_t k = 0; k < n; ++k) x *= in.ops[0].lit;
            rauw(r, L(x, rt));
            changed = true;
          }
          break;
        case Op::Negate:
        case Op::Transpose: {
          if (in.ops[0].is_lit()) {
            rauw(r, L(in.op == Op::Negate ? -in.ops[0].lit : in.ops[0].lit, rt));
            changed = true;
            break;
          }
          const Operand& a = in.ops[0];
          if (a.is_lit() || d[a.value] < 0) break;
          const Inst& inner = f.insts[d[a.value]];
          if (inner.op == in.op && !inner.ops[0].is_lit() && inner.ops[0].type == rt) {
            rauw(r, inner.ops[0]);
            changed = true;
          }
          break;
        }
        default:
          break;
      }
    }
    return changed;
  }

  static std::string key(const Inst& in) {
    std::ostringstream k;
    k << (int)in.op;
    for (auto& o : in.ops) {
      if (o.is_lit())
        k << "|L" << o.lit << ":" << o.type.str();
      else
        k << "|v" << o.value;
    }
    k << "|a" << in.axis << (in.reduce_mul ? "m" : in.reduce_max ? "x" : "a") << "|c" << (int)in.cast_to << "|f" << in.from << ":" << in.upto
      << "|s";
    for (auto s : in.shape) k << s << ",";
    return k.str();
  }

  bool cse() {
    bool changed = false;
    std::map<std::string, int> seen;
    for (auto& in : f.insts) {
      const std::string k = key(in);
      auto it = seen.find(k);
      if (it != seen.end() && f.types[it->second] == f.types[in.result]) {
        rauw(in.result, V(it->second));
        changed = true;
      } else {
        seen.emplace(k, in.result);
      }
    }
    return changed;
  }

  // (A.B).C <-> A.(B.C): multiply-adds m*k*n + m*n*p versus k*n*p + m*k*p
  bool reorder_chains() {
    std::vector<int> d = defs(), u = uses();
    for (size_t k = 0; k < f.insts.size(); ++k) {
      const Inst in = f.insts[k];
      if (in.op != Op::Dot || in.ops[0].is_lit() || in.ops[1].is_lit()) continue;
      for (int side = 0; side < 2; ++side) {
        const Operand& inner_op = in.ops[side];
        const int di = d[inner_op.value];
        if (di < 0 || u[inner_op.value] != 1) continue;
        const Inst inner = f.insts[di];
        if (inner.op != Op::Dot || inner.ops[0].is_lit() || inner.ops[1].is_lit()) continue;
        // left-nested (side 0): (A.B).C ; right-nested (side 1): A.(B.C)
        const Operand A = side == 0 ? inner.ops[0] : in.ops[0];
        const Operand B = side == 0 ? inner.ops[1] : inner.ops[0];
        const Operand C = side == 0 ? in.ops[1] : inner.ops[1];
        const double m = (double)A.type.shape[0], kk = (double)A.type.shape[1], n = (double)B.type.shape[1],
                     p = (double)C.type.shape[1];
        const double left = m * kk * n + m * n * p, right = kk * n * p + m * kk * p;
        const bool to_right = side == 0 && right < left;
        const bool to_left = side == 1 && left < right;
        if (!to_right && !to_left) continue;
        Inst t;
        t.op = Op::Dot;
        t.ops = to_right ? std::vector<Operand>{B, C} : std::vector<Operand>{A, B};
        std::vector<Type> tys{t.ops[0].type, t.ops[1].type};
        const Type tt = infer_inst(t, tys);
        t.rname = fresh();
        t.result = f.add_value(t.rname, tt);
        Inst& out = f.insts[k];
        out.ops = to_right ? std::vector<Operand>{A, V(t.result)} : std::vector<Operand>{V(t.result), C};
        f.insts.insert(f.insts.begin() + (long)k, t);  // operands are all defined before `in`
        return true;
      }
    }
    return false;
  }

  void run() {
    for (int round = 0; round < 16; ++round) {
      bool changed = simplify();
      changed |= cse();
      dead_code_elim(f);
      while (reorder_chains()) changed = true;
      dead_code_elim(f);
      if (!changed) break;
    }
  }
};

}  // namespace

void optimize_function(Function& f) {
  if (!f.has_body) return;
  Optimizer(f).run();
}

}  // namespace dlvm
