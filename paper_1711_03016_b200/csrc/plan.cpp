// Launch planner (see plan.h).  Create-time only; host C++.
//
// Steps:
//  1. peepholes: `subtract(1, multiply(tanh z, tanh z))` -> sech2(z)
//     (reading A12: derivative closed forms evaluated from the
//     pre-activation, cancellation-free in fp32); reduce(reduce(x, a), b)
//     with a single-use inner reduce -> one multi-axis reduction.
//  2. availability: every SSA value is an argument, a literal, inlined
//     (recomputed in registers inside each kernel that needs it) or
//     materialised (stored by the kernel that produces it).  `dot` and
//     `reduce` results are always materialised; element-wise values are
//     materialised when returned, used by a `dot`, or needed by two
//     kernels; transpose / shapeCast / slice are views (strided refs, or
//     index maps when inlined).
//  3. regions: every materialised element-wise value and every reduction is
//     a root; its region is the DAG of inlined values it needs.  Independent
//     roots over the same iteration space merge into one kernel (P:L19,
//     "fuse compatible element-wise operators to a single kernel").
//  4. a kernel reading a `dot` result at the dot's own index space becomes
//     that dot's GEMM epilogue ("Wx + b" fusion, B200 form: the
//     bias/activation run on the accumulator tile instead of padding).
//  5. schedule (program order, topological), lay out the workspace, emit
//     reduction finalizes and gradient-ready events.
#include "plan.h"

#include <algorithm>
#include <cstdlib>
#include <functional>
#include <map>
#include <set>
#include <sstream>

namespace dlvm {

bool TensorRef::contiguous() const {
  int64_t s = 1;
  for (int i = (int)shape.size() - 1; i >= 0; --i) {
    if (shape[i] != 1 && strides[i] != s) return false;
    s *= shape[i];
  }
  return nchunks == 1;
}

std::string program_signature(const EwProgram& p) {
  std::ostringstream o;
  o << "i" << (int)p.n_in << "l" << (int)p.n_lits << "|";
  for (int k = 0; k < p.n_ins; ++k)
    o << (k ? ";" : "") << (int)p.ins[k].op << "," << (int)p.ins[k].a << "," << (int)p.ins[k].b << ","
      << (int)p.ins[k].c;
  o << "|s";
  for (int k = 0; k < p.n_stores; ++k) o << (k ? "," : "") << (int)p.store_slot[k];
  o << "|r";
  for (int k = 0; k < p.n_reduces; ++k) o << (k ? "," : "") << (int)p.reduce_slot[k] << ":" << (int)p.reduce_kind[k];
  return o.str();
}

int Plan::launches() const {
  int n = 0;
  for (auto& s : steps) n += s.counted_launch() ? 1 : 0;
  return n;
}

std::string Plan::str() const {
  std::ostringstream o;
  o << "plan: " << steps.size() << " steps, " << launches() << " launches, workspace " << workspace_bytes
    << " bytes\n";
  for (size_t i = 0; i < steps.size(); ++i) o << "  [" << i << "] " << steps[i].desc << "\n";
  return o.str();
}

namespace {
void print_group(std::ostringstream& o, const EwGroup& g) {
  o << "    space [";
  for (int d = 0; d < g.ndims; ++d) o << (d ? "," : "") << g.dims[d];
  o << "] ncols " << g.ncols << " vec " << g.vec << " block " << g.bx << "x" << g.by << " rpt " << g.rpt << " grid "
    << g.gx << "x" << g.gy << "  prog " << g.sig << "\n";
  auto ref = [&](const char* what, size_t k, const IterRef& r) {
    o << "    " << what << k << ": buf " << r.buf << " +" << r.offset << " strides [";
    for (int d = 0; d < g.ndims; ++d) o << (d ? "," : "") << r.strides[d];
    o << "] st " << (int)r.st;
    if (r.nchunks != 1) o << " chunks " << r.nchunks << "x" << r.chunk_stride << (r.chunk_op == 1 ? " (product)" : r.chunk_op == 2 ? " (max)" : "");
    if (r.direct_buf >= 0) o << " direct buf " << r.direct_buf;
    o << "\n";
  };
  for (size_t k = 0; k < g.inputs.size(); ++k) ref("in", k, g.inputs[k]);
  for (size_t k = 0; k < g.stores.size(); ++k) ref("store", k, g.stores[k]);
  for (size_t k = 0; k < g.reduces.size(); ++k) ref("reduce", k, g.reduces[k]);
}
}  // namespace

std::string Plan::detail() const {
  std::ostringstream o;
  o << str() << "buffers:\n";
  for (size_t b = 0; b < bufs.size(); ++b) {
    const BufferSlot& x = bufs[b];
    static const char* kinds[] = {"input", "output", "seed", "work"};
    o << "  buf " << b << ": " << kinds[(int)x.kind] << " " << x.index << " bytes " << x.bytes << " st " << (int)x.st;
    if (x.kind == BufferSlot::Work) o << " offset " << x.offset;
    o << "\n";
  }
  for (size_t i = 0; i < steps.size(); ++i) {
    const Step& s = steps[i];
    o << "  [" << i << "] " << s.desc << "\n";
    if (s.kind == Step::EW) print_group(o, s.ew);
    if (s.kind == Step::GEMM) print_group(o, s.gemm.epi);
  }
  return o.str();
}

namespace {

std::vector<int64_t> contig_strides(const std::vector<int64_t>& shape) {
  std::vector<int64_t> st(shape.size());
  int64_t s = 1;
  for (int i = (int)shape.size() - 1; i >= 0; --i) {
    st[i] = s;
    s *= shape[i];
  }
  return st;
}
size_t stype_size(SType t) { return (size_t)st_bytes((uint8_t)t); }

[[noreturn]] void unsupported(const std::string& m) { throw Error(kStatusUnsupported, 0, 0, m); }

using Map = std::vector<int>;  // value dim -> iteration dim, or -1 (index 0)
constexpr int kGemmEpiReds = 2;  // gemm_tc.cuh kEpiReds

Map identity(int r) {
  Map m(r);
  for (int i = 0; i < r; ++i) m[i] = i;
  return m;
}
bool is_identity(const std::vector<int>& p) {
  for (size_t i = 0; i < p.size(); ++i)
    if (p[i] != (int)i) return false;
  return true;
}

// size-1 dims carry no index: canonical maps send them to -1
Map canon(Map m, const std::vector<int64_t>& shape) {
  for (size_t j = 0; j < m.size(); ++j)
    if (shape[j] == 1) m[j] = -1;
  return m;
}
bool ident_map(const Map& m, const std::vector<int64_t>& shape, int rk) {
  if ((int)m.size() != rk) return false;
  for (size_t j = 0; j < m.size(); ++j)
    if (shape[j] != 1 && m[j] != (int)j) return false;
  return true;
}

struct Home {
  int buf = -1;
  SType st = SType::F32;
  TensorRef ref;
};

struct VInfo {
  int def = -1;            // defining instruction index, -1 for arguments
  int arg = -1;            // argument index
  std::vector<int> users;  // instruction indices
  std::vector<int> outs;   // output indices returning this value
  bool mat = false;        // element-wise/view value stored by its own root
  bool inl = false;        // element-wise/view value recomputed in registers
  bool dead = false;       // fused away (inner reduce of a chain)
  bool dot_use = false;    // operand of a dot (through views)
  bool prod_use = false;   // operand of a `reduce ... by multiply` (through views)
  bool group_use = false;  // read by an element-wise kernel
  std::vector<Home> homes; // materialised copies
  int out_home = -1;       // output index this value is produced into directly
  std::vector<int> more_outs;  // further outputs returning the same stored value (extra stores, no copy)
};

struct Root {
  enum Kind { Store, Reduce, Copy, Fill } kind = Store;
  int v = -1;              // Store: value; Reduce: reduced operand x; Copy: source value
  int red = -1;            // Reduce: the (outermost) reduce result value
  uint8_t rkind = RED_ALL; // Reduce: kind in the node's iteration space
  int out = -1;            // Copy / Fill: output index
  double lit = 0;          // Fill
  std::vector<int64_t> fill_shape;
};

struct Node {
  bool is_dot = false;         // an opaque node reading materialised operands: a dot,
  bool is_prod = false;        // or (is_prod) a `reduce ... by multiply`
  int dot_inst = -1;
  std::vector<int64_t> shape;  // iteration shape
  std::vector<int> perm;       // iteration dim i <- reduced-operand dim perm[i] (reduce nodes)
  int split = -1;              // number of row dims, -1 if free
  std::vector<Root> roots;
  std::set<int> reads, writes, inl;
  std::set<int> nonident;      // values read at a non-identity index map
  std::set<int> stored;        // element-wise values stored by this group's Store roots
  int pos = 0;
  int merged_into = -1;
  int fused_epilogue = -1;     // dot: group fused as its epilogue
  bool fused = false;          // group fused into a dot
};

struct RedInfo {
  int value;
  int slot_index;
  uint8_t kind;
};

struct Planner {
  Function f;
  PlanOptions opt;
  Plan plan;
  std::vector<VInfo> vi;
  std::vector<Node> nodes;
  std::set<int> force_mat;
  std::map<int, std::pair<int, std::vector<int>>> red_root;  // outer reduce -> (x, summed axes of x)
  std::vector<int> node_of_value;
  std::vector<std::set<int>> succ;
  std::vector<int> cast_buf;

  Planner(const Function& fn, const PlanOptions& o) : f(fn), opt(o) {}

  const Type& ty(int v) const { return f.types[v]; }
  const Inst* def(int v) const { return vi[v].def >= 0 ? &f.insts[vi[v].def] : nullptr; }
  static bool is_view(const Inst* in) {
    return in && (in->op == Op::Transpose || in->op == Op::ShapeCast || in->op == Op::Slice);
  }
  static bool is_dotlike(Op op) { return op == Op::Dot || op == Op::DotSum; }
  // reductions by multiply or max: one element-wise step of their own (emit_prod)
  static bool is_prod(const Inst* in) { return in && in->op == Op::Reduce && (in->reduce_mul || in->reduce_max); }
  static bool is_ew(const Inst* in) {
    return in && (is_elementwise(in->op) || in->op == Op::Sech2 || in->op == Op::DataTypeCast);
  }
  bool produced(int v) const {
    const Inst* in = def(v);
    if (!in || vi[v].dead) return false;
    return is_dotlike(in->op) || is_prod(in) || (in->op == Op::Reduce && red_root.count(v)) || vi[v].mat;
  }
  SType natural(int v) const { return ty(v).dtype == DType::Bool ? SType::U8 : SType::F32; }

  // ---------------------------------------------------------------- checks
  void check_supported() {
    for (size_t i = 0; i < f.types.size(); ++i) {
      DType d = f.types[i].dtype;
      if (d != DType::F32 && d != DType::Bool)
        unsupported("value %" + f.names[i] + " has type " + f.types[i].str() +
                    "; the GPU path executes f32 and bool tensors");
      if (f.types[i].rank() > kPlanDims) unsupported("rank > 8 tensors are not supported");
    }
    for (auto& in : f.insts) {
      if (in.op == Op::DataTypeCast && !((in.cast_to == DType::F32 || in.cast_to == DType::Bool)))
        unsupported("dataTypeCast target");
      for (auto& o : in.ops)
        if (o.is_lit() && o.type.dtype != DType::F32 && o.type.dtype != DType::Bool)
          unsupported("literal of type " + o.type.str());
    }
  }

  // ------------------------------------------------------------- peepholes
  void peepholes() {
    // a splat literal feeding a dot is materialised by an element-wise
    // `add(lit, 0)` (stored, since it is a dot operand)
    for (size_t k = 0; k < f.insts.size(); ++k) {
      if (f.insts[k].op != Op::Dot) continue;
      for (int j = 0; j < 2; ++j) {
        if (!f.insts[k].ops[j].is_lit()) continue;
        Operand lit = f.insts[k].ops[j];
        Inst splat;
        splat.op = Op::Add;
        Operand zero;
        zero.lit = 0.0;
        zero.type = Type{{}, lit.type.dtype};
        splat.ops = {lit, zero};
        splat.rname = "splat" + std::to_string(k) + "_" + std::to_string(j);
        splat.result = f.add_value(splat.rname, lit.type);
        Operand use;
        use.value = splat.result;
        use.vname = splat.rname;
        use.type = lit.type;
        f.insts[k].ops[j] = use;
        f.insts.insert(f.insts.begin() + k, splat);
        ++k;
      }
    }
    std::vector<int> defidx(f.types.size(), -1);
    for (size_t k = 0; k < f.insts.size(); ++k) defidx[f.insts[k].result] = (int)k;
    // linear algebra fusion: add(dot(A1,B1), dot(A2,B2))
    // of single-use, same-shape products -> one DotSum (a GEMM whose K loop
    // walks every product into one accumulator); chains of adds keep growing
    // the sum, e.g. W x + U h + b -> DotSum(x, W, h, U) + b (the bias and the
    // activation then fuse into the GEMM epilogue like any other)
    {
      std::vector<int> uses(f.types.size(), 0), is_ret(f.types.size(), 0);
      for (auto& in : f.insts)
        for (auto& o : in.ops)
          if (!o.is_lit()) ++uses[o.value];
      for (auto& o : f.ret)
        if (!o.is_lit()) is_ret[o.value] = 1;
      for (auto& in : f.insts) {
        if (in.op != Op::Add || in.ops[0].is_lit() || in.ops[1].is_lit()) continue;
        if (in.ops[0].value == in.ops[1].value) continue;
        const auto& rs = f.types[in.result].shape;
        auto fusable = [&](const Operand& o) {
          const int d = defidx[o.value];
          if (d < 0) return false;
          const Op op = f.insts[d].op;
          return (op == Op::Dot || op == Op::DotSum) && uses[o.value] == 1 && !is_ret[o.value] &&
                 f.types[o.value].shape == rs;
        };
        if (!fusable(in.ops[0]) || !fusable(in.ops[1])) continue;
        const Inst& x = f.insts[defidx[in.ops[0].value]];
        const Inst& y = f.insts[defidx[in.ops[1].value]];
        if ((int)(x.ops.size() + y.ops.size()) / 2 > kPlanMaxSeg) continue;
        std::vector<Operand> ops = x.ops;
        ops.insert(ops.end(), y.ops.begin(), y.ops.end());
        --uses[in.ops[0].value];
        --uses[in.ops[1].value];
        in.op = Op::DotSum;
        in.ops = ops;
      }
    }
    for (auto& in : f.insts) {  // subtract(1, multiply(t, t)), t = tanh(z) -> sech2(z)
      if (in.op != Op::Subtract || !in.ops[0].is_lit() || in.ops[0].lit != 1.0 || in.ops[1].is_lit()) continue;
      int m = defidx[in.ops[1].value];
      if (m < 0) continue;
      const Inst& mi = f.insts[m];
      if (mi.op != Op::Multiply || mi.ops[0].is_lit() || mi.ops[1].is_lit() || mi.ops[0].value != mi.ops[1].value)
        continue;
      int t = defidx[mi.ops[0].value];
      if (t < 0 || f.insts[t].op != Op::Tanh) continue;
      const Operand z = f.insts[t].ops[0];
      if (z.is_lit() || f.types[z.value].shape != f.types[in.result].shape) continue;
      in.op = Op::Sech2;
      in.ops = {z};
    }
    dead_code_elim(f);
  }

  // ------------------------------------------------------------- analysis
  void analyse() {
    vi.assign(f.types.size(), VInfo{});
    for (int i = 0; i < f.num_args(); ++i) vi[i].arg = i;
    for (size_t k = 0; k < f.insts.size(); ++k) {
      const Inst& in = f.insts[k];
      vi[in.result].def = (int)k;
      for (auto& o : in.ops)
        if (!o.is_lit()) vi[o.value].users.push_back((int)k);
    }
    for (size_t k = 0; k < f.ret.size(); ++k)
      if (!f.ret[k].is_lit()) vi[f.ret[k].value].outs.push_back((int)k);
    for (auto& in : f.insts) {
      const bool prod = is_prod(&in);
      if (!is_dotlike(in.op) && !prod) continue;
      for (auto& o : in.ops) {
        if (o.is_lit()) continue;
        int v = o.value;
        (prod ? vi[v].prod_use : vi[v].dot_use) = true;
        while (is_view(def(v))) {
          v = def(v)->ops[0].value;
          (prod ? vi[v].prod_use : vi[v].dot_use) = true;
        }
      }
    }
  }

  void reduce_chains() {
    for (auto& in : f.insts) {
      if (in.op != Op::Reduce) continue;
      if (in.ops[0].is_lit()) unsupported("reduce of a literal");
      if (in.reduce_mul || in.reduce_max) continue;  // its own step (emit_prod), never chained into a sum
      int x = in.ops[0].value;
      auto it = red_root.find(x);
      if (it != red_root.end() && vi[x].users.size() == 1 && vi[x].outs.empty()) {
        auto [x0, ax0] = it->second;
        std::vector<int> keep;
        for (int d = 0; d < ty(x0).rank(); ++d)
          if (std::find(ax0.begin(), ax0.end(), d) == ax0.end()) keep.push_back(d);
        std::vector<int> ax = ax0;
        ax.push_back(keep[in.axis]);
        std::sort(ax.begin(), ax.end());
        red_root.erase(it);
        vi[x].dead = true;
        red_root[in.result] = {x0, ax};
      } else {
        red_root[in.result] = {x, {in.axis}};
      }
    }
  }

  // ------------------------------------------------------------ index maps
  Map bcast_map(const std::vector<int64_t>& sa, const std::vector<int64_t>& su, const Map& mu) const {
    Map ma(sa.size(), -1);
    size_t off = su.size() - sa.size();
    for (size_t j = 0; j < sa.size(); ++j) ma[j] = (sa[j] == 1) ? -1 : mu[j + off];
    return ma;
  }
  // index map through a view (result map mu -> source map)
  bool view_map(const Inst& in, const Map& mu, Map* ma) const {
    const auto& sa = ty(in.ops[0].value).shape;
    const auto& su = ty(in.result).shape;
    if (in.op == Op::Transpose) {
      ma->assign(sa.size(), -1);
      for (size_t j = 0; j < sa.size(); ++j) (*ma)[j] = mu[sa.size() - 1 - j];
      return true;
    }
    if (in.op == Op::ShapeCast) {
      std::vector<int> nu, na;
      for (size_t j = 0; j < su.size(); ++j)
        if (su[j] != 1) nu.push_back((int)j);
      for (size_t j = 0; j < sa.size(); ++j)
        if (sa[j] != 1) na.push_back((int)j);
      if (nu.size() != na.size()) return false;
      for (size_t k = 0; k < nu.size(); ++k)
        if (su[nu[k]] != sa[na[k]]) return false;
      ma->assign(sa.size(), -1);
      for (size_t k = 0; k < na.size(); ++k) (*ma)[na[k]] = mu[nu[k]];
      return true;
    }
    return false;
  }
  bool composable(const Inst& in) const {
    Map m;
    return in.op != Op::Slice && view_map(in, identity(ty(in.result).rank()), &m);
  }
  // strides of a row-major reshape of a strided tensor, when one exists:
  // old and new dims are grouped into blocks of equal element count; each
  // old block must be contiguous within itself (e.g. the rows of a padded
  // home may be split or merged, its last dim kept)
  static bool reshape_strides(const std::vector<int64_t>& os, const std::vector<int64_t>& ost,
                              const std::vector<int64_t>& ns, std::vector<int64_t>* nst) {
    std::vector<int64_t> a, as;  // old dims without unit dims
    for (size_t i = 0; i < os.size(); ++i)
      if (os[i] != 1) {
        a.push_back(os[i]);
        as.push_back(ost[i]);
      }
    nst->assign(ns.size(), 0);
    size_t oi = 0, ni = 0;
    while (ni < ns.size() && ns[ni] == 1) ++ni;
    while (oi < a.size() && ni < ns.size()) {
      int64_t np = ns[ni], op = a[oi];
      size_t nj = ni + 1, oj = oi + 1;
      while (np != op) {
        if (np < op) {
          if (nj >= ns.size()) return false;
          np *= ns[nj++];
        } else {
          if (oj >= a.size()) return false;
          op *= a[oj++];
        }
      }
      for (size_t k = oi; k + 1 < oj; ++k)
        if (as[k] != a[k + 1] * as[k + 1]) return false;
      // new dims ni..nj-1 (unit dims among them get stride 0)
      int64_t st = as[oj - 1];
      for (size_t k = nj; k-- > ni;) {
        (*nst)[k] = ns[k] == 1 ? 0 : st;
        if (ns[k] != 1) st *= ns[k];
      }
      oi = oj;
      ni = nj;
      while (ni < ns.size() && ns[ni] == 1) ++ni;
    }
    return oi == a.size() && ni == ns.size();
  }

  // strided view of a materialised source
  bool view_ref(const Inst& in, const TensorRef& src, TensorRef* out) const {
    *out = src;
    const auto& su = ty(in.result).shape;
    if (in.op == Op::Transpose) {
      std::reverse(out->shape.begin(), out->shape.end());
      std::reverse(out->strides.begin(), out->strides.end());
      return true;
    }
    if (in.op == Op::Slice) {
      out->offset += in.from * src.strides[0];
      out->shape[0] = in.upto - in.from;
      return true;
    }
    if (src.contiguous()) {
      out->shape = su;
      out->strides = contig_strides(su);
      return true;
    }
    if (in.op == Op::ShapeCast && reshape_strides(src.shape, src.strides, su, &out->strides)) {
      out->shape = su;
      return true;
    }
    Map m;
    if (!view_map(in, identity((int)su.size()), &m)) return false;
    out->shape = su;
    out->strides.assign(su.size(), 0);
    for (size_t j = 0; j < m.size(); ++j)
      if (m[j] >= 0) out->strides[m[j]] = src.strides[j];
    return true;
  }
  // a materialised shapeCast view that merges or splits dims: its copy
  // kernel iterates in the source's shape (any source layout reads at the
  // identity map) and stores into the value's unpadded home viewed in that
  // shape (row-major homes of equal size share their element order)
  // may the value's workspace homes have padded rows?  Not for reshaped
  // copies (stored in another shape's element order) nor for reductions
  // (their finalize, and a single-partial producer, write the result
  // contiguously)
  bool row_padded(int v) const {
    const Inst* in = def(v);
    return !reshape_copy(v) && !(in && in->op == Op::Reduce && red_root.count(v));
  }

  bool reshape_copy(int v) const {
    const Inst* in = def(v);
    if (!in || in->op != Op::ShapeCast || !vi[v].mat) return false;
    Map m;
    return !view_map(*in, identity(ty(v).rank()), &m);
  }

  // -------------------------------------------------------- availability
  void decide() {
    for (size_t v = 0; v < f.types.size(); ++v) {
      VInfo& x = vi[v];
      x.mat = x.inl = false;
      const Inst* in = def((int)v);
      if (!in || x.dead) continue;
      if (is_ew(in)) {
        x.mat = !x.outs.empty() || x.dot_use || x.prod_use || force_mat.count((int)v) || opt.no_fusion;
        x.inl = !x.mat;
      } else if (is_view(in)) {
        x.mat = force_mat.count((int)v) > 0;
        x.inl = !x.mat;
      }
    }
  }

  // outputs produced in place by their producer (no copy kernel)
  void alias_outputs() {
    for (auto& x : vi) {
      x.out_home = -1;
      x.more_outs.clear();
    }
    std::set<int> used;
    for (size_t k = 0; k < f.ret.size(); ++k) {
      const Operand& o = f.ret[k];
      if (o.is_lit()) continue;
      int v = o.value;
      if (used.count(v) && vi[v].out_home >= 0 && produced(v) && vi[v].mat) {
        vi[v].more_outs.push_back((int)k);  // returned again: one more store by its producer
        continue;
      }
      if (used.count(v) || vi[v].arg >= 0) continue;
      // follow single-use contiguous shapeCast views back to their producer
      std::vector<int> chain{v};
      int u = v;
      while (vi[u].inl && def(u) && def(u)->op == Op::ShapeCast) {
        int s = def(u)->ops[0].value;
        if (vi[s].users.size() != 1 || !vi[s].outs.empty() || vi[s].arg >= 0) break;
        chain.push_back(s);
        u = s;
      }
      if (!produced(u) || used.count(u)) continue;
      if (ty(u).dtype != ty(v).dtype) continue;
      for (int c : chain) {
        vi[c].out_home = (int)k;
        used.insert(c);
      }
    }
  }

  // ----------------------------------------------------------- the nodes
  bool need_iterate = false;
  void build_nodes() {
    nodes.clear();
    node_of_value.assign(f.types.size(), -1);
    for (size_t k = 0; k < f.insts.size(); ++k) {
      const Inst& in = f.insts[k];
      int v = in.result;
      if (vi[v].dead) continue;
      Node n;
      n.pos = (int)k;
      n.writes.insert(v);
      if (is_dotlike(in.op) || is_prod(&in)) {
        n.is_dot = true;
        n.is_prod = is_prod(&in);
        n.dot_inst = (int)k;
      } else if (in.op == Op::Reduce && red_root.count(v)) {
        auto [x, axes] = red_root[v];
        const auto& sx = ty(x).shape;
        int rk = (int)sx.size();
        Root r;
        r.kind = Root::Reduce;
        r.v = x;
        r.red = v;
        bool leading = true;
        for (size_t i = 0; i < axes.size(); ++i) leading &= axes[i] == (int)i;
        if ((int)axes.size() == rk) {
          n.perm = identity(rk);
          r.rkind = RED_ALL;
        } else if (leading) {
          n.perm = identity(rk);
          n.split = (int)axes.size();
          r.rkind = RED_COL;
        } else {
          for (int d = 0; d < rk; ++d)
            if (std::find(axes.begin(), axes.end(), d) == axes.end()) n.perm.push_back(d);
          n.split = (int)n.perm.size();
          for (int d : axes) n.perm.push_back(d);
          r.rkind = RED_ROW;
        }
        for (int d : n.perm) n.shape.push_back(sx[d]);
        n.roots.push_back(r);
      } else if (vi[v].mat) {
        Root r;
        r.kind = Root::Store;
        r.v = v;
        n.roots.push_back(r);
        n.shape = reshape_copy(v) ? ty(in.ops[0].value).shape : ty(v).shape;
        n.perm = identity((int)n.shape.size());
      } else {
        continue;
      }
      nodes.push_back(n);
      node_of_value[v] = (int)nodes.size() - 1;
    }
    for (size_t k = 0; k < f.ret.size(); ++k) {
      const Operand& o = f.ret[k];
      Node n;
      Root r;
      n.pos = (int)f.insts.size() + (int)k;
      if (o.is_lit()) {
        r.kind = Root::Fill;
        r.out = (int)k;
        r.lit = o.lit;
        r.fill_shape = o.type.shape;
        n.shape = o.type.shape;
      } else {
        if (vi[o.value].out_home == (int)k) continue;  // produced in place
        if (std::find(vi[o.value].more_outs.begin(), vi[o.value].more_outs.end(), (int)k) !=
            vi[o.value].more_outs.end())
          continue;  // an extra store of the producer
        r.kind = Root::Copy;
        r.v = o.value;
        r.out = (int)k;
        n.shape = ty(o.value).shape;
      }
      n.perm = identity((int)n.shape.size());
      n.roots.push_back(r);
      nodes.push_back(n);
    }
  }

  int base_of(int v) const {  // materialised value behind a chain of inlined views
    while (vi[v].inl && is_view(def(v))) v = def(v)->ops[0].value;
    return v;
  }

  void region_of(Node& n) {
    n.reads.clear();
    n.inl.clear();
    n.nonident.clear();
    n.stored.clear();
    if (n.is_dot) {
      for (auto& o : f.insts[n.dot_inst].ops)
        if (!o.is_lit()) {
          n.reads.insert(base_of(o.value));
          n.nonident.insert(base_of(o.value));
        }
      return;
    }
    const int rk = (int)n.shape.size();
    std::function<void(int, const Map&)> walk = [&](int v, const Map& m) {
      if (vi[v].arg >= 0 || !vi[v].inl) {
        n.reads.insert(v);
        if (!(ident_map(m, ty(v).shape, rk) && ty(v).shape == n.shape)) n.nonident.insert(v);
        return;
      }
      const Inst* in = def(v);
      n.inl.insert(v);
      if (is_view(in)) {
        int src = in->ops[0].value;
        Map ma;
        if (in->op != Op::Slice && view_map(*in, m, &ma)) {
          walk(src, ma);
        } else {
          if (vi[src].inl) {
            force_mat.insert(src);
            need_iterate = true;
          }
          n.reads.insert(base_of(src));
          n.nonident.insert(base_of(src));
        }
        return;
      }
      const auto& su = ty(v).shape;
      for (auto& o : in->ops)
        if (!o.is_lit()) walk(o.value, bcast_map(ty(o.value).shape, su, m));
    };
    for (auto& r : n.roots) {
      if (r.kind == Root::Fill) continue;
      if (r.kind == Root::Store) {
        n.stored.insert(r.v);
        const Inst* in = def(r.v);
        const auto& su = ty(r.v).shape;
        Map id = identity(ty(r.v).rank());
        if (is_view(in)) {  // forced view copy: reads its source through the view
          int src = in->ops[0].value;
          Map ma;
          if (reshape_copy(r.v)) {
            walk(src, identity(ty(src).rank()));
          } else if (in->op != Op::Slice && view_map(*in, id, &ma)) {
            walk(src, ma);
          } else {
            n.reads.insert(base_of(src));
            n.nonident.insert(base_of(src));
          }
          continue;
        }
        for (auto& o : in->ops)
          if (!o.is_lit()) walk(o.value, bcast_map(ty(o.value).shape, su, id));
      } else if (r.kind == Root::Reduce) {
        Map mx(ty(r.v).rank(), -1);
        for (size_t i = 0; i < n.perm.size(); ++i) mx[n.perm[i]] = (int)i;
        walk(r.v, mx);
      } else {
        walk(r.v, identity(ty(r.v).rank()));
      }
    }
  }

  // a region whose program would exceed the fixed-size EwProgram gets a value
  // in the middle of its inlined DAG materialised (splits it in two kernels)
  static constexpr int kInsBudget = kMaxIns - 8, kInBudget = kMaxIn - 2;
  bool split_oversized() {
    for (auto& n : nodes) {
      if (n.is_dot) continue;
      if ((int)n.inl.size() <= kInsBudget && (int)n.reads.size() <= kInBudget) continue;
      std::vector<int> cand;
      for (int v : n.inl)
        if (is_ew(def(v)) && !force_mat.count(v)) cand.push_back(v);
      if (cand.empty()) continue;
      std::sort(cand.begin(), cand.end(), [&](int a, int b) { return vi[a].def < vi[b].def; });
      force_mat.insert(cand[cand.size() / 2]);
      return true;
    }
    return false;
  }

  int find(int a) const {
    while (nodes[a].merged_into >= 0) a = nodes[a].merged_into;
    return a;
  }
  void build_edges() {
    std::map<int, int> writer;
    for (size_t i = 0; i < nodes.size(); ++i)
      for (int v : nodes[i].writes) writer[v] = (int)i;
    succ.assign(nodes.size(), {});
    for (size_t i = 0; i < nodes.size(); ++i)
      for (int v : nodes[i].reads) {
        auto it = writer.find(v);
        if (it != writer.end() && it->second != (int)i) succ[it->second].insert((int)i);
      }
  }
  // is there a dependency path from group `from` to group `to` (merged view)?
  // With skip_direct, the direct edges from -> to are ignored (they are
  // satisfied in registers when the two merge).
  bool reaches(int from, int to, bool skip_direct = false) const {
    from = find(from);
    to = find(to);
    std::vector<char> seen(nodes.size(), 0);
    std::vector<int> st{from};
    seen[from] = 1;
    while (!st.empty()) {
      int a = st.back();
      st.pop_back();
      for (size_t i = 0; i < nodes.size(); ++i) {
        if (find((int)i) != a) continue;
        for (int b : succ[i]) {
          int g = find(b);
          if (g == a) continue;
          if (g == to) {
            if (skip_direct && a == from) continue;
            return true;
          }
          if (!seen[g]) {
            seen[g] = 1;
            st.push_back(g);
          }
        }
      }
    }
    return false;
  }

  void merge_groups() {
    if (opt.no_fusion) return;
    for (size_t i = 0; i < nodes.size(); ++i) {
      Node& a = nodes[i];
      if (a.is_dot) continue;
      for (size_t j = 0; j < i; ++j) {
        Node& g = nodes[j];
        if (g.is_dot || g.merged_into >= 0) continue;
        if (g.shape != a.shape || g.perm != a.perm) continue;
        if (a.split >= 0 && g.split >= 0 && a.split != g.split) continue;
        if (store_count(g) + store_count(a) > kMaxStores) continue;
        {  // the merged program must fit the fixed-size EwProgram
          std::set<int> inl = g.inl, rd = g.reads;
          inl.insert(a.inl.begin(), a.inl.end());
          rd.insert(a.reads.begin(), a.reads.end());
          int nred = 0;
          for (auto& r : g.roots) nred += r.kind == Root::Reduce;
          for (auto& r : a.roots) nred += r.kind == Root::Reduce;
          if ((int)inl.size() > kInsBudget || (int)rd.size() > kInBudget || nred > kMaxReduces) continue;
        }
        if (reaches((int)i, (int)j)) continue;
        // direct dependencies are allowed when `a` only reads values that `g`
        // stores, element for element (identity map): they stay in registers
        bool direct_ok = true, direct = false;
        for (int v : a.reads) {
          bool written_by_g = false;
          for (size_t k = 0; k < nodes.size(); ++k)
            if (find((int)k) == (int)j && nodes[k].writes.count(v)) written_by_g = true;
          if (!written_by_g) continue;
          direct = true;
          if (!g.stored.count(v) || a.nonident.count(v) || !is_ew(def(v))) direct_ok = false;
        }
        if (direct && !direct_ok) continue;
        if (reaches((int)j, (int)i, direct)) continue;
        a.merged_into = (int)j;
        for (auto& r : a.roots) g.roots.push_back(r);
        g.reads.insert(a.reads.begin(), a.reads.end());
        g.writes.insert(a.writes.begin(), a.writes.end());
        g.inl.insert(a.inl.begin(), a.inl.end());
        g.nonident.insert(a.nonident.begin(), a.nonident.end());
        g.stored.insert(a.stored.begin(), a.stored.end());
        g.pos = std::max(g.pos, a.pos);
        g.split = std::max(g.split, a.split);
        break;
      }
    }
  }

  // stores a group will issue (homes are assigned later: estimate)
  int store_count(const Node& n) const {
    int c = 0;
    for (auto& r : n.roots) {
      if (r.kind == Root::Store) {
        const VInfo& x = vi[r.v];
        c += 1 + (int)x.more_outs.size() + (x.dot_use && opt.policy == Policy::BF16 ? 1 : 0);
      } else if (r.kind != Root::Reduce) {
        c += 1;
      }
    }
    return c;
  }

  // an inlined element-wise value computed by two kernels is materialised,
  // unless it is a small broadcast value (cheaper to recompute)
  bool duplicates() {
    std::map<int, std::set<int>> where;
    for (size_t i = 0; i < nodes.size(); ++i) {
      if (nodes[i].merged_into >= 0 || nodes[i].is_dot) continue;
      for (int v : nodes[i].inl) where[v].insert((int)i);
    }
    // materialise one value per round, the latest in program order (closest
    // to its consumers), so that its producers can stay inlined
    int pick = -1;
    for (auto& [v, gs] : where) {
      if (gs.size() < 2 || !is_ew(def(v)) || force_mat.count(v)) continue;
      int64_t big = 0;
      for (int g : gs) {
        int64_t n = 1;
        for (auto d : nodes[g].shape) n *= d;
        big = std::max(big, n);
      }
      if (ty(v).numel() * 16 <= big) continue;
      if (pick < 0 || vi[v].def > vi[pick].def) pick = v;
    }
    if (pick < 0) return false;
    force_mat.insert(pick);
    return true;
  }

  void fuse_epilogues() {
    if (opt.no_fusion) return;
    for (size_t d = 0; d < nodes.size(); ++d) {
      if (!nodes[d].is_dot || nodes[d].is_prod) continue;
      int dv = f.insts[nodes[d].dot_inst].result;
      for (size_t g = 0; g < nodes.size(); ++g) {
        Node& G = nodes[g];
        if (G.is_dot || G.merged_into >= 0 || G.fused || !G.reads.count(dv)) continue;
        if (G.shape != ty(dv).shape || !is_identity(G.perm) || !(G.split < 0 || G.split == 1)) break;
        bool via_view = false;
        for (int v : G.inl)
          if (is_view(def(v)) && def(v)->ops[0].value == dv) via_view = true;
        if (via_view) break;
        int n_red = 0;  // the GEMM epilogue has smem for kGemmEpiReds reductions
        for (auto& r : G.roots) n_red += r.kind == Root::Reduce;
        if (n_red > kGemmEpiReds) break;
        bool ok = true;
        for (int v : G.reads) {
          if (v == dv) continue;
          int p = node_of_value[v];
          if (p < 0 || find(p) == (int)g) continue;  // argument, or stored by G itself
          if (find(p) == (int)d || reaches((int)d, p)) ok = false;
        }
        if (ok) {
          nodes[d].fused_epilogue = (int)g;
          G.fused = true;
        }
        break;
      }
    }
  }

  // ----------------------------------------------------------- buffers
  int add_buf(BufferSlot::Kind k, int index, size_t bytes, SType st) {
    BufferSlot b;
    b.kind = k;
    b.index = index;
    b.bytes = bytes;
    b.st = st;
    if (k == BufferSlot::Work) {
      plan.workspace_bytes = (plan.workspace_bytes + 255) / 256 * 256;
      b.offset = plan.workspace_bytes;
      plan.workspace_bytes += bytes;
    }
    plan.bufs.push_back(b);
    return (int)plan.bufs.size() - 1;
  }
  Home make_home(int buf, int v, SType st, int64_t ld = 0) {
    Home h;
    h.buf = buf;
    h.st = st;
    h.ref.buf = buf;
    h.ref.shape = ty(v).shape;
    h.ref.strides = contig_strides(ty(v).shape);
    if (ld > 0) {  // padded row stride for the last dim
      int r = (int)h.ref.shape.size();
      int64_t s = ld;
      h.ref.strides[r - 1] = 1;
      for (int i = r - 2; i >= 0; --i) {
        h.ref.strides[i] = s;
        s *= h.ref.shape[i];
      }
    }
    h.ref.st = st;
    return h;
  }
  // Workspace tensors of rank >= 2 get their rows padded to 64 elements: a TMA
  // box row (128 B) then never straddles two L2 lines (a 1000-element row
  // costs ~35-60% GEMM throughput, tools/gemm_probe.py).
  static int64_t padded_ld(const Type& t) {
    if (t.rank() < 2) return 0;
    int64_t c = t.shape.back();
    if (c % 64 == 0 || c < 64) return 0;
    return (c + 63) / 64 * 64;
  }
  // the most output rows of any dot reading value v (through views)
  int64_t max_dot_rows(int v) const {
    int64_t m = 0;
    for (auto& in : f.insts) {
      if (!is_dotlike(in.op)) continue;
      for (auto& o : in.ops)
        if (!o.is_lit() && base_of(o.value) == v) m = std::max(m, ty(in.result).shape[0]);
    }
    return m;
  }
  size_t padded_bytes(const Type& t, SType st) const {
    int64_t ld = padded_ld(t);
    int64_t n = ld ? t.numel() / t.shape.back() * ld : t.numel();
    return (size_t)n * stype_size(st);
  }
  int output_buf(int k) const {
    for (size_t b = 0; b < plan.bufs.size(); ++b)
      if (plan.bufs[b].kind == BufferSlot::Output && plan.bufs[b].index == k) return (int)b;
    return -1;
  }

  void assign_homes() {
    plan.bufs.clear();
    plan.workspace_bytes = 0;
    for (auto& x : vi) {  // (re-planning after force_unaddressable_operands)
      x.homes.clear();
      x.group_use = false;
    }
    // group_use: read by a (non-dot) kernel, through views
    for (auto& n : nodes) {  // reads by another kernel (values a group stores itself stay in registers)
      if (n.is_dot || n.merged_into >= 0) continue;
      for (int v : n.reads)
        if (!n.stored.count(v)) vi[v].group_use = true;
    }
    for (int i = 0; i < f.num_args(); ++i) {
      bool seed = plan.seed_is_input && i == f.num_args() - 1;
      int b = add_buf(seed ? BufferSlot::Seed : BufferSlot::Input, seed ? 0 : i,
                      ty(i).numel() * stype_size(natural(i)), natural(i));
      vi[i].homes.push_back(make_home(b, i, natural(i)));
    }
    for (size_t k = 0; k < f.ret.size(); ++k) {
      SType st = f.results[k].dtype == DType::Bool ? SType::U8 : SType::F32;
      add_buf(BufferSlot::Output, (int)k, f.results[k].numel() * stype_size(st), st);
    }
    std::map<int, int> fused_dot_group;  // dot value -> fused group node
    for (auto& n : nodes)
      if (n.is_dot && n.fused_epilogue >= 0) fused_dot_group[f.insts[n.dot_inst].result] = n.fused_epilogue;
    for (size_t v = 0; v < f.types.size(); ++v) {
      VInfo& x = vi[v];
      if (!produced((int)v)) continue;
      bool is_dot = is_dotlike(def((int)v)->op);
      bool others_read = false;
      if (is_dot && fused_dot_group.count((int)v)) {
        int g = fused_dot_group[(int)v];
        for (size_t i = 0; i < nodes.size(); ++i)
          if (!nodes[i].is_dot && nodes[i].merged_into < 0 && (int)i != g && nodes[i].reads.count((int)v))
            others_read = true;
      } else {
        others_read = x.group_use;
      }
      bool need32 = others_read || !x.outs.empty() || x.out_home >= 0 || x.prod_use ||
                    (x.dot_use && opt.policy == Policy::F32);
      if (x.out_home >= 0) {
        x.homes.push_back(make_home(output_buf(x.out_home), (int)v,
                                    ty(v).dtype == DType::Bool ? SType::U8 : SType::F32));
        for (int k : x.more_outs)
          x.homes.push_back(make_home(output_buf(k), (int)v, ty(v).dtype == DType::Bool ? SType::U8 : SType::F32));
      } else if (need32) {
        const bool pad = row_padded((int)v);
        int b = add_buf(BufferSlot::Work, -1, pad ? padded_bytes(ty(v), natural((int)v)) : ty(v).numel() * stype_size(natural((int)v)),
                        natural((int)v));
        x.homes.push_back(make_home(b, (int)v, natural((int)v), pad ? padded_ld(ty(v)) : 0));
      }
      if (x.dot_use && opt.policy == Policy::BF16) {
        const bool pad = row_padded((int)v);
        int b = add_buf(BufferSlot::Work, -1, pad ? padded_bytes(ty(v), SType::BF16) : ty(v).numel() * 2, SType::BF16);
        x.homes.push_back(make_home(b, (int)v, SType::BF16, pad ? padded_ld(ty(v)) : 0));
      }
      if (x.homes.empty() && !(is_dot && fused_dot_group.count((int)v))) {
        int b = add_buf(BufferSlot::Work, -1, ty(v).numel() * stype_size(natural((int)v)), natural((int)v));
        x.homes.push_back(make_home(b, (int)v, natural((int)v)));
      }
    }
    cast_buf.assign(f.num_args(), -1);
    // an f32 argument may be passed as bf16 (its values are then exactly the
    // f32 widening of the bf16 elements): every consumer reads the storage
    // type at run time, except an fp32-policy SIMT dot (both operands f32)
    plan.input_bf16_ok.assign(f.num_args(), 0);
    for (int i = 0; i < f.num_args(); ++i)
      plan.input_bf16_ok[i] = ty(i).dtype == DType::F32 && (opt.policy == Policy::BF16 || !vi[i].dot_use);
    // ... or as bool bytes (value 1.0 where nonzero, else 0.0: exact for 0/1
    // data such as one-hot targets), unless a dot reads it (the bf16 cast /
    // pack of dot operands and fp32 SIMT operands read f32 or bf16)
    plan.input_u8_ok.assign(f.num_args(), 0);
    for (int i = 0; i < f.num_args(); ++i) plan.input_u8_ok[i] = ty(i).dtype == DType::F32 && !vi[i].dot_use;
    if (opt.policy == Policy::BF16) {
      for (int i = 0; i < f.num_args(); ++i) {
        if (!vi[i].dot_use || ty(i).dtype != DType::F32) continue;
        // row-padded copy (a pack launch every run) only where the dots
        // reading the argument are large enough to repay it: c4's N=1000
        // GEMM 0.754 -> 0.474 ms padded, while c3's (1024 rows) pays ~12 us
        // per step for the pack
        const int64_t ld = max_dot_rows(i) >= 8192 ? padded_ld(ty(i)) : 0;
        int b = add_buf(BufferSlot::Work, -1, ld ? padded_bytes(ty(i), SType::BF16) : ty(i).numel() * 2, SType::BF16);
        plan.bufs[b].cast_of = i;
        plan.bufs[b].cast_ld = ld;
        cast_buf[i] = b;
        vi[i].homes.push_back(make_home(b, i, SType::BF16, ld));
      }
    }
  }

  // materialised ref of value v (through views), preferring bf16 or not
  bool ref_of(int v, bool want_bf16, TensorRef* out) {
    const Inst* in = def(v);
    if (vi[v].inl && is_view(in)) {
      TensorRef src;
      if (!ref_of(in->ops[0].value, want_bf16, &src)) return false;
      return view_ref(*in, src, out);
    }
    const auto& hs = vi[v].homes;
    if (hs.empty()) return false;
    const Home* pick = &hs[0];
    for (auto& h : hs)
      if ((h.st == SType::BF16) == want_bf16) {
        pick = &h;
        break;
      }
    *out = pick->ref;
    return true;
  }

  // ----------------------------------------------------- program building
  struct ProgBuilder {
    Planner& P;
    int acc_value = -1;
    std::set<int> stored;            // element-wise values this group stores (computed in registers)
    std::vector<int64_t> shape;      // iteration shape
    std::map<std::pair<int, Map>, int> memo;
    std::vector<float> lits;
    std::vector<EwIns> ins;
    std::vector<std::array<int, 3>> raw;
    std::vector<IterRef> inputs;
    explicit ProgBuilder(Planner& p) : P(p) {}

    int lit(float v) {
      for (size_t i = 0; i < lits.size(); ++i)
        if (lits[i] == v) return 100 + (int)i;
      if ((int)lits.size() >= kMaxLits) unsupported("too many literals in one fused kernel");
      lits.push_back(v);
      return 100 + (int)lits.size() - 1;
    }
    int input(const TensorRef& r, const Map& m) {
      IterRef it;
      it.buf = r.buf;
      it.offset = r.offset;
      it.nchunks = r.nchunks;
      it.chunk_stride = r.chunk_stride;
      it.st = r.st;
      for (size_t j = 0; j < m.size(); ++j)
        if (m[j] >= 0) it.strides[m[j]] += r.strides[j];
      for (size_t i = 0; i < inputs.size(); ++i) {
        const IterRef& o = inputs[i];
        bool same = o.buf == it.buf && o.offset == it.offset && o.st == it.st && o.nchunks == it.nchunks;
        for (int d = 0; d < kPlanDims && same; ++d) same = o.strides[d] == it.strides[d];
        if (same) return (int)i;
      }
      if ((int)inputs.size() >= kMaxIn) unsupported("too many inputs in one fused kernel");
      inputs.push_back(it);
      return (int)inputs.size() - 1;
    }
    int emit(uint8_t op, int a, int b, int c) {
      // identities the AD emits to broadcast (multiply by a splat 1, add a
      // splat 0): broadcasting is done by the index maps, so they are exact no-ops
      auto is_lit = [&](int s, float x) { return s >= 100 && s < 200 && lits[s - 100] == x; };
      if (op == VM_MUL && is_lit(b, 1.0f)) return a;
      if (op == VM_MUL && is_lit(a, 1.0f)) return b;
      if (op == VM_ADD && is_lit(b, 0.0f) && !is_lit(a, 0.0f) && a >= 200) return a;
      // common subexpressions (the AD emits g*r twice for multiply(r, r))
      for (size_t k = 0; k < ins.size(); ++k)
        if (ins[k].op == op && raw[k][0] == a && raw[k][1] == b && raw[k][2] == c) return 200 + (int)k;
      if ((int)ins.size() >= kMaxIns) unsupported("fused kernel program too long");
      ins.push_back(EwIns{op, 0, 0, 0});
      raw.push_back({a, b, c});
      return 200 + (int)ins.size() - 1;
    }
    int operand(const Operand& o, const std::vector<int64_t>& su, const Map& mu) {
      if (o.is_lit()) return lit((float)o.lit);
      return node(o.value, P.bcast_map(P.ty(o.value).shape, su, mu));
    }
    int node(int v, const Map& m0) {
      const Map m = canon(m0, P.ty(v).shape);
      auto key = std::make_pair(v, m);
      auto it = memo.find(key);
      if (it != memo.end()) return it->second;
      int s = compute(v, m, false);
      memo[key] = s;
      return s;
    }
    // force: compute a root's own value even though it is materialised
    int compute(int v, const Map& m, bool force) {
      const Inst* in = P.def(v);
      const VInfo& x = P.vi[v];
      if (!force && stored.count(v) && ident_map(m, P.ty(v).shape, (int)shape.size()) && P.ty(v).shape == shape &&
          is_ew(in))
        force = true;
      bool inline_it = in && x.arg < 0 && (x.inl || force);
      if (inline_it && is_view(in)) {
        int src = in->ops[0].value;
        Map ma;
        // through the view to an inlined source, or to a value this group
        // stores (computed in registers: merge_groups lets a group read its
        // own stores only at the identity map, so a load would race the store)
        if ((P.vi[src].inl || stored.count(src)) && P.view_map(*in, m, &ma)) return node(src, ma);
        TensorRef sr, r;
        if (!P.ref_of(src, false, &sr) || !P.view_ref(*in, sr, &r))
          unsupported("cannot address view %" + P.f.names[v]);
        return input(r, m);
      }
      if (inline_it && is_ew(in)) {
        const auto& su = P.ty(v).shape;
        uint8_t op;
        switch (in->op) {
          case Op::Negate: op = VM_NEG; break;
          case Op::Tanh: op = VM_TANH; break;
          case Op::Exp: op = VM_EXP; break;
          case Op::Log: op = VM_LOG; break;
          case Op::Sqrt: op = VM_SQRT; break;
          case Op::Abs: op = VM_ABS; break;
          case Op::Sign: op = VM_SIGN; break;
          case Op::Add: op = VM_ADD; break;
          case Op::Subtract: op = VM_SUB; break;
          case Op::Multiply: op = VM_MUL; break;
          case Op::Divide: op = VM_DIV; break;
          case Op::Power: op = VM_POW; break;
          case Op::Lt: op = VM_LT; break;
          case Op::Le: op = VM_LE; break;
          case Op::Gt: op = VM_GT; break;
          case Op::Ge: op = VM_GE; break;
          case Op::Eq: op = VM_EQ; break;
          case Op::Ne: op = VM_NE; break;
          case Op::Select: op = VM_SELECT; break;
          case Op::Sech2: op = VM_SECH2; break;
          case Op::DataTypeCast:
            op = (P.ty(v).dtype == DType::Bool && in->ops[0].type.dtype != DType::Bool) ? VM_TOBOOL : VM_COPY;
            break;
          default:
            unsupported(std::string("op ") + op_name(in->op) + " in a fused kernel");
        }
        // FMA contraction: add(multiply(a, b), c) / subtract(multiply(a, b), c)
        // with a single-use inlined multiply (reading A13)
        if (op == VM_ADD || op == VM_SUB) {
          for (int side = 0; side < 2; ++side) {
            const Operand& mo = in->ops[side];
            if (op == VM_SUB && side == 1) break;
            if (mo.is_lit() || !fusable_mul(mo.value)) continue;
            const Inst* mi = P.def(mo.value);
            Map mm = P.bcast_map(P.ty(mo.value).shape, su, m);
            const auto& sm = P.ty(mo.value).shape;
            int a = operand(mi->ops[0], sm, mm);
            int b = operand(mi->ops[1], sm, mm);
            int c = operand(in->ops[1 - side], su, m);
            if (op == VM_SUB) c = emit(VM_NEG, c, 0, 0);
            return emit(VM_FMA, a, b, c);
          }
        }
        int a = operand(in->ops[0], su, m);
        int b = in->ops.size() > 1 ? operand(in->ops[1], su, m) : 0;
        int c = in->ops.size() > 2 ? operand(in->ops[2], su, m) : 0;
        return emit(op, a, b, c);
      }
      TensorRef r;
      if (!P.ref_of(v, false, &r)) unsupported("value %" + P.f.names[v] + " is not addressable");
      return input(r, m);
    }
    bool fusable_mul(int v) const {
      const Inst* mi = P.def(v);
      const VInfo& x = P.vi[v];
      return mi && mi->op == Op::Multiply && x.inl && x.users.size() == 1 && x.outs.empty() && !stored.count(v);
    }
    uint8_t fix(int s) const {
      if (s >= 200) return (uint8_t)(inputs.size() + lits.size() + (s - 200));
      if (s >= 100) return (uint8_t)(inputs.size() + (s - 100));
      return (uint8_t)s;
    }
  };

  IterRef store_ref(const TensorRef& r, const Map& m) const {
    IterRef it;
    it.buf = r.buf;
    it.offset = r.offset;
    it.st = r.st;
    for (size_t j = 0; j < m.size(); ++j)
      if (m[j] >= 0) it.strides[m[j]] += r.strides[j];
    return it;
  }

  // program + refs of a group; acc_value >= 0 binds that dot value to slot 0
  void build_group(const Node& n, EwGroup& g, int acc_value, std::vector<RedInfo>* reds) {
    ProgBuilder pb(*this);
    int rk = (int)n.shape.size();
    pb.stored = n.stored;
    pb.shape = n.shape;
    if (acc_value >= 0) {
      IterRef acc;
      acc.buf = -2;
      pb.inputs.push_back(acc);
      pb.memo[{acc_value, canon(identity(2), ty(acc_value).shape)}] = 0;
    }
    std::vector<int> store_slots, red_slots;
    std::vector<uint8_t> red_kinds;
    std::vector<IterRef> stores;
    for (auto& r : n.roots) {
      if (r.kind == Root::Fill) {
        TensorRef out;
        out.buf = output_buf(r.out);
        out.shape = r.fill_shape;
        out.strides = contig_strides(r.fill_shape);
        out.st = plan.bufs[out.buf].st;
        store_slots.push_back(pb.lit((float)r.lit));
        stores.push_back(store_ref(out, identity(rk)));
        continue;
      }
      if (r.kind == Root::Reduce) {
        Map mx(ty(r.v).rank(), -1);
        for (size_t i = 0; i < n.perm.size(); ++i) mx[n.perm[i]] = (int)i;
        red_slots.push_back(pb.node(r.v, mx));
        red_kinds.push_back(r.rkind);
        reds->push_back(RedInfo{r.red, (int)red_slots.size() - 1, r.rkind});
        continue;
      }
      int v = r.v;
      if (r.kind == Root::Copy) {
        int s = pb.node(v, identity(ty(v).rank()));
        TensorRef out;
        out.buf = output_buf(r.out);
        out.shape = ty(v).shape;
        out.strides = contig_strides(out.shape);
        out.st = plan.bufs[out.buf].st;
        store_slots.push_back(s);
        stores.push_back(store_ref(out, identity(rk)));
        continue;
      }
      if (reshape_copy(v)) {  // iterate in the source's shape (see reshape_copy)
        const int src = def(v)->ops[0].value;
        const int s = pb.node(src, identity(ty(src).rank()));
        for (auto& h : vi[v].homes) {
          TensorRef hr = h.ref;
          if (!hr.contiguous()) unsupported("padded home of a reshaped copy");
          hr.shape = ty(src).shape;
          hr.strides = contig_strides(hr.shape);
          store_slots.push_back(s);
          IterRef st = store_ref(hr, identity(rk));
          st.st = h.st;
          stores.push_back(st);
        }
        continue;
      }
      int s;
      auto key = std::make_pair(v, canon(identity(ty(v).rank()), ty(v).shape));
      if (pb.memo.count(key))
        s = pb.memo[key];
      else {
        s = pb.compute(v, identity(ty(v).rank()), true);
        pb.memo[key] = s;
      }
      for (auto& h : vi[v].homes) {
        store_slots.push_back(s);
        IterRef st = store_ref(h.ref, identity(rk));
        st.st = h.st;
        stores.push_back(st);
      }
    }
    EwProgram& p = g.prog;
    p.n_in = (uint8_t)pb.inputs.size();
    p.n_lits = (uint8_t)pb.lits.size();
    p.n_ins = (uint8_t)pb.ins.size();
    for (size_t k = 0; k < pb.ins.size(); ++k) {
      p.ins[k] = pb.ins[k];
      p.ins[k].a = pb.fix(pb.raw[k][0]);
      p.ins[k].b = pb.fix(pb.raw[k][1]);
      p.ins[k].c = pb.fix(pb.raw[k][2]);
    }
    for (size_t k = 0; k < pb.lits.size(); ++k) p.lits[k] = pb.lits[k];
    if (store_slots.size() > (size_t)kMaxStores) unsupported("too many stores in one fused kernel");
    if (red_slots.size() > (size_t)kMaxReduces) unsupported("too many reductions in one fused kernel");
    p.n_stores = (uint8_t)store_slots.size();
    p.n_reduces = (uint8_t)red_slots.size();
    for (size_t k = 0; k < store_slots.size(); ++k) p.store_slot[k] = pb.fix(store_slots[k]);
    for (size_t k = 0; k < red_slots.size(); ++k) {
      p.reduce_slot[k] = pb.fix(red_slots[k]);
      p.reduce_kind[k] = red_kinds[k];
    }
    g.inputs = pb.inputs;
    g.stores = stores;
    g.reduces.assign(red_slots.size(), IterRef{});
  }

  // collapse the iteration space to <= kMaxIterDims dims: row dims + one column dim
  void collapse(EwGroup& g, std::vector<int64_t> dims, int split) {
    int r = (int)dims.size();
    std::vector<std::vector<int64_t>> in_s(g.inputs.size()), st_s(g.stores.size());
    for (size_t i = 0; i < g.inputs.size(); ++i) in_s[i].assign(g.inputs[i].strides, g.inputs[i].strides + r);
    for (size_t i = 0; i < g.stores.size(); ++i) st_s[i].assign(g.stores[i].strides, g.stores[i].strides + r);
    std::vector<std::vector<int64_t>*> refs;
    for (auto& v : in_s) refs.push_back(&v);
    for (auto& v : st_s) refs.push_back(&v);
    std::vector<int> part(r);  // 0 = row, 1 = column
    for (int i = 0; i < r; ++i) part[i] = split < 0 ? 0 : (i < split ? 0 : 1);
    auto erase = [&](int i) {
      dims.erase(dims.begin() + i);
      part.erase(part.begin() + i);
      for (auto* s : refs) s->erase(s->begin() + i);
    };
    for (int i = r - 1; i >= 0; --i)  // unit dims carry no data
      if (dims[i] == 1 && dims.size() > 1) erase(i);
    for (int i = (int)dims.size() - 2; i >= 0; --i) {
      if (part[i] != part[i + 1]) continue;
      bool ok = true;
      for (auto* s : refs) ok &= (*s)[i] == (*s)[i + 1] * dims[i + 1];
      if (!ok) continue;
      dims[i] *= dims[i + 1];
      for (auto* s : refs) (*s)[i] = (*s)[i + 1];
      erase(i + 1);
    }
    if (dims.empty() || (dims.size() == 1 && dims[0] == 1)) {
      dims = {1};
      part = {1};
      for (auto* s : refs) s->assign(1, 0);
    }
    int n_col = 0;
    for (int p : part) n_col += p;
    if (split < 0) {  // free split: the last dim is the column dim
      n_col = 1;
    } else if (n_col == 0) {  // every dim is a row dim: append a unit column
      dims.push_back(1);
      for (auto* s : refs) s->push_back(0);
      n_col = 1;
    }
    if ((int)dims.size() > kMaxIterDims) unsupported("iteration space does not collapse to " + std::to_string(kMaxIterDims) + " dims");
    g.ndims = (int)dims.size();
    g.ncols = n_col;
    for (int d = 0; d < kMaxIterDims; ++d) g.dims[d] = d < g.ndims ? dims[d] : 1;
    for (size_t i = 0; i < g.inputs.size(); ++i)
      for (int d = 0; d < kPlanDims; ++d) g.inputs[i].strides[d] = d < g.ndims ? in_s[i][d] : 0;
    for (size_t i = 0; i < g.stores.size(); ++i)
      for (int d = 0; d < kPlanDims; ++d) g.stores[i].strides[d] = d < g.ndims ? st_s[i][d] : 0;
  }

  // A long 1-D iteration space (every operand contiguous or a scalar; only
  // full reductions) is viewed as [n/W, W] rows so the 2-D kernel streams
  // several rows per thread (the 1-D form gives each thread one vector)
  static void rows_of_long_1d(EwGroup& g) {
    if (g.ndims != 1 || g.ncols != 1 || g.dims[0] < (1 << 20)) return;
    for (int q = 0; q < g.prog.n_reduces; ++q)
      if (g.prog.reduce_kind[q] != RED_ALL) return;
    const int64_t n = g.dims[0];
    int64_t W = 0;
    for (int64_t w : {4096, 2048, 1024})
      if (n % w == 0) {
        W = w;
        break;
      }
    if (!W) return;
    auto ok = [](const IterRef& r) { return r.buf == -2 || r.strides[0] == 0 || r.strides[0] == 1; };
    for (auto& r : g.inputs) if (!ok(r)) return;
    for (auto& r : g.stores) if (!ok(r)) return;
    auto split = [&](IterRef& r) {
      const int64_t st = r.strides[0];
      r.strides[0] = st * W;
      r.strides[1] = st;
    };
    for (auto& r : g.inputs) split(r);
    for (auto& r : g.stores) split(r);
    g.ndims = 2;
    g.dims[0] = n / W;
    g.dims[1] = W;
  }

  static void ew_launch(EwGroup& g) {
    int64_t C = 1, R = 1;
    for (int d = 0; d < g.ndims; ++d) (d < g.ndims - g.ncols ? R : C) *= g.dims[d];
    bool v4 = C % 4 == 0 && g.ncols == 1;
    auto ok4 = [&](const IterRef& r) {
      if (r.buf == -2) return true;
      int64_t cs = r.strides[g.ndims - 1];
      if (r.nchunks != 1 && (cs != 1 || r.chunk_stride % 4)) return false;
      if (cs == 0) return true;
      if (cs != 1 || r.offset % 4) return false;
      for (int d = 0; d < g.ndims - 1; ++d)
        if (r.strides[d] % 4) return false;
      return true;
    };
    for (auto& r : g.inputs) v4 &= ok4(r);
    for (auto& r : g.stores) v4 &= ok4(r);
    g.vec = v4 ? 4 : 1;
    int64_t cols = (C + g.vec - 1) / g.vec;
    int bx = 32;
    // column threads per CTA: at most 64 (by = 4 rows per step), measured on
    // c2 (GB/s fwd / fwd+adj): bx 256 6288 / 5803, 128 6255 / 5799, 64 6293 /
    // 5857, 32 6255 / 5835.  DLVM_EW_BX overrides.
    static const int bx_max = [] {
      const char* e = std::getenv("DLVM_EW_BX");
      return e ? std::atoi(e) : 64;
    }();
    while (bx < bx_max && bx < cols) bx *= 2;
    g.bx = bx;
    g.by = 256 / bx;
    g.gx = (cols + bx - 1) / bx;
    // rows per thread cap: 64, or 128 for programs with column sums (fewer
    // CTAs and partial rows; measured on c2, GB/s fwd / fwd+adj: cap 64
    // 6150 / 5840, 128 6117 / 5962, 256 5963 / 5955, 32 6168 / 5629).
    // DLVM_EW_RPT overrides.
    bool colsum = false;
    for (int q = 0; q < g.prog.n_reduces; ++q) colsum |= g.prog.reduce_kind[q] == RED_COL;
    static const int rpt_env = [] {
      const char* e = std::getenv("DLVM_EW_RPT");
      return e ? std::atoi(e) : 0;
    }();
    const int rpt_max = rpt_env > 0 ? rpt_env : (colsum ? 128 : 64);
    static const int ctas_per_sm = [] {  // DLVM_EW_CPS: target CTAs per SM of the row grid
      const char* e = std::getenv("DLVM_EW_CPS");
      return e ? std::atoi(e) : 8;
    }();
    int64_t want_gy = std::max<int64_t>(1, (148 * (int64_t)ctas_per_sm) / g.gx);
    int64_t rpt = (R + (int64_t)g.by * want_gy - 1) / ((int64_t)g.by * want_gy);
    g.rpt = (int)std::min<int64_t>(rpt_max, std::max<int64_t>(1, rpt));
    g.gy = (R + (int64_t)g.by * g.rpt - 1) / ((int64_t)g.by * g.rpt);
    if (g.gy > 65535) {  // tall, thin spaces: more rows per thread keep the grid's y extent legal
      g.rpt = (int)((R + (int64_t)g.by * 65535 - 1) / ((int64_t)g.by * 65535));
      g.gy = (R + (int64_t)g.by * g.rpt - 1) / ((int64_t)g.by * g.rpt);
    }
  }

  // ------------------------------------------------------------ schedule
  int rep_of(int i) const {
    i = find(i);
    if (nodes[i].fused)
      for (size_t d = 0; d < nodes.size(); ++d)
        if (nodes[d].is_dot && nodes[d].fused_epilogue == i) return (int)d;
    return i;
  }
  std::vector<int> schedule() {
    std::vector<int> reps;
    for (size_t i = 0; i < nodes.size(); ++i)
      if (nodes[i].merged_into < 0 && !nodes[i].fused) reps.push_back((int)i);
    std::map<int, std::set<int>> preds;
    for (int a : reps) preds[a];
    for (size_t i = 0; i < nodes.size(); ++i)
      for (int b : succ[i]) {
        int ga = rep_of((int)i), gb = rep_of(b);
        if (ga != gb) preds[gb].insert(ga);
      }
    auto pos = [&](int a) {
      int p = nodes[a].pos;
      if (nodes[a].is_dot && nodes[a].fused_epilogue >= 0) p = std::max(p, nodes[nodes[a].fused_epilogue].pos);
      return p;
    };
    std::vector<int> order;
    std::set<int> done;
    while (order.size() < reps.size()) {
      int best = -1;
      for (int a : reps) {
        if (done.count(a)) continue;
        bool ready = true;
        for (int p : preds[a]) ready &= done.count(p) > 0;
        if (ready && (best < 0 || pos(a) < pos(best))) best = a;
      }
      if (best < 0) throw Error(kStatusRuntime, 0, 0, "planner: dependency cycle");
      order.push_back(best);
      done.insert(best);
    }
    return order;
  }

  // --------------------------------------------------------------- emit
  // The reductions of one producer share ONE finalize launch (blockIdx.y
  // selects the reduction, dims[q] is its length n_out, its stores are the
  // ones whose store_slot names input q).  The kernel's summation order
  // depends only on n_out, so every reduction is summed exactly as a launch of
  // its own would (kept outputs stay bit-equal to dlvm_fn_run, reading A20).
  void finalize_reds(const std::vector<RedInfo>& reds, int step_index, int64_t gx, int64_t gy, int64_t R,
                     int64_t C, const std::string& who) {
    EwGroup fg;
    std::string names, shape;
    auto flush = [&]() {
      if (fg.inputs.empty()) return;
      fg.prog.n_in = (uint8_t)fg.inputs.size();
      fg.prog.n_stores = (uint8_t)fg.stores.size();
      ew_launch(fg);
      fg.sig = program_signature(fg.prog);
      fg.finalize = true;
      Step s;
      s.kind = Step::EW;
      s.ew = fg;
      s.desc = "finalize " + names + " (" + shape + ") of " + who +
               (fg.direct_buf >= 0 ? " [only when the output is bound as bf16; else written by the producer]" : "");
      s.ew.desc = s.desc;
      plan.steps.push_back(s);
      fg = EwGroup();
      names.clear();
      shape.clear();
    };
    for (auto& ri : reds) {
      int64_t n_out = ri.kind == RED_COL ? C : ri.kind == RED_ROW ? R : 1;
      int64_t nch = ri.kind == RED_COL ? gy : ri.kind == RED_ROW ? gx : gx * gy;
      Step& prod = plan.steps[step_index];
      EwGroup& pg = prod.kind == Step::GEMM ? prod.gemm.epi : prod.ew;
      const auto& homes = vi[ri.value].homes;
      // one partial: its layout is the value's own [n_out] row, so the
      // producer writes an f32 home directly and the finalize is skipped
      const int direct = nch == 1 && homes.size() == 1 && homes[0].st == SType::F32 ? homes[0].buf : -1;
      int pbuf = add_buf(BufferSlot::Work, -1, (size_t)(n_out * nch) * 4, SType::F32);
      pg.reduces[ri.slot_index].buf = pbuf;
      pg.reduces[ri.slot_index].direct_buf = direct;
      // a skippable finalize keeps a launch of its own; others merge while
      // n_out matches and the input/store tables have room
      const bool merge = !fg.inputs.empty() && direct < 0 && fg.direct_buf < 0 &&
                         (int)fg.inputs.size() < kMaxIterDims && fg.stores.size() + homes.size() <= (size_t)kMaxStores;
      if (!merge) flush();
      fg.ndims = 1;
      fg.dims[fg.inputs.size()] = n_out;
      if (fg.inputs.empty()) fg.direct_buf = direct;
      IterRef in;
      in.buf = pbuf;
      in.nchunks = (int)nch;
      if (ri.kind == RED_COL) {
        in.strides[0] = 1;
        in.chunk_stride = C;
      } else if (ri.kind == RED_ROW) {
        in.strides[0] = gx;
        in.chunk_stride = 1;
      } else {
        in.chunk_stride = 1;
      }
      const uint8_t q = (uint8_t)fg.inputs.size();
      fg.inputs.push_back(in);
      for (auto& h : homes) {
        if (!h.ref.contiguous())  // the partial layout is the value's row-major order
          throw Error(kStatusRuntime, 0, 0, "planner: reduction %" + f.names[ri.value] + " has a strided home");
        IterRef o;
        o.buf = h.buf;
        o.st = h.st;
        o.strides[0] = 1;
        fg.prog.store_slot[fg.stores.size()] = q;
        fg.stores.push_back(o);
      }
      names += (names.empty() ? "%" : ", %") + f.names[ri.value];
      shape += (shape.empty() ? "" : ", ") + std::to_string(nch) + " partials x " + std::to_string(n_out);
      if (direct >= 0) flush();
    }
    flush();
  }

  void emit_steps(const std::vector<int>& order) {
    plan.steps.clear();
    for (int i = 0; i < f.num_args(); ++i) {
      if (cast_buf[i] < 0) continue;
      Step s;
      s.kind = Step::CAST;
      s.cast.input = i;
      s.cast.dst_buf = cast_buf[i];
      s.cast.numel = ty(i).numel();
      s.cast.cols = ty(i).rank() ? ty(i).shape.back() : 1;
      s.cast.ld = plan.bufs[cast_buf[i]].cast_ld;
      s.desc = s.cast.ld ? "pack %" + f.names[i] + " to bf16 rows of " + std::to_string(s.cast.ld)
                         : "cast %" + f.names[i] + " f32->bf16 (skipped when passed as bf16)";
      plan.steps.push_back(s);
    }
    for (int ni : order) {
      Node& n = nodes[ni];
      if (n.is_dot) {
        if (n.is_prod) emit_prod(n);
        else emit_gemm(n);
        continue;
      }
      Step s;
      s.kind = Step::EW;
      std::vector<RedInfo> reds;
      build_group(n, s.ew, -1, &reds);
      std::vector<int64_t> shape = n.shape;
      int split = n.split;
      bool only_all = true;
      for (auto& ri : reds) only_all &= ri.kind == RED_ALL;
      if (reds.empty() || only_all) split = -1;
      if (shape.empty()) shape = {1};
      collapse(s.ew, shape, split);
      // kinds in the collapsed space.  A column reduction whose row dims were
      // all unit (erased) keeps its kind: R = 1, one partial per column.
      for (auto& ri : reds) s.ew.prog.reduce_kind[ri.slot_index] = ri.kind;
      rows_of_long_1d(s.ew);
      ew_launch(s.ew);
      s.ew.sig = program_signature(s.ew.prog);
      int64_t C = 1, R = 1;
      for (int d = 0; d < s.ew.ndims; ++d) (d < s.ew.ndims - s.ew.ncols ? R : C) *= s.ew.dims[d];
      std::ostringstream d;
      d << "ew [";
      for (int k = 0; k < s.ew.ndims; ++k) d << (k ? "," : "") << s.ew.dims[k];
      d << "] vec" << s.ew.vec << " in=" << (int)s.ew.prog.n_in << " ops=" << (int)s.ew.prog.n_ins
        << " stores=" << (int)s.ew.prog.n_stores << " reductions=" << (int)s.ew.prog.n_reduces << " roots:";
      for (auto& r : n.roots) {
        if (r.kind == Root::Fill) d << " fill(out" << r.out << ")";
        else if (r.kind == Root::Copy) d << " copy(%" << f.names[r.v] << "->out" << r.out << ")";
        else if (r.kind == Root::Reduce) d << " reduce(%" << f.names[r.red] << ")";
        else d << " %" << f.names[r.v];
      }
      s.desc = d.str();
      s.ew.desc = s.desc;
      plan.steps.push_back(s);
      finalize_reds(reds, (int)plan.steps.size() - 1, s.ew.gx, s.ew.gy, R, C, "ew");
    }
    add_events();
    for (auto& st : plan.steps)
      if (st.kind == Step::GEMM && st.gemm.tensor_core) {
        st.gemm.sched_index = plan.n_sched++;
        // large enough for a hybrid multicast + pair launch (its counter is
        // zeroed every run; the launcher decides per launch)
        const double flops = 2.0 * st.gemm.M * st.gemm.N * st.gemm.K;
        if (flops >= 68.7e9 && st.gemm.bn == 256 && st.gemm.M >= 1024) plan.hybrid_counters = true;
      }
    // 8 bytes per GEMM: a work counter (low word) or a hybrid claim state
    if (plan.n_sched) plan.sched_buf = add_buf(BufferSlot::Work, -1, (size_t)plan.n_sched * 8, SType::U8);
    plan.workspace_bytes = (plan.workspace_bytes + 255) / 256 * 256;
    plan.n_inputs = plan.seed_is_input ? f.num_args() - 1 : f.num_args();
    plan.n_outputs = (int)f.ret.size();
  }

  // `reduce %x by multiply along a` (Table 1; forward only):
  // an element-wise step over the result's index space whose one input walks
  // the reduced axis as nchunks = shape[a] chunks at the axis stride,
  // multiplied in index order by the load (chunk_op 1; `by max`: chunk_op 2,
  // the maximum, reading A26), then stored to every
  // home of the result.  Its consumers read those homes.
  void emit_prod(Node& n) {
    const Inst& in = f.insts[n.dot_inst];
    const int v = in.result, x = in.ops[0].value;
    TensorRef r;
    if (!ref_of(x, false, &r)) unsupported("reduce operand not addressable");
    const int rx = ty(x).rank();
    Step s;
    s.kind = Step::EW;
    EwGroup& g = s.ew;
    IterRef it;
    it.buf = r.buf;
    it.offset = r.offset;
    it.st = r.st;
    it.nchunks = (int)r.shape[in.axis];
    it.chunk_stride = r.strides[in.axis];
    it.chunk_op = in.reduce_max ? 2 : 1;
    for (int d = 0, j = 0; d < rx; ++d)
      if (d != in.axis) it.strides[j++] = r.strides[d];
    g.inputs.push_back(it);
    g.prog.n_in = 1;
    const int rk = ty(v).rank();
    for (auto& h : vi[v].homes) {
      if ((int)g.stores.size() >= kMaxStores) unsupported("too many stores in one fused kernel");
      IterRef o = store_ref(h.ref, identity(rk));
      o.st = h.st;
      g.prog.store_slot[g.stores.size()] = 0;
      g.stores.push_back(o);
    }
    g.prog.n_stores = (uint8_t)g.stores.size();
    std::vector<int64_t> shape = ty(v).shape;
    if (shape.empty()) shape = {1};
    collapse(g, shape, -1);
    rows_of_long_1d(g);
    ew_launch(g);
    g.sig = program_signature(g.prog);
    std::ostringstream d;
    d << "ew [";
    for (int k = 0; k < g.ndims; ++k) d << (k ? "," : "") << g.dims[k];
    d << "] vec" << g.vec << (in.reduce_max ? " max of %" : " product of %") << f.names[x] << " along " << in.axis
      << " (" << it.nchunks << (in.reduce_max ? " values" : " factors") << ") -> %" << f.names[v];
    s.desc = d.str();
    g.desc = s.desc;
    plan.steps.push_back(s);
  }

  void emit_gemm(Node& n) {
    const Inst& in = f.insts[n.dot_inst];
    int dv = in.result;
    Step s;
    s.kind = Step::GEMM;
    GemmStep& gm = s.gemm;
    gm.M = ty(dv).shape[0];
    gm.N = ty(dv).shape[1];
    bool bf = opt.policy == Policy::BF16;
    bool tc = bf && gm.M >= 128 && gm.N >= 64;
    for (size_t p = 0; p + 1 < in.ops.size(); p += 2) {
      GemmSeg sg;
      sg.K = in.ops[p].type.shape[1];
      for (int k = 0; k < 2; ++k) {
        const Operand& o = in.ops[p + k];
        if (o.is_lit()) unsupported("dot of a literal operand");
        TensorRef r;
        if (!ref_of(o.value, bf, &r)) unsupported("dot operand not addressable");
        if (bf && r.st != SType::BF16) unsupported("missing bf16 copy of a dot operand");
        if (r.strides.size() != 2 || !(r.strides[1] == 1 || r.strides[0] == 1 || r.shape[0] == 1 || r.shape[1] == 1))
          unsupported("dot operand needs a unit stride");
        (k == 0 ? sg.a : sg.b) = r;
      }
      // A [M,K]: K-major if K is the contiguous dim; B [K,N]: K-major if K is contiguous
      sg.a_kmajor = sg.a.strides[1] == 1 && (sg.a.shape[0] == 1 || sg.a.strides[0] != 1 || sg.a.shape[1] == 1);
      if (sg.a.strides[1] == 1 && sg.a.shape[1] != 1) sg.a_kmajor = true;
      if (sg.a.strides[0] == 1 && sg.a.shape[0] != 1 && sg.a.strides[1] != 1) sg.a_kmajor = false;
      sg.b_kmajor = sg.b.strides[0] == 1 && sg.b.shape[0] != 1 && sg.b.strides[1] != 1;
      int64_t lda = sg.a_kmajor ? sg.a.strides[0] : sg.a.strides[1];
      int64_t ldb = sg.b_kmajor ? sg.b.strides[1] : sg.b.strides[0];
      tc = tc && lda % 8 == 0 && ldb % 8 == 0 && sg.a.offset % 8 == 0 && sg.b.offset % 8 == 0;
      gm.K += sg.K;
      gm.seg.push_back(sg);
    }
    gm.tensor_core = tc && gm.K >= 64;
    // SIMT: 32-row tiles when 64-row tiles would not fill the SMs twice over
    // (the tile fixes the epilogue partial layout, so it is chosen here)
    const int64_t simt_tiles64 = ((gm.M + 63) / 64) * ((gm.N + 63) / 64);
    gm.bm = gm.tensor_core ? 128 : (simt_tiles64 < 2 * 148 ? 32 : 64);
    gm.bn = gm.tensor_core ? (gm.N >= 256 ? 256 : 128) : 64;
    // very few 256 x 256 pair tiles (under half the 74 CTA pairs): 128 x 128
    // single-CTA tiles spread the contraction over 4x as many SMs
    if (gm.tensor_core && gm.bn == 256 && ((gm.M + 255) / 256) * ((gm.N + 255) / 256) < 37) gm.bn = 128;
    if (!gm.tensor_core && (gm.M + gm.bm - 1) / gm.bm > 65535)
      unsupported("SIMT dot with more than 65535 row tiles (over 4M rows under the fp32 dot policy)");
    Node epi;
    if (n.fused_epilogue >= 0) epi = nodes[n.fused_epilogue];
    epi.shape = ty(dv).shape;
    epi.perm = identity(2);
    std::vector<Root> roots;
    if (!vi[dv].homes.empty()) {
      Root self;
      self.kind = Root::Store;
      self.v = dv;
      roots.push_back(self);
    }
    for (auto& r : epi.roots) roots.push_back(r);
    epi.roots = roots;
    std::vector<RedInfo> reds;
    build_group(epi, gm.epi, dv, &reds);
    gm.epi.ndims = 2;
    gm.epi.dims[0] = gm.M;
    gm.epi.dims[1] = gm.N;
    for (auto& ri : reds) gm.epi.prog.reduce_kind[ri.slot_index] = ri.kind;
    int64_t gx = (gm.N + gm.bn - 1) / gm.bn, gy = (gm.M + gm.bm - 1) / gm.bm;
    gm.epi.gx = gx;
    gm.epi.gy = gy;
    gm.epi.sig = program_signature(gm.epi.prog);
    // split K when the tile grid fills the SMs badly (wave quantization):
    // the GEMM stores S raw partial tiles and the epilogue program moves to
    // an EW step that sums them in split order (deterministic)
    const int S = split_k(gm);
    // An epilogue reading two or more f32 [M, N] operands (mlp_hvp's
    // second-order terms %o: two, %d9: four) cannot stage them through
    // shared memory (128 KB per operand per 256-wide tile) and loads them row
    // per lane at a fraction of HBM bandwidth: the GEMM stores its raw
    // accumulator and the epilogue program runs as the next EW step instead
    // (same program on the same f32 values: bit-identical).  DLVM_EPI_DEFER=n
    // sets the operand count (0: never).  Measured (mlp_hvp step, one B200):
    // 1.414 ms fused, 1.326 deferring at 3 operands, 1.318 at 2
    const int heavy = f32_row_inputs(gm.epi);
    static const int defer_min = [] {  // DLVM_EPI_DEFER=n: the operand count that defers (0: never)
      const char* e = std::getenv("DLVM_EPI_DEFER");
      return e ? std::atoi(e) : 2;
    }();
    // likewise stores whose TMA staging (one 32 x 64 group of each per
    // epilogue warp: 8 KB f32, 4 KB bf16, 2 KB bytes) exceeds the 12 KB per
    // warp the pipeline can give up: they would fall back to row-per-lane
    // stores (mlp_hvp %z: two f32 + two bf16 stores, 24 KB; 367 us fused vs
    // 200 us for the same GEMM storing only its accumulator)
    const int stage_kb = store_stage_kb(gm.epi);
    // (not epilogues with reductions: the EW kernel sums in another order
    // than the epilogue's butterflies, so the result would be equal only to
    // rounding, A17, where the fused and deferred forms are now bit-identical)
    const bool defer = S == 1 && defer_min > 0 && gm.tensor_core && gm.epi.prog.n_reduces == 0 &&
                       (heavy >= defer_min || stage_kb > 12);
    EwGroup split_ew;
    if (S > 1 || defer) {
      split_ew = gm.epi;
      const int pbuf = add_buf(BufferSlot::Work, -1, (size_t)S * gm.M * gm.N * 4, SType::F32);
      IterRef part;
      part.buf = pbuf;
      part.strides[0] = gm.N;
      part.strides[1] = 1;
      part.nchunks = S;
      part.chunk_stride = gm.M * gm.N;
      split_ew.inputs[0] = part;
      split_ew.ndims = 2;
      split_ew.ncols = 1;
      split_ew.dims[0] = gm.M;
      split_ew.dims[1] = gm.N;
      ew_launch(split_ew);
      split_ew.sig = program_signature(split_ew.prog);
      EwGroup st;
      st.ndims = 2;
      st.dims[0] = gm.M;
      st.dims[1] = gm.N;
      IterRef acc;
      acc.buf = -2;
      st.inputs.push_back(acc);
      IterRef o;
      o.buf = pbuf;
      o.strides[0] = gm.N;
      o.strides[1] = 1;
      st.stores.push_back(o);
      st.prog.n_in = 1;
      st.prog.n_stores = 1;
      st.prog.store_slot[0] = 0;
      st.gx = gx;
      st.gy = gy;
      st.sig = program_signature(st.prog);
      gm.epi = st;
      gm.ksplit = S;
      gm.split_bytes = gm.M * gm.N * 4;
      const EwProgram& sp = split_ew.prog;
      gm.split_red_ok = S == 2 && sp.n_ins == 0 && sp.n_lits == 0 && sp.n_in == 1 && sp.n_stores == 1 &&
                        sp.n_reduces == 0 && sp.store_slot[0] == 0 && split_ew.stores.size() == 1 &&
                        split_ew.stores[0].buf >= 0 && split_ew.stores[0].strides[1] == 1 &&
                        split_ew.stores[0].strides[0] == gm.N;
    }
    std::ostringstream d;
    d << (gm.tensor_core ? "gemm tcgen05 bf16" : (bf ? "gemm simt bf16" : "gemm simt f32")) << " %"
      << f.names[dv] << " M=" << gm.M << " N=" << gm.N << " K=" << gm.K;
    if (gm.seg.size() > 1) {
      d << " (" << gm.seg.size() << " K segments:";
      for (auto& sg : gm.seg) d << " " << sg.K;
      d << ")";
    }
    d << " A:" << (gm.seg[0].a_kmajor ? "K" : "M") << "-major B:" << (gm.seg[0].b_kmajor ? "K" : "N")
      << "-major; epilogue ops=" << (int)gm.epi.prog.n_ins
      << " in=" << (int)gm.epi.prog.n_in << " stores=" << (int)gm.epi.prog.n_stores
      << " reductions=" << (int)gm.epi.prog.n_reduces;
    if (n.fused_epilogue >= 0) {
      d << " roots:";
      for (auto& r : nodes[n.fused_epilogue].roots) {
        if (r.kind == Root::Reduce) d << " reduce(%" << f.names[r.red] << ")";
        else if (r.kind == Root::Store) d << " %" << f.names[r.v];
        else if (r.kind == Root::Copy) d << " copy(%" << f.names[r.v] << ")";
      }
    }
    if (S > 1) d << " (K split " << S << ", raw partials; epilogue in the next step)";
    if (defer)
      d << " (raw accumulator; epilogue with " << heavy << " f32 [M,N] operands, " << stage_kb
        << " KB of store staging per warp, in the next step)";
    s.desc = d.str();
    gm.epi.desc = s.desc;
    plan.steps.push_back(s);
    if (S > 1 || defer) {
      Step e;
      e.kind = Step::EW;
      e.ew = split_ew;
      std::ostringstream de;
      de << "ew [" << gm.M << "," << gm.N << "] vec" << split_ew.vec;
      if (S > 1)
        de << " sum of " << S << " K-split partials of %" << f.names[dv];
      else
        de << " deferred epilogue of %" << f.names[dv];
      de << " + epilogue ops=" << (int)split_ew.prog.n_ins << " stores=" << (int)split_ew.prog.n_stores
         << " reductions=" << (int)split_ew.prog.n_reduces;
      if (gm.split_red_ok) de << " (skipped when the home is bound as f32: the GEMM adds the splits into it)";
      e.desc = de.str();
      e.ew.desc = e.desc;
      plan.steps.push_back(e);
      finalize_reds(reds, (int)plan.steps.size() - 1, split_ew.gx, split_ew.gy, gm.M, gm.N, "%" + f.names[dv]);
      return;
    }
    finalize_reds(reds, (int)plan.steps.size() - 1, gx, gy, gm.M, gm.N, "%" + f.names[dv]);
  }

  // K split factor for a tcgen05 GEMM: the tile grid over the persistent
  // CTAs (148 SMs; CTA pairs for 256-wide tiles with M >= 512, as the
  // launcher chooses) leaves the last wave partly idle; splitting K into S
  // work items per tile is worth it when it raises the busy fraction by > 5
  // points and every split keeps K/S >= 4096 (DLVM_GEMM_SPLITK=0 disables)
  // [M, N] row-contiguous f32 operands of a GEMM epilogue (slot 0, the
  // accumulator, excluded); caller inputs count as f32 (their usual binding)
  int f32_row_inputs(const EwGroup& g) const {
    int n = 0;
    for (size_t q = 1; q < g.inputs.size(); ++q) {
      const IterRef& r = g.inputs[q];
      if (r.buf < 0 || r.nchunks != 1 || r.strides[1] != 1 || r.strides[0] == 0) continue;
      if (plan.bufs[r.buf].st == SType::F32) ++n;
    }
    return n;
  }

  // TMA store staging per epilogue warp in KB (setup_tma_epilogue): one
  // 32 x 64 group of every store; caller outputs count as f32
  int store_stage_kb(const EwGroup& g) const {
    int kb = 0;
    for (auto& r : g.stores) {
      const SType st = r.buf >= 0 ? plan.bufs[r.buf].st : SType::F32;
      kb += st == SType::F32 ? 8 : st == SType::BF16 ? 4 : 2;
    }
    return kb;
  }

  static int split_k(const GemmStep& gm) {
    static const bool on = [] {
      const char* e = std::getenv("DLVM_GEMM_SPLITK");
      return !(e && e[0] == '0');
    }();
    if (!on || !gm.tensor_core || gm.seg.size() != 1) return 1;
    const int ctas = (gm.bn == 256 && gm.M >= 512) ? 2 : 1;
    const int64_t clusters = 148 / ctas;
    const int64_t tiles = ((gm.M + 128 * ctas - 1) / (128 * ctas)) * ((gm.N + gm.bn - 1) / gm.bn);
    auto busy = [&](int64_t w) {
      const int64_t waves = (w + clusters - 1) / clusters;
      return (double)w / (double)(waves * clusters);
    };
    double best = busy(tiles);
    int bs = 1;
    for (int S = 2; S <= 4; ++S)
      if (gm.K / S >= 4096 && busy(tiles * S) > best + 0.05) {
        best = busy(tiles * S);
        bs = S;
      }
    return bs;
  }

  void add_events() {
    if (opt.n_grads <= 0) return;
    std::vector<int> last(opt.n_grads, -1);
    for (size_t si = 0; si < plan.steps.size(); ++si) {
      const Step& s = plan.steps[si];
      const std::vector<IterRef>* st =
          s.kind == Step::EW ? &s.ew.stores : s.kind == Step::GEMM ? &s.gemm.epi.stores : nullptr;
      if (!st) continue;
      const EwGroup& g = s.kind == Step::EW ? s.ew : s.gemm.epi;
      std::vector<int> written;
      for (auto& r : *st) written.push_back(r.buf);
      for (auto& r : g.reduces)  // single-partial reductions write their home directly
        if (r.direct_buf >= 0) written.push_back(r.direct_buf);
      for (int buf : written) {
        const BufferSlot& b = plan.bufs[buf];
        if (b.kind == BufferSlot::Output && b.index < opt.n_grads) last[b.index] = (int)si;
      }
    }
    std::vector<Step> out;
    auto ev = [&](int k) {
      Step e;
      e.kind = Step::EVENT;
      e.event_index = k;
      e.desc = "event: gradient " + std::to_string(k) + " ready";
      out.push_back(e);
    };
    for (int k = 0; k < opt.n_grads; ++k)
      if (last[k] < 0) ev(k);
    for (size_t si = 0; si < plan.steps.size(); ++si) {
      out.push_back(plan.steps[si]);
      for (int k = 0; k < opt.n_grads; ++k)
        if (last[k] == (int)si) ev(k);
    }
    plan.steps.swap(out);
  }

  // a dot / product operand reached through views must be one strided ref
  // (dots: a unit stride in one dim); a view that is not (e.g. a shapeCast
  // merging the dims of a transposed or row-padded home) is materialised by
  // its own copy root, and planning repeats
  bool force_unaddressable_operands() {
    // a view of a materialised value read by an element-wise kernel at a
    // map that does not pass through it (merging / splitting shapeCast,
    // slice) must have a strided ref
    for (size_t v = 0; v < f.types.size(); ++v) {
      const Inst* in = def((int)v);
      if (!in || !is_view(in) || !vi[v].inl || vi[v].dead || force_mat.count((int)v)) continue;
      const int src = in->ops[0].value;
      Map ma;
      if (vi[src].inl && in->op != Op::Slice && view_map(*in, identity(ty((int)v).rank()), &ma)) continue;
      bool read = false;
      for (auto& n : nodes)
        if (!n.is_dot && n.merged_into < 0 && n.inl.count((int)v)) read = true;
      if (!read) continue;
      TensorRef r;
      if (ref_of((int)v, false, &r)) continue;
      force_mat.insert((int)v);
      return true;
    }
    for (auto& in : f.insts) {
      const bool dot = is_dotlike(in.op);
      if (!dot && !is_prod(&in)) continue;
      const bool bf = dot && opt.policy == Policy::BF16;
      for (auto& o : in.ops) {
        if (o.is_lit() || vi[o.value].dead) continue;
        const int v = o.value;
        TensorRef r;
        bool ok = ref_of(v, bf, &r) && (!bf || r.st == SType::BF16);
        if (ok && dot)
          ok = r.strides.size() == 2 &&
               (r.strides[1] == 1 || r.strides[0] == 1 || r.shape[0] == 1 || r.shape[1] == 1);
        if (ok) continue;
        int u = v;  // the outermost inlined view that is not addressable
        if (!(vi[u].inl && is_view(def(u))) || force_mat.count(u))
          unsupported(dot ? "dot operand not addressable" : "reduce operand not addressable");
        force_mat.insert(u);
        return true;
      }
    }
    return false;
  }

  void run() {
    check_supported();
    peepholes();
    analyse();
    reduce_chains();
    for (int outer = 0;; ++outer) {
      if (outer > 100) throw Error(kStatusRuntime, 0, 0, "planner did not converge");
      for (int iter = 0;; ++iter) {
        if (iter > 1000) throw Error(kStatusRuntime, 0, 0, "planner did not converge");
        need_iterate = false;
        decide();
        alias_outputs();
        build_nodes();
        for (auto& n : nodes) region_of(n);
        if (need_iterate) continue;
        if (split_oversized()) continue;
        build_edges();
        merge_groups();
        if (!duplicates()) break;
      }
      fuse_epilogues();
      assign_homes();
      if (!force_unaddressable_operands()) break;
    }
    emit_steps(schedule());
    check_no_self_reads();
  }

  // every launch reads only buffers it does not write: a load of a value the
  // same launch stores would race the store (another thread's, or its own
  // later in program order)
  void check_no_self_reads() const {
    for (size_t i = 0; i < plan.steps.size(); ++i) {
      const Step& s = plan.steps[i];
      const EwGroup* g = s.kind == Step::EW ? &s.ew : s.kind == Step::GEMM ? &s.gemm.epi : nullptr;
      if (!g) continue;
      std::set<int> w;
      for (auto& r : g->stores) w.insert(r.buf);
      for (auto& r : g->reduces) {
        w.insert(r.buf);
        if (r.direct_buf >= 0) w.insert(r.direct_buf);
      }
      std::vector<int> rd;
      for (auto& r : g->inputs)
        if (r.buf >= 0) rd.push_back(r.buf);
      if (s.kind == Step::GEMM)
        for (auto& sg : s.gemm.seg) {
          rd.push_back(sg.a.buf);
          rd.push_back(sg.b.buf);
        }
      for (int b : rd)
        if (w.count(b))
          throw Error(kStatusRuntime, 0, 0,
                      "planner: step " + std::to_string(i) + " (" + s.desc + ") reads buffer " + std::to_string(b) +
                          " that it writes");
    }
  }
};

}  // namespace

Plan make_plan(const Function& f, const PlanOptions& opt) {
  Planner p(f, opt);
  p.plan.seed_is_input = f.grad.has_value() && f.grad->seedable;
  p.run();
  return p.plan;
}

}  // namespace dlvm
