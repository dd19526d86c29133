// Parser for the textual DLVM IR (*.dl).
//
// Syntax follows Fig. 3 and Table 1 (L170-181):
//   module "name" / stage raw|optimizable
//   [gradient @f wrt i, j keeping k from o seedable]   (Fig. 3)
//   func @name: (T, ...) -> T | (T, ...) [{ 'label(%a: T, ...): insts return }]
// Every operand carries its type annotation (`%a: <10 x f32>`, Table 1);
// literals are `2: f32` (Table 1, reading A8); tuple return is
// `return (%a: T, %b: T)` (reading A22).  Names are resolved later by the
// verifier, so a malformed text is always reported as a parse error (2)
// before any type error (1).
#include <cerrno>
#include <cctype>
#include <cmath>
#include <cstdlib>

#include "ir.h"

namespace dlvm {

namespace {

enum class Tk { Str, Global, Local, Label, Num, Arrow, Punct, Ident, Eof };

struct Token {
  Tk kind;
  std::string text;
  int line, col;
};

std::vector<Token> tokenize(const std::string& s) {
  std::vector<Token> out;
  size_t i = 0, n = s.size();
  int line = 1, col = 1;
  auto adv = [&](size_t k) {
    for (size_t j = 0; j < k; ++j) {
      if (s[i] == '\n') {
        ++line;
        col = 1;
      } else {
        ++col;
      }
      ++i;
    }
  };
  auto is_id = [](char c) { return std::isalnum((unsigned char)c) || c == '_' || c == '.'; };
  while (i < n) {
    char c = s[i];
    if (c == ' ' || c == '\t' || c == '\r' || c == '\n') {
      adv(1);
      continue;
    }
    if (c == '/' && i + 1 < n && s[i + 1] == '/') {
      while (i < n && s[i] != '\n') adv(1);
      continue;
    }
    int ln = line, cl = col;
    size_t st = i;
    if (c == '"') {
      size_t j = i + 1;
      while (j < n && s[j] != '"' && s[j] != '\n') ++j;
      if (j >= n || s[j] != '"') throw Error(kStatusParse, ln, cl, "unterminated string");
      adv(j + 1 - i);
      out.push_back({Tk::Str, s.substr(st, i - st), ln, cl});
      continue;
    }
    if (c == '@' || c == '%' || c == '\'') {
      size_t j = i + 1;
      while (j < n && is_id(s[j])) ++j;
      if (j == i + 1) throw Error(kStatusParse, ln, cl, std::string("expected name after '") + c + "'");
      adv(j - i);
      out.push_back({c == '@' ? Tk::Global : c == '%' ? Tk::Local : Tk::Label, s.substr(st, i - st), ln, cl});
      continue;
    }
    if (c == '-' && i + 1 < n && s[i + 1] == '>') {
      adv(2);
      out.push_back({Tk::Arrow, "->", ln, cl});
      continue;
    }
    bool num_start = std::isdigit((unsigned char)c) ||
                     (c == '.' && i + 1 < n && std::isdigit((unsigned char)s[i + 1])) ||
                     (c == '-' && i + 1 < n &&
                      (std::isdigit((unsigned char)s[i + 1]) || s[i + 1] == '.' ||
                       s.compare(i + 1, 3, "inf") == 0 || s.compare(i + 1, 3, "nan") == 0));
    if (num_start) {
      size_t j = i;
      if (s[j] == '-') ++j;
      if (s.compare(j, 3, "inf") == 0 || s.compare(j, 3, "nan") == 0) {
        j += 3;
      } else {
        while (j < n && std::isdigit((unsigned char)s[j])) ++j;
        if (j < n && s[j] == '.') {
          ++j;
          while (j < n && std::isdigit((unsigned char)s[j])) ++j;
        }
        if (j < n && (s[j] == 'e' || s[j] == 'E')) {
          size_t k = j + 1;
          if (k < n && (s[k] == '+' || s[k] == '-')) ++k;
          if (k < n && std::isdigit((unsigned char)s[k])) {
            j = k;
            while (j < n && std::isdigit((unsigned char)s[j])) ++j;
          }
        }
      }
      adv(j - i);
      out.push_back({Tk::Num, s.substr(st, i - st), ln, cl});
      continue;
    }
    if (std::string("(){}[]<>,:=").find(c) != std::string::npos) {
      adv(1);
      out.push_back({Tk::Punct, std::string(1, c), ln, cl});
      continue;
    }
    if (std::isalpha((unsigned char)c) || c == '_') {
      size_t j = i;
      while (j < n && (std::isalnum((unsigned char)s[j]) || s[j] == '_')) ++j;
      adv(j - i);
      std::string w = s.substr(st, i - st);
      out.push_back({(w == "inf" || w == "nan") ? Tk::Num : Tk::Ident, w, ln, cl});
      continue;
    }
    throw Error(kStatusParse, ln, cl, std::string("unexpected character '") + c + "'");
  }
  out.push_back({Tk::Eof, "", line, col});
  return out;
}

struct Parser {
  std::vector<Token> t;
  size_t i = 0;

  const Token& peek(size_t k = 0) const { return t[std::min(i + k, t.size() - 1)]; }
  const Token& next() {
    const Token& x = t[i];
    if (i + 1 < t.size()) ++i;
    return x;
  }
  [[noreturn]] void fail(const Token& x, const std::string& m) { throw Error(kStatusParse, x.line, x.col, m); }
  const Token& expect(const std::string& s) {
    const Token& x = next();
    if (x.text != s || x.kind == Tk::Str) fail(x, "expected '" + s + "', found '" + (x.text.empty() ? "<eof>" : x.text) + "'");
    return x;
  }
  bool accept(const std::string& s) {
    if (peek().text == s && peek().kind != Tk::Str) {
      next();
      return true;
    }
    return false;
  }
  int64_t integer() {
    const Token& x = next();
    bool ok = x.kind == Tk::Num && !x.text.empty();
    for (size_t k = 0; ok && k < x.text.size(); ++k)
      ok = std::isdigit((unsigned char)x.text[k]) || (k == 0 && x.text[k] == '-' && x.text.size() > 1);
    if (!ok) fail(x, "expected integer, found '" + x.text + "'");
    errno = 0;
    const long long v = std::strtoll(x.text.c_str(), nullptr, 10);
    if (errno == ERANGE) fail(x, "integer '" + x.text + "' out of range");
    return v;
  }
  // element count of a shape; rejects shapes of more than 2^59 elements
  // (2^62 bytes at 8 bytes per element), so numel() and every byte size
  // derived from it stay far from int64 overflow
  void check_numel(const Token& at, const std::vector<int64_t>& shape) {
    int64_t n = 1;
    for (int64_t d : shape)
      if (__builtin_mul_overflow(n, d, &n) || n > (int64_t(1) << 59))
        fail(at, "tensor has too many elements (more than 2^59)");
  }
  DType dtype() {
    const Token& x = next();
    DType d;
    if (x.kind != Tk::Ident || !dtype_from_name(x.text, &d)) fail(x, "expected data type, found '" + x.text + "'");
    return d;
  }
  bool peek_dtype() const {
    DType d;
    return peek().kind == Tk::Ident && dtype_from_name(peek().text, &d);
  }
  Type type() {
    Type ty;
    if (peek().text == "<" && peek().kind == Tk::Punct) {
      next();
      const Token& first = peek();
      while (!peek_dtype()) {
        const Token& u = peek();
        int64_t d = integer();
        if (d < 1) fail(u, "tensor dimensions must be >= 1");
        ty.shape.push_back(d);
        expect("x");
      }
      check_numel(first, ty.shape);
      ty.dtype = dtype();
      expect(">");
      return ty;
    }
    ty.dtype = dtype();
    return ty;
  }
  std::vector<Type> type_list(bool* tuple) {
    std::vector<Type> v;
    *tuple = false;
    if (peek().text == "(" && peek().kind == Tk::Punct) {
      next();
      *tuple = true;
      if (accept(")")) return v;
      for (;;) {
        v.push_back(type());
        if (accept(")")) break;
        expect(",");
      }
      return v;
    }
    v.push_back(type());
    return v;
  }
  Operand operand() {
    const Token& x = next();
    Operand o;
    o.line = x.line;
    o.col = x.col;
    if (x.kind == Tk::Local) {
      o.vname = x.text.substr(1);
      expect(":");
      o.type = type();
      return o;
    }
    if (x.kind == Tk::Num || (x.kind == Tk::Ident && (x.text == "true" || x.text == "false"))) {
      expect(":");
      o.type = type();
      if (x.kind == Tk::Ident) {
        if (o.type.dtype != DType::Bool) fail(x, "boolean literal must have type bool");
        o.lit = x.text == "true" ? 1.0 : 0.0;
      } else {
        o.lit = std::strtod(x.text.c_str(), nullptr);
      }
      return o;
    }
    fail(x, "expected operand, found '" + (x.text.empty() ? std::string("<eof>") : x.text) + "'");
  }
  Inst inst() {
    const Token& x = peek();
    Inst in;
    in.line = x.line;
    in.col = x.col;
    bool named = false;
    if (x.kind == Tk::Local) {
      in.rname = next().text.substr(1);
      named = true;
      expect("=");
    }
    const Token& opk = next();
    Op op;
    if (opk.kind != Tk::Ident || !op_from_name(opk.text, &op)) fail(opk, "unknown opcode '" + opk.text + "'");
    in.op = op;
    if (is_unary(op) || op == Op::Transpose) {
      in.ops.push_back(operand());
    } else if (is_binary(op) || is_compare(op) || op == Op::Dot) {
      in.ops.push_back(operand());
      expect(",");
      in.ops.push_back(operand());
    } else if (op == Op::Select) {
      in.ops.push_back(operand());
      expect(",");
      in.ops.push_back(operand());
      expect(",");
      in.ops.push_back(operand());
    } else if (op == Op::Reduce) {
      in.ops.push_back(operand());
      expect("by");
      const Token& r = next();
      if (r.text != "add" && r.text != "multiply" && r.text != "max") fail(r, "unknown reduction '" + r.text + "'");
      in.reduce_mul = r.text == "multiply";
      in.reduce_max = r.text == "max";  // extension (reading A26)
      expect("along");
      in.axis = (int)integer();
    } else if (op == Op::ShapeCast) {
      in.ops.push_back(operand());
      expect("to");
      const Token& first = peek();
      in.shape.push_back(integer());
      while (peek().text == "x" && peek().kind == Tk::Ident) {
        next();
        in.shape.push_back(integer());
      }
      check_numel(first, in.shape);
    } else if (op == Op::DataTypeCast) {
      in.ops.push_back(operand());
      expect("to");
      in.cast_to = dtype();
    } else if (op == Op::Slice) {
      in.ops.push_back(operand());
      expect("from");
      in.from = integer();
      expect("upto");
      in.upto = integer();
    }
    if (!named) fail(opk, "instruction result must be named");
    return in;
  }
  std::vector<int> int_list() {
    std::vector<int> v{(int)integer()};
    while (accept(",")) v.push_back((int)integer());
    return v;
  }
  GradConfig attr() {
    const Token& lb = expect("[");
    expect("gradient");
    const Token& src = next();
    if (src.kind != Tk::Global) fail(src, "expected function name after 'gradient'");
    GradConfig c;
    c.source = src.text.substr(1);
    c.line = lb.line;
    c.col = lb.col;
    std::vector<std::string> seen;
    while (!accept("]")) {
      const Token& k = next();
      for (auto& s : seen)
        if (s == k.text) fail(k, "duplicate '" + k.text + "' in gradient attribute");
      seen.push_back(k.text);
      if (k.text == "wrt") {
        c.has_wrt = true;
        c.wrt = int_list();
      } else if (k.text == "keeping") {
        c.keeping = int_list();
      } else if (k.text == "from") {
        c.has_from = true;
        c.from = (int)integer();
      } else if (k.text == "seedable") {
        c.seedable = true;
      } else {
        fail(k, "unexpected '" + k.text + "' in gradient attribute");
      }
    }
    return c;
  }
  Function function(std::optional<GradConfig> g) {
    const Token& ft = expect("func");
    const Token& nm = next();
    if (nm.kind != Tk::Global) fail(nm, "expected function name");
    Function f;
    f.name = nm.text.substr(1);
    f.line = ft.line;
    f.col = ft.col;
    f.grad = g;
    expect(":");
    bool tup;
    f.params = type_list(&tup);
    expect("->");
    f.results = type_list(&f.result_tuple);
    if (!(peek().text == "{" && peek().kind == Tk::Punct)) return f;
    next();
    const Token& lab = next();
    if (lab.kind != Tk::Label) fail(lab, "expected basic block label");
    f.has_body = true;
    f.label = lab.text.substr(1);
    expect("(");
    if (!accept(")")) {
      for (;;) {
        const Token& p = next();
        if (p.kind != Tk::Local) fail(p, "expected block argument");
        expect(":");
        f.names.push_back(p.text.substr(1));
        f.arg_types.push_back(type());
        f.arg_locs.push_back({p.line, p.col});
        if (accept(")")) break;
        expect(",");
      }
    }
    expect(":");
    for (;;) {
      const Token& x = peek();
      if (x.kind == Tk::Ident && x.text == "return") {
        next();
        f.ret_line = x.line;
        if (peek().text == "(" && peek().kind == Tk::Punct) {
          next();
          if (!accept(")")) {
            for (;;) {
              f.ret.push_back(operand());
              if (accept(")")) break;
              expect(",");
            }
          }
        } else if (!(peek().text == "}" && peek().kind == Tk::Punct)) {
          f.ret.push_back(operand());
        }
        break;
      }
      if ((x.text == "}" && x.kind == Tk::Punct) || x.kind == Tk::Eof) fail(x, "basic block must end with 'return'");
      if (x.kind == Tk::Label) fail(x, "multiple basic blocks are not supported (straight-line only)");
      f.insts.push_back(inst());
    }
    expect("}");
    return f;
  }
  Module module() {
    expect("module");
    const Token& nm = next();
    if (nm.kind != Tk::Str) fail(nm, "expected module name string");
    Module m;
    m.name = nm.text.substr(1, nm.text.size() - 2);
    expect("stage");
    const Token& st = next();
    if (st.text != "raw" && st.text != "optimizable") fail(st, "unknown stage '" + st.text + "'");
    m.stage = st.text;
    while (peek().kind != Tk::Eof) {
      std::optional<GradConfig> g;
      if (peek().text == "[" && peek().kind == Tk::Punct) g = attr();
      const Token& at = peek();
      Function f = function(g);
      if (m.find(f.name)) throw Error(kStatusParse, at.line, at.col, "redefinition of function @" + f.name);
      m.fns.push_back(std::move(f));
    }
    return m;
  }
};

}  // namespace

Module parse_module(const std::string& text) {
  Parser p;
  p.t = tokenize(text);
  return p.module();
}

}  // namespace dlvm
