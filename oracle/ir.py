"""Oracle IR data model, parser and printer (test infrastructure only).

The textual form follows Fig. 3 and Table 1; the
grammar sketch is S:L181-189.  Readings taken where the paper is silent
(DESIGN.md §Readings):
  A4  Fig. 3's garbled body is `%0 = dot ...; %1 = add ...; return %1`.
  A8  a literal `2: f32` may appear in any operand slot.
  A22 tuple return is written `return (%a: T, %b: T)`.
  A23 gradient declarations are body-less `func` lines preceded by a
      `[gradient @f wrt .. keeping .. from .. seedable]` attribute.
"""

from __future__ import annotations

import re
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

DTYPES = ("bool", "i8", "i16", "i32", "i64", "f16", "f32", "f64")
FLOAT_DTYPES = ("f16", "f32", "f64")

UNARY = ("negate", "tanh", "exp", "log", "sqrt", "abs", "sign")
BINARY = ("add", "subtract", "multiply", "divide", "power")
COMPARE = ("lt", "le", "gt", "ge", "eq", "ne")
OPCODES = UNARY + BINARY + COMPARE + (
    "select", "dot", "reduce", "transpose", "shapeCast", "dataTypeCast", "slice")


class ParseError(Exception):
    """Exit class 2."""

    def __init__(self, line: int, col: int, msg: str):
        super().__init__(f"{line}:{col}: error: {msg}")
        self.line, self.col, self.msg = line, col, msg


class VerifyError(Exception):
    """Exit class 1: type, shape, gradient-config errors."""

    def __init__(self, line: int, col: int, msg: str):
        super().__init__(f"{line}:{col}: error: {msg}")
        self.line, self.col, self.msg = line, col, msg


@dataclass(frozen=True)
class TensorType:
    shape: Tuple[int, ...]
    dtype: str

    def __str__(self) -> str:
        if not self.shape:
            return self.dtype
        return "<" + " x ".join(str(d) for d in self.shape) + " x " + self.dtype + ">"

    @property
    def rank(self) -> int:
        return len(self.shape)


@dataclass
class Operand:
    kind: str                      # "value" | "literal"
    type: TensorType               # the annotation written in the text
    name: Optional[str] = None     # for values, without the leading '%'
    literal: Optional[float] = None
    line: int = 0
    col: int = 0

    def __str__(self) -> str:
        if self.kind == "value":
            return f"%{self.name}: {self.type}"
        lit = self.literal
        if self.type.dtype == "bool":
            s = "true" if lit else "false"
        elif float(lit).is_integer() and abs(lit) < 1e15:
            s = str(int(lit))
        else:
            s = repr(float(lit))
        return f"{s}: {self.type}"


@dataclass
class Inst:
    result: Optional[str]
    opcode: str
    operands: List[Operand]
    attrs: Dict[str, object] = field(default_factory=dict)
    line: int = 0
    col: int = 0

    def __str__(self) -> str:
        ops = ", ".join(str(o) for o in self.operands)
        if self.opcode == "reduce":
            body = f"reduce {ops} by {self.attrs['op']} along {self.attrs['axis']}"
        elif self.opcode == "shapeCast":
            body = f"shapeCast {ops} to " + " x ".join(str(d) for d in self.attrs["shape"])
        elif self.opcode == "dataTypeCast":
            body = f"dataTypeCast {ops} to {self.attrs['dtype']}"
        elif self.opcode == "slice":
            body = f"slice {ops} from {self.attrs['from']} upto {self.attrs['upto']}"
        else:
            body = f"{self.opcode} {ops}"
        return (f"%{self.result} = " if self.result is not None else "") + body


@dataclass
class GradConfig:
    source: str
    wrt: Optional[List[int]] = None
    keeping: List[int] = field(default_factory=list)
    from_: Optional[int] = None
    seedable: bool = False
    line: int = 0
    col: int = 0


@dataclass
class Function:
    name: str
    param_types: List[TensorType]
    result_types: List[TensorType]
    result_is_tuple: bool
    label: Optional[str] = None
    param_names: List[str] = field(default_factory=list)
    arg_types: List[TensorType] = field(default_factory=list)
    arg_locs: List[Tuple[int, int]] = field(default_factory=list)
    types: Dict[str, TensorType] = field(default_factory=dict)
    insts: List[Inst] = field(default_factory=list)
    ret: List[Operand] = field(default_factory=list)
    ret_line: int = 0
    gradient: Optional[GradConfig] = None
    line: int = 0
    col: int = 0

    @property
    def has_body(self) -> bool:
        return self.label is not None


@dataclass
class Module:
    name: str
    stage: str
    functions: Dict[str, Function]


# --------------------------------------------------------------------------
# tokenizer

_TOKEN_RE = re.compile(r"""
    (?P<ws>[ \t\r\n]+)
  | (?P<comment>//[^\n]*)
  | (?P<string>"[^"\n]*")
  | (?P<global>@[A-Za-z_][A-Za-z0-9_.]*)
  | (?P<local>%[A-Za-z0-9_.]+)
  | (?P<label>'[A-Za-z_][A-Za-z0-9_.]*)
  | (?P<number>-?(?:\d+\.\d*(?:[eE][-+]?\d+)?|\d+[eE][-+]?\d+|\.\d+(?:[eE][-+]?\d+)?|\d+|inf|nan))
  | (?P<arrow>->)
  | (?P<punct>[(){}\[\]<>,:=])
  | (?P<ident>[A-Za-z_][A-Za-z0-9_]*)
""", re.VERBOSE)


@dataclass
class Tok:
    kind: str
    text: str
    line: int
    col: int


def tokenize(text: str) -> List[Tok]:
    toks: List[Tok] = []
    pos, line, col = 0, 1, 1
    n = len(text)
    while pos < n:
        m = _TOKEN_RE.match(text, pos)
        if not m:
            raise ParseError(line, col, f"unexpected character {text[pos]!r}")
        kind = m.lastgroup
        s = m.group()
        if kind not in ("ws", "comment"):
            toks.append(Tok(kind, s, line, col))
        nl = s.count("\n")
        if nl:
            line += nl
            col = len(s) - s.rfind("\n")
        else:
            col += len(s)
        pos = m.end()
    toks.append(Tok("eof", "", line, col))
    return toks


# --------------------------------------------------------------------------
# parser

class _Parser:
    def __init__(self, text: str):
        self.toks = tokenize(text)
        self.i = 0

    # helpers
    def peek(self, k: int = 0) -> Tok:
        return self.toks[min(self.i + k, len(self.toks) - 1)]

    def next(self) -> Tok:
        t = self.toks[self.i]
        self.i = min(self.i + 1, len(self.toks) - 1)
        return t

    def err(self, tok: Tok, msg: str):
        raise ParseError(tok.line, tok.col, msg)

    def expect(self, text: str) -> Tok:
        t = self.next()
        if t.text != text:
            self.err(t, f"expected '{text}', found '{t.text or '<eof>'}'")
        return t

    def accept(self, text: str) -> bool:
        if self.peek().text == text:
            self.next()
            return True
        return False

    def int_(self) -> int:
        t = self.next()
        if t.kind != "number" or not re.fullmatch(r"-?\d+", t.text):
            self.err(t, f"expected integer, found '{t.text}'")
        return int(t.text)

    # types
    def dtype(self) -> str:
        t = self.next()
        if t.kind != "ident" or t.text not in DTYPES:
            self.err(t, f"expected data type, found '{t.text}'")
        return t.text

    def type_(self) -> TensorType:
        t = self.peek()
        if t.text == "<":
            self.next()
            dims: List[int] = []
            while True:
                u = self.peek()
                if u.kind == "ident" and u.text in DTYPES:
                    dt = self.dtype()
                    break
                d = self.int_()
                if d < 1:
                    self.err(u, "tensor dimensions must be >= 1")
                dims.append(d)
                self.expect("x")
            self.expect(">")
            return TensorType(tuple(dims), dt)
        return TensorType((), self.dtype())

    def type_list(self) -> Tuple[List[TensorType], bool]:
        if self.peek().text == "(":
            self.next()
            tys: List[TensorType] = []
            if not self.accept(")"):
                while True:
                    tys.append(self.type_())
                    if self.accept(")"):
                        break
                    self.expect(",")
            return tys, True
        return [self.type_()], False

    # operands
    def operand(self) -> Operand:
        t = self.next()
        if t.kind == "local":
            self.expect(":")
            ty = self.type_()
            return Operand("value", ty, name=t.text[1:], line=t.line, col=t.col)
        if t.kind == "number" or (t.kind == "ident" and t.text in ("true", "false")):
            self.expect(":")
            ty = self.type_()
            if t.kind == "ident":
                if ty.dtype != "bool":
                    self.err(t, "boolean literal must have type bool")
                val = 1.0 if t.text == "true" else 0.0
            else:
                val = float(t.text)
            return Operand("literal", ty, literal=val, line=t.line, col=t.col)
        self.err(t, f"expected operand, found '{t.text or '<eof>'}'")

    def inst(self) -> Inst:
        t = self.peek()
        result = None
        if t.kind == "local":
            self.next()
            result = t.text[1:]
            self.expect("=")
        op = self.next()
        if op.kind != "ident" or op.text not in OPCODES:
            self.err(op, f"unknown opcode '{op.text}'")
        name = op.text
        attrs: Dict[str, object] = {}
        if name in UNARY or name in ("transpose",):
            ops = [self.operand()]
        elif name in BINARY or name in COMPARE or name == "dot":
            a = self.operand()
            self.expect(",")
            ops = [a, self.operand()]
        elif name == "select":
            a = self.operand()
            self.expect(",")
            b = self.operand()
            self.expect(",")
            ops = [a, b, self.operand()]
        elif name == "reduce":
            ops = [self.operand()]
            self.expect("by")
            r = self.next()
            if r.text not in ("add", "multiply", "max"):  # max: extension (reading A26)
                self.err(r, f"unknown reduction '{r.text}'")
            self.expect("along")
            attrs = {"op": r.text, "axis": self.int_()}
        elif name == "shapeCast":
            ops = [self.operand()]
            self.expect("to")
            dims = [self.int_()]
            while self.peek().text == "x":
                self.next()
                dims.append(self.int_())
            attrs = {"shape": tuple(dims)}
        elif name == "dataTypeCast":
            ops = [self.operand()]
            self.expect("to")
            attrs = {"dtype": self.dtype()}
        elif name == "slice":
            ops = [self.operand()]
            self.expect("from")
            f = self.int_()
            self.expect("upto")
            attrs = {"from": f, "upto": self.int_()}
        else:  # pragma: no cover
            self.err(op, f"unknown opcode '{name}'")
        if result is None:
            self.err(op, "instruction result must be named")
        return Inst(result, name, ops, attrs, line=t.line, col=t.col)

    def attr(self) -> GradConfig:
        lb = self.expect("[")
        self.expect("gradient")
        src = self.next()
        if src.kind != "global":
            self.err(src, "expected function name after 'gradient'")
        cfg = GradConfig(src.text[1:], line=lb.line, col=lb.col)
        seen = set()
        while not self.accept("]"):
            k = self.next()
            if k.text in seen:
                self.err(k, f"duplicate '{k.text}' in gradient attribute")
            seen.add(k.text)
            if k.text == "wrt":
                cfg.wrt = self.int_list()
            elif k.text == "keeping":
                cfg.keeping = self.int_list()
            elif k.text == "from":
                cfg.from_ = self.int_()
            elif k.text == "seedable":
                cfg.seedable = True
            else:
                self.err(k, f"unexpected '{k.text}' in gradient attribute")
        return cfg

    def int_list(self) -> List[int]:
        xs = [self.int_()]
        while self.accept(","):
            xs.append(self.int_())
        return xs

    def function(self, grad: Optional[GradConfig]) -> Function:
        ft = self.expect("func")
        nm = self.next()
        if nm.kind != "global":
            self.err(nm, "expected function name")
        self.expect(":")
        params, _ = self.type_list()
        self.expect("->")
        results, is_tuple = self.type_list()
        fn = Function(nm.text[1:], params, results, is_tuple, gradient=grad,
                      line=ft.line, col=ft.col)
        if self.peek().text != "{":
            return fn
        self.next()
        lab = self.next()
        if lab.kind != "label":
            self.err(lab, "expected basic block label")
        fn.label = lab.text[1:]
        self.expect("(")
        if not self.accept(")"):
            while True:
                p = self.next()
                if p.kind != "local":
                    self.err(p, "expected block argument")
                self.expect(":")
                fn.param_names.append(p.text[1:])
                fn.arg_types.append(self.type_())
                fn.arg_locs.append((p.line, p.col))
                if self.accept(")"):
                    break
                self.expect(",")
        self.expect(":")
        while True:
            t = self.peek()
            if t.text == "return":
                self.next()
                fn.ret_line = t.line
                if self.peek().text == "(":
                    self.next()
                    if not self.accept(")"):
                        while True:
                            fn.ret.append(self.operand())
                            if self.accept(")"):
                                break
                            self.expect(",")
                elif self.peek().text != "}":
                    fn.ret.append(self.operand())
                break
            if t.text == "}" or t.kind == "eof":
                self.err(t, "basic block must end with 'return'")
            if t.kind == "label":
                self.err(t, "multiple basic blocks are not supported (straight-line only)")
            fn.insts.append(self.inst())
        self.expect("}")
        return fn

    def module(self) -> Module:
        self.expect("module")
        nm = self.next()
        if nm.kind != "string":
            self.err(nm, "expected module name string")
        self.expect("stage")
        st = self.next()
        if st.text not in ("raw", "optimizable"):
            self.err(st, f"unknown stage '{st.text}'")
        mod = Module(nm.text[1:-1], st.text, {})
        while self.peek().kind != "eof":
            grad = None
            if self.peek().text == "[":
                grad = self.attr()
            t = self.peek()
            fn = self.function(grad)
            if fn.name in mod.functions:
                raise ParseError(t.line, t.col, f"redefinition of function @{fn.name}")
            mod.functions[fn.name] = fn
        return mod


def parse(text: str) -> Module:
    """Parse a `.dl` module (raises ParseError) and verify it (raises
    VerifyError); returns the module with every function's body typed."""
    from .infer import infer_module
    mod = _Parser(text).module()
    infer_module(mod)
    return mod


def print_function(fn: Function, types: Dict[str, TensorType]) -> str:
    def tl(tys, tup):
        s = ", ".join(str(t) for t in tys)
        return f"({s})" if tup else s
    out = [f"func @{fn.name}: ({', '.join(str(t) for t in fn.param_types)}) -> "
           f"{tl(fn.result_types, fn.result_is_tuple)}"]
    if fn.has_body:
        out[0] += " {"
        args = ", ".join(f"%{n}: {t}" for n, t in zip(fn.param_names, fn.param_types))
        out.append(f"'{fn.label}({args}):")
        for ins in fn.insts:
            out.append("    " + str(ins))
        rets = ", ".join(str(o) for o in fn.ret)
        out.append("    return " + (f"({rets})" if len(fn.ret) > 1 else rets))
        out.append("}")
    return "\n".join(out)
