"""Oracle adjoint code generation: the IR a gradient declaration canonicalises
to (test infrastructure only; shares no code with the CUDA path).

PAPER.md §3.1.3: "The differentiation pass ... canonicalizes every
gradient declaration in the module to a normal function definition with
basic blocks and instructions.  The canonicalization process first copies
basic blocks and instructions from the original function to the new
function body, and then applies adjoint code generation to the function."
L311-312: "This approach also makes higher-order differentiation possible;
this can be accomplished by declaring a higher-order gradient function that
differentiates the original gradient function" (Fig. 4 `d2g_dw2`, L367-370).

`canonical(mod, name)` returns a function WITH a body for any function of
the module: a definition as written, or a gradient declaration turned into
IR by the steps above (recursively, so a declaration of a declaration is a
second-order gradient).  The adjoint rules are the vector-Jacobian rules of
vjp.py (rule table) written as IR instructions; multi-use adjoints
are summed with `add`; every element-wise contribution is unbroadcast with
`reduce ... by add` over the broadcast axes then `shapeCast`.
Only values that depend on a `wrt` argument get adjoints (forward activity).
The emitted text is parsed and typed by the oracle's own parser/inference,
so every generated instruction is verified against Table 1's typing rules.

No dead-code elimination: the oracle keeps every copied primal instruction
(values are the same either way).
"""

from __future__ import annotations

from typing import Dict, List, Optional, Sequence

from .infer import infer_inst
from .ir import COMPARE, FLOAT_DTYPES, Function, Inst, Module, Operand, TensorType, VerifyError


class _Gen:
    """Emits instructions as text, typing each with infer_inst (Table 1)."""

    def __init__(self, used: Sequence[str]):
        self.used = set(used)
        self.lines: List[str] = []
        self.k = 0

    def fresh(self, stem: str = "a") -> str:
        while True:
            n = f"{stem}{self.k}"
            self.k += 1
            if n not in self.used:
                self.used.add(n)
                return n

    def emit(self, opcode: str, ops: List[Operand], attrs: Optional[dict] = None) -> Operand:
        ins = Inst(self.fresh(), opcode, list(ops), dict(attrs or {}))
        rt = infer_inst(ins, [o.type for o in ops])
        self.lines.append("    " + str(ins))
        return Operand("value", rt, name=ins.result)


def _lit(v: float, t: TensorType) -> Operand:
    return Operand("literal", t, literal=float(v))


def _scalar(t: TensorType) -> TensorType:
    return TensorType((), t.dtype)


def _unbroadcast(G: _Gen, c: Operand, t: TensorType) -> Operand:
    """Sum contribution c over the axes broadcasting expanded, back to t."""
    cs, ts = c.type.shape, t.shape
    if cs == ts:
        return c
    extra = len(cs) - len(ts)
    axes = list(range(extra)) + [i + extra for i, d in enumerate(ts) if d == 1 and cs[i + extra] != 1]
    for ax in sorted(axes, reverse=True):  # highest first: lower indices stay valid
        c = G.emit("reduce", [c], {"op": "add", "axis": ax})
    if c.type.shape != ts:
        if ts:
            c = G.emit("shapeCast", [c], {"shape": tuple(ts)})
        else:  # rank 0 target: sum the remaining unit axes away
            while c.type.shape:
                c = G.emit("reduce", [c], {"op": "add", "axis": len(c.type.shape) - 1})
    return c


def _rules(G: _Gen, ins: Inst, g: Operand, y: Operand, ops: List[Operand], active) -> List[tuple]:
    """(operand index, contribution) pairs: the VJP rules of vjp.vjp_rule as IR."""
    op = ins.opcode
    one = lambda: _lit(1.0, _scalar(y.type))
    act = lambda i: ops[i].kind == "value" and active(ops[i].name)
    E = G.emit
    if op == "add":
        return [(0, g), (1, g)]
    if op == "subtract":
        return [(0, g)] + ([(1, E("negate", [g]))] if act(1) else [])
    if op == "multiply":
        out = []
        if act(0):
            out.append((0, E("multiply", [g, ops[1]])))
        if act(1):
            out.append((1, E("multiply", [g, ops[0]])))
        return out
    if op == "divide":
        a, b = ops
        out = []
        if act(0):
            out.append((0, E("divide", [g, b])))
        if act(1):
            num = E("multiply", [g, a])
            den = E("multiply", [b, b])
            out.append((1, E("negate", [E("divide", [num, den])])))
        return out
    if op == "power":
        a, n = ops
        out = []
        if act(0):
            nm1 = _lit(n.literal - 1.0, n.type) if n.kind == "literal" else E("subtract", [n, one()])
            out.append((0, E("multiply", [g, E("multiply", [n, E("power", [a, nm1])])])))
        if act(1):
            out.append((1, E("multiply", [g, E("multiply", [y, E("log", [a])])])))
        return out
    if op == "negate":
        return [(0, E("negate", [g]))]
    if op == "tanh":
        return [(0, E("multiply", [g, E("subtract", [one(), E("multiply", [y, y])])]))]
    if op == "exp":
        return [(0, E("multiply", [g, y]))]
    if op == "log":
        return [(0, E("divide", [g, ops[0]]))]
    if op == "sqrt":
        return [(0, E("divide", [g, E("multiply", [_lit(2.0, _scalar(y.type)), y])]))]
    if op == "abs":
        return [(0, E("multiply", [g, E("sign", [ops[0]])]))]
    if op == "sign" or op in COMPARE:
        return []
    if op == "select":
        c = ops[0]
        zero = _lit(0.0, _scalar(y.type))
        out = []
        if act(1):
            out.append((1, E("select", [c, g, zero])))
        if act(2):
            out.append((2, E("select", [c, zero, g])))
        return out
    if op == "dot":
        a, b = ops
        out = []
        if act(0):
            out.append((0, E("dot", [g, E("transpose", [b])])))
        if act(1):
            out.append((1, E("dot", [E("transpose", [a]), g])))
        return out
    if op == "transpose":
        return [(0, E("transpose", [g]))]
    if op == "reduce" and ins.attrs["op"] == "max":
        # reading A26: g / (number of tied maxima) at every position equal to the max
        a = ops[0]
        keep = list(a.type.shape)
        keep[ins.attrs["axis"]] = 1
        yk = E("shapeCast", [y], {"shape": tuple(keep)})
        at = E("eq", [a, yk])
        cnt = E("reduce", [E("dataTypeCast", [at], {"dtype": a.type.dtype})], {"op": "add", "axis": ins.attrs["axis"]})
        q = E("divide", [E("shapeCast", [g], {"shape": tuple(keep)}), E("shapeCast", [cnt], {"shape": tuple(keep)})])
        return [(0, E("select", [at, q, _lit(0.0, _scalar(a.type))]))]
    if op == "reduce":
        if ins.attrs["op"] != "add":
            raise VerifyError(ins.line, ins.col, "'reduce by multiply' is not differentiable")
        a = ops[0]
        keep = list(a.type.shape)
        keep[ins.attrs["axis"]] = 1
        e = E("shapeCast", [g], {"shape": tuple(keep)})
        return [(0, E("multiply", [e, _lit(1.0, a.type)]))]  # broadcast back along the axis
    if op == "shapeCast":
        a = ops[0]
        if a.type.shape:
            return [(0, E("shapeCast", [g], {"shape": tuple(a.type.shape)}))]
        return [(0, _unbroadcast(G, g, a.type))]
    if op == "dataTypeCast":
        a = ops[0]
        if a.type.dtype not in FLOAT_DTYPES:
            return []
        return [(0, g if g.type.dtype == a.type.dtype else E("dataTypeCast", [g], {"dtype": a.type.dtype}))]
    raise VerifyError(ins.line, ins.col, f"no adjoint rule for '{op}'")


def adjoint_text(src: Function, cfg, name: str) -> str:
    """IR text of the gradient function `name` of `src` (which has a body)."""
    n_in = len(src.param_types)
    wrt = list(range(n_in)) if cfg.wrt is None else list(cfg.wrt)
    frm = 0 if cfg.from_ is None else cfg.from_
    G = _Gen(list(src.param_names) + list(src.types))
    params = list(zip(src.param_names, src.param_types))
    seed_name = None
    if cfg.seedable:
        seed_name = "seed"
        k = 0
        while seed_name in G.used:
            seed_name = f"seed{k}"
            k += 1
        G.used.add(seed_name)
        params.append((seed_name, src.result_types[frm]))
    # 1. copy the primal body (L296)
    G.lines += ["    " + str(ins) for ins in src.insts]
    # forward activity
    active = {src.param_names[i] for i in wrt}
    for ins in src.insts:
        if src.types[ins.result].dtype in FLOAT_DTYPES and any(
                o.kind == "value" and o.name in active for o in ins.operands):
            active.add(ins.result)
    is_active = lambda n: n in active and src.types[n].dtype in FLOAT_DTYPES
    # 2. adjoint code generation in reverse program order
    adj: Dict[str, Operand] = {}

    def acc(target: Operand, c: Operand):
        if target.kind != "value" or not is_active(target.name):
            return
        c = _unbroadcast(G, c, src.types[target.name])
        adj[target.name] = G.emit("add", [adj[target.name], c]) if target.name in adj else c

    out = src.ret[frm]
    if out.kind == "value":
        t = src.types[out.name]
        acc(out, Operand("value", t, name=seed_name) if seed_name else _lit(1.0, t))
    for ins in reversed(src.insts):
        if ins.result not in adj:
            continue
        y = Operand("value", src.types[ins.result], name=ins.result)
        ops = [Operand("value", src.types[o.name], name=o.name) if o.kind == "value" else o
               for o in ins.operands]
        for idx, c in _rules(G, ins, adj[ins.result], y, ops, is_active):
            acc(ops[idx], c)
    # 3. results: grads in wrt order, then kept outputs (reading A7)
    rets = [adj.get(src.param_names[i], _lit(0.0, src.param_types[i])) for i in wrt]
    rets += [src.ret[j] for j in cfg.keeping]
    r_types = [src.param_types[i] for i in wrt] + [src.result_types[j] for j in cfg.keeping]
    tup = len(r_types) > 1
    rt = ", ".join(str(t) for t in r_types)
    head = (f"func @{name}: ({', '.join(str(t) for _, t in params)}) -> " + (f"({rt})" if tup else rt) + " {\n"
            + "'entry(" + ", ".join(f"%{n}: {t}" for n, t in params) + "):\n")
    ret = ", ".join(str(o) for o in rets)
    return head + "\n".join(G.lines) + ("\n" if G.lines else "") + (
        f"    return ({ret})\n" if tup else f"    return {ret}\n") + "}\n"


def canonical(mod: Module, name: str, _stack=()) -> Function:
    """The function `name` with a body: as written, or its gradient
    declaration canonicalised (recursively for higher order)."""
    fn = mod.functions[name]
    if fn.has_body:
        return fn
    cfg = fn.gradient
    if cfg is None:
        raise VerifyError(fn.line, fn.col, f"function @{name} has no body and no gradient attribute")
    if name in _stack:
        raise VerifyError(cfg.line, cfg.col, f"cyclic gradient declaration @{name}")
    if cfg.source not in mod.functions:
        raise VerifyError(cfg.line, cfg.col, f"unknown function @{cfg.source}")
    src = canonical(mod, cfg.source, _stack + (name,))
    from .ir import parse
    text = f'module "adjoint"\nstage optimizable\n\n' + adjoint_text(src, cfg, name)
    return parse(text).functions[name]
