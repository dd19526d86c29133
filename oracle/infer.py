"""Oracle type / shape inference and verification (test infrastructure only).

One rule per opcode, Table 1 and S:L224-232:
  * element-wise unary: same type
  * element-wise binary / compare / select: broadcast shape      (P:L213,
    "All element-wise binary operators support broadcasting"; reading A1:
    right-aligned, each pair equal or one of them 1, missing leading dims
    are 1); compare yields bool (Table 1 `gt` row P:L176)
  * dot: rank-2 [m,k].[k,n] -> [m,n], equal dtypes               (A19)
  * reduce ... along d: axis removed                             (A2)
  * transpose: all axes reversed                                 (A3)
  * shapeCast: element count preserved
  * dataTypeCast: shape preserved
  * slice from a upto b: axis-0 half-open
Gradient declarations (Fig. 3): expected type =
source params (+ seed of the selected output's type if `seedable`, appended
last) -> grads in `wrt` order then `keeping` outputs; singleton collapses
(reading A7; Fig. 4).
"""

from __future__ import annotations

from typing import Dict, List, Optional, Tuple

from .ir import (BINARY, COMPARE, FLOAT_DTYPES, UNARY, Function, Inst, Module,
                 Operand, TensorType, VerifyError)


def broadcast_shapes(a: Tuple[int, ...], b: Tuple[int, ...]) -> Tuple[int, ...]:
    """Reading A1 (Table 1).  Raises ValueError if the shapes
    are incompatible."""
    n = max(len(a), len(b))
    pa = (1,) * (n - len(a)) + tuple(a)
    pb = (1,) * (n - len(b)) + tuple(b)
    out = []
    for x, y in zip(pa, pb):
        if x == y or y == 1:
            out.append(x)
        elif x == 1:
            out.append(y)
        else:
            raise ValueError(f"shapes {a} and {b} are not broadcast-compatible")
    return tuple(out)


def _numel(shape) -> int:
    n = 1
    for d in shape:
        n *= d
    return n


def infer_inst(ins: Inst, tys: List[TensorType]) -> TensorType:
    """Result type of one instruction from its operand types (raises
    VerifyError at the instruction's location)."""
    op = ins.opcode

    def fail(msg):
        raise VerifyError(ins.line, ins.col, f"'{op}': {msg}")

    def bcast(*shapes):
        s = shapes[0]
        try:
            for t in shapes[1:]:
                s = broadcast_shapes(s, t)
        except ValueError as e:
            fail(str(e))
        return s

    if op in UNARY:
        (a,) = tys
        if a.dtype == "bool":
            fail("operand must be numeric")
        if op in ("tanh", "exp", "log", "sqrt") and a.dtype not in FLOAT_DTYPES:
            fail("operand must have a floating-point type")
        return a
    if op in BINARY:
        a, b = tys
        if a.dtype != b.dtype:
            fail(f"operand data types differ ({a.dtype} vs {b.dtype})")
        if a.dtype == "bool":
            fail("operands must be numeric")
        if op == "power" and a.dtype not in FLOAT_DTYPES:
            fail("operands must have a floating-point type")
        return TensorType(bcast(a.shape, b.shape), a.dtype)
    if op in COMPARE:
        a, b = tys
        if a.dtype != b.dtype:
            fail(f"operand data types differ ({a.dtype} vs {b.dtype})")
        return TensorType(bcast(a.shape, b.shape), "bool")
    if op == "select":
        c, a, b = tys
        if c.dtype != "bool":
            fail("condition must have type bool")
        if a.dtype != b.dtype:
            fail(f"branch data types differ ({a.dtype} vs {b.dtype})")
        return TensorType(bcast(c.shape, a.shape, b.shape), a.dtype)
    if op == "dot":
        a, b = tys
        if a.rank != 2 or b.rank != 2:
            fail("operands must be rank 2")
        if a.shape[1] != b.shape[0]:
            fail(f"inner dimensions differ ({a.shape[1]} vs {b.shape[0]})")
        if a.dtype != b.dtype:
            fail(f"operand data types differ ({a.dtype} vs {b.dtype})")
        if a.dtype == "bool":
            fail("operands must be numeric")
        return TensorType((a.shape[0], b.shape[1]), a.dtype)
    if op == "reduce":
        (a,) = tys
        d = ins.attrs["axis"]
        if a.rank == 0 or not (0 <= d < a.rank):
            fail(f"axis {d} out of range for rank {a.rank}")
        if a.dtype == "bool":
            fail("operand must be numeric")
        return TensorType(a.shape[:d] + a.shape[d + 1:], a.dtype)
    if op == "transpose":
        (a,) = tys
        return TensorType(tuple(reversed(a.shape)), a.dtype)
    if op == "shapeCast":
        (a,) = tys
        s = tuple(ins.attrs["shape"])
        if _numel(s) != _numel(a.shape):
            fail(f"element count differs ({_numel(a.shape)} vs {_numel(s)})")
        return TensorType(s, a.dtype)
    if op == "dataTypeCast":
        (a,) = tys
        return TensorType(a.shape, ins.attrs["dtype"])
    if op == "slice":
        (a,) = tys
        f, u = ins.attrs["from"], ins.attrs["upto"]
        if a.rank == 0 or not (0 <= f < u <= a.shape[0]):
            fail(f"bounds [{f}, {u}) out of range")
        return TensorType((u - f,) + a.shape[1:], a.dtype)
    fail("unknown opcode")  # pragma: no cover


def infer_function(fn: Function) -> None:
    """Types every value of a function body, in program order (single block:
    program order is dominance).  Fills `fn.types`."""
    if not fn.has_body:
        return
    if len(fn.arg_types) != len(fn.param_types):
        raise VerifyError(fn.line, fn.col,
                          f"entry block has {len(fn.arg_types)} arguments, "
                          f"function type has {len(fn.param_types)}")
    types: Dict[str, TensorType] = {}
    for name, ty, pty, (ln, cl) in zip(fn.param_names, fn.arg_types,
                                        fn.param_types, fn.arg_locs):
        if ty != pty:
            raise VerifyError(ln, cl, f"argument %{name} has type {ty}, "
                                      f"function type says {pty}")
        if name in types:
            raise VerifyError(ln, cl, f"redefinition of %{name}")
        types[name] = ty

    def operand_type(o: Operand) -> TensorType:
        if o.kind == "literal":
            return o.type
        if o.name not in types:
            raise VerifyError(o.line, o.col, f"use of undefined value %{o.name}")
        if types[o.name] != o.type:
            raise VerifyError(o.line, o.col, f"%{o.name} has type {types[o.name]}, "
                                             f"annotated {o.type}")
        return o.type

    for ins in fn.insts:
        tys = [operand_type(o) for o in ins.operands]
        rt = infer_inst(ins, tys)
        if ins.result in types:
            raise VerifyError(ins.line, ins.col, f"redefinition of %{ins.result}")
        types[ins.result] = rt
    rts = [operand_type(o) for o in fn.ret]
    if rts != list(fn.result_types):
        raise VerifyError(fn.ret_line, 1, "return type does not match function type")
    fn.types = types


def _is_float(t: TensorType) -> bool:
    return t.dtype in FLOAT_DTYPES


def expected_gradient_type(src: Function, cfg) -> Tuple[List[TensorType], List[TensorType]]:
    """(params, results) of a gradient declaration (Fig. 3 P:L262-272,
    reading A7).  Raises VerifyError on a bad configuration."""
    def fail(msg):
        raise VerifyError(cfg.line, cfg.col, msg)

    n_in, n_out = len(src.param_types), len(src.result_types)
    wrt = list(range(n_in)) if cfg.wrt is None else list(cfg.wrt)
    if len(set(wrt)) != len(wrt):
        fail("duplicate index in 'wrt'")
    if len(set(cfg.keeping)) != len(cfg.keeping):
        fail("duplicate index in 'keeping'")
    for i in wrt:
        if not 0 <= i < n_in:
            fail(f"'wrt' index {i} out of range")
        if not _is_float(src.param_types[i]):
            fail(f"argument {i} has non-differentiable type {src.param_types[i]}")
    for j in cfg.keeping:
        if not 0 <= j < n_out:
            fail(f"'keeping' index {j} out of range")
    frm = 0 if cfg.from_ is None else cfg.from_
    if not 0 <= frm < n_out:
        fail(f"'from' index {frm} out of range")
    if not _is_float(src.result_types[frm]):
        fail(f"output {frm} has non-differentiable type {src.result_types[frm]}")
    params = list(src.param_types) + ([src.result_types[frm]] if cfg.seedable else [])
    results = [src.param_types[i] for i in wrt] + [src.result_types[j] for j in cfg.keeping]
    return params, results


def check_differentiable(src: Function, cfg) -> None:
    """Every active instruction (float result depending on a `wrt` argument)
    must have an adjoint rule; reduce-by-multiply has none."""
    wrt = set(range(len(src.param_types)) if cfg.wrt is None else cfg.wrt)
    active = {src.param_names[i] for i in wrt}
    for ins in src.insts:
        rt = src.types[ins.result]
        if not _is_float(rt):
            continue
        if any(o.kind == "value" and o.name in active for o in ins.operands):
            if ins.opcode == "reduce" and ins.attrs["op"] == "multiply":
                raise VerifyError(ins.line, ins.col,
                                  "'reduce by multiply' is not differentiable")
            if ins.opcode == "dataTypeCast" and not _is_float(
                    src.types.get(ins.operands[0].name, rt)):
                continue
            active.add(ins.result)


def infer_module(mod: Module) -> None:
    """Types every defined function, then checks every gradient declaration
    against its source (declared type == expected type)."""
    for fn in mod.functions.values():
        if fn.gradient is None and not fn.has_body:
            raise VerifyError(fn.line, fn.col,
                              f"function @{fn.name} has no body and no gradient attribute")
        infer_function(fn)
    for fn in mod.functions.values():
        cfg = fn.gradient
        if cfg is None:
            continue
        if fn.has_body:
            raise VerifyError(fn.line, fn.col, "a gradient declaration has no body")
        src = mod.functions.get(cfg.source)
        if src is None:
            raise VerifyError(cfg.line, cfg.col, f"unknown function @{cfg.source}")
        if not src.has_body:
            # higher order: the source is itself a gradient
            # declaration; differentiate its canonical body (adjoint.py)
            from .adjoint import canonical
            src = canonical(mod, cfg.source, (fn.name,))
        params, results = expected_gradient_type(src, cfg)
        if list(fn.param_types) != params or list(fn.result_types) != results:
            raise VerifyError(fn.line, fn.col,
                              f"declared type of @{fn.name} does not match the "
                              "expected gradient type")
        check_differentiable(src, cfg)
