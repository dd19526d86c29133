"""Oracle gradient: the result a gradient declaration denotes, computed by a
plain value-level reverse sweep (test infrastructure only).

Definition (§3.1.3; readings A6, A7 of SURVEY.md §8(c)): for
`[gradient @f wrt W keeping K from o seedable]`, the result is
    ( (seed^T J_{f_o}(x))_i  for i in W ,  f_j(x) for j in K )
with seed = the extra last argument if `seedable`, else all-ones of the type
of output o.  The reverse sweep visits instructions in reverse program order
("backward direction ... top-down traversal"), applying one
vector-Jacobian rule per opcode and summing contributions of
multi-use values; every element-wise contribution is unbroadcast to the
operand's shape.  float64 throughout.
"""

from __future__ import annotations

from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from .interp import bf16_round, evaluate, literal_value
from .ir import BINARY, COMPARE, FLOAT_DTYPES, Function, Inst, Module


def unbroadcast(c: np.ndarray, shape: Tuple[int, ...]) -> np.ndarray:
    """Sum `c` over the axes broadcasting expanded, back to `shape`
    (S:L344-352): leading extra axes, and axes where `shape` has extent 1."""
    c = np.asarray(c, dtype=np.float64)
    extra = c.ndim - len(shape)
    if extra > 0:
        c = c.sum(axis=tuple(range(extra)))
    axes = tuple(i for i, d in enumerate(shape) if d == 1 and c.shape[i] != 1)
    if axes:
        c = c.sum(axis=axes, keepdims=True)
    assert c.shape == tuple(shape), (c.shape, shape)
    return c


def vjp_rule(ins: Inst, g: np.ndarray, y: np.ndarray, args: List[np.ndarray], dot_policy=None
             ) -> List[Tuple[int, Optional[np.ndarray]]]:
    """Contributions (operand index, adjoint before unbroadcast) of one
    instruction, given its incoming adjoint g, result y and operand values.
    Rule table S:L338."""
    op = ins.opcode
    if op == "add":
        return [(0, g), (1, g)]
    if op == "subtract":
        return [(0, g), (1, -g)]
    if op == "multiply":
        return [(0, g * args[1]), (1, g * args[0])]
    if op == "divide":
        a, b = args
        return [(0, g / b), (1, -g * a / (b * b))]
    if op == "power":
        a, n = args
        out = [(0, g * n * np.power(a, n - 1))]
        if ins.operands[1].kind == "value":
            out.append((1, g * y * np.log(a)))
        return out
    if op == "negate":
        return [(0, -g)]
    if op == "tanh":
        return [(0, g * (1.0 - y * y))]
    if op == "exp":
        return [(0, g * y)]
    if op == "log":
        return [(0, g / args[0])]
    if op == "sqrt":
        return [(0, g / (2.0 * y))]
    if op == "abs":
        return [(0, g * np.sign(args[0]))]
    if op == "sign":
        return [(0, np.zeros_like(args[0], dtype=np.float64))]
    if op == "select":
        c = args[0]
        return [(1, np.where(c, g, 0.0)), (2, np.where(c, 0.0, g))]
    if op in COMPARE:
        return []
    if op == "dot":
        a, b = args
        if dot_policy == "bf16":  # the adjoint dots round their operands too (reading A15)
            a, b, g = bf16_round(a), bf16_round(b), bf16_round(g)
        return [(0, g @ b.T), (1, a.T @ g)]
    if op == "transpose":
        return [(0, np.transpose(g, tuple(reversed(range(g.ndim)))))]
    if op == "reduce":
        d = ins.attrs["axis"]
        if ins.attrs["op"] == "max":
            # reading A26: the adjoint goes to the positions attaining the
            # max, split equally among ties (each of k tied positions gets g/k)
            x = args[0]
            at = x == np.expand_dims(y, d)
            k = at.sum(axis=d, keepdims=True)
            return [(0, np.where(at, np.expand_dims(g, d) / k, 0.0))]
        if ins.attrs["op"] != "add":
            raise ValueError("'reduce by multiply' is not differentiable")
        return [(0, np.broadcast_to(np.expand_dims(g, d), args[0].shape))]
    if op == "shapeCast":
        return [(0, np.reshape(g, args[0].shape))]
    if op == "dataTypeCast":
        return [(0, g)]
    if op == "slice":
        z = np.zeros(args[0].shape, dtype=np.float64)
        z[ins.attrs["from"]:ins.attrs["upto"]] = g
        return [(0, z)]
    raise NotImplementedError(op)  # pragma: no cover


def reverse_sweep(src: Function, env: Dict[str, np.ndarray], out_index: int,
                  seed: np.ndarray, dot_policy=None, wrt: Optional[Sequence[int]] = None) -> Dict[str, np.ndarray]:
    """Adjoints of every value that the selected output depends on.  With
    `wrt`, only values that depend on those arguments (forward activity, as
    adjoint.py does) get adjoints: the others never reach a `wrt` gradient,
    and may be computed by ops without a derivative rule (`reduce ... by
    multiply`; reading A24)."""
    adj: Dict[str, np.ndarray] = {}

    def is_float(name: str) -> bool:
        t = src.types[name]
        return t.dtype in FLOAT_DTYPES

    active = None
    if wrt is not None:
        active = {src.param_names[i] for i in wrt}
        for ins in src.insts:
            if is_float(ins.result) and any(o.kind == "value" and o.name in active for o in ins.operands):
                active.add(ins.result)

    def acc(name: str, c: np.ndarray):
        if active is not None and name not in active:
            return
        c = unbroadcast(c, src.types[name].shape)
        adj[name] = adj[name] + c if name in adj else c

    out = src.ret[out_index]
    if out.kind == "value":
        acc(out.name, np.asarray(seed, dtype=np.float64))
    for ins in reversed(src.insts):
        if ins.result not in adj:
            continue
        g = adj[ins.result]
        args = [literal_value(o) if o.kind == "literal" else env[o.name] for o in ins.operands]
        args = [a.astype(np.float64) if a.dtype != np.bool_ else a for a in args]
        for idx, c in vjp_rule(ins, g, env[ins.result], args, dot_policy):
            o = ins.operands[idx]
            if o.kind == "value" and is_float(o.name):
                acc(o.name, c)
    return adj


def grad(src: Function, inputs: Sequence, wrt: Optional[Sequence[int]] = None,
         keeping: Sequence[int] = (), from_: int = 0, seed=None, dot_policy=None) -> List[np.ndarray]:
    """Gradient result of `src` at `inputs` (reading A7 order: grads in `wrt`
    order, then kept outputs)."""
    env = evaluate(src, inputs, dot_policy)
    outs = [literal_value(o) if o.kind == "literal" else env[o.name] for o in src.ret]
    if seed is None:
        seed = np.ones(src.result_types[from_].shape, dtype=np.float64)
    seed = np.asarray(seed, dtype=np.float64).reshape(src.result_types[from_].shape)
    wrt = list(range(len(src.param_types))) if wrt is None else list(wrt)
    adj = reverse_sweep(src, env, from_, seed, dot_policy, wrt)
    res = []
    for i in wrt:
        n = src.param_names[i]
        res.append(adj[n] if n in adj else np.zeros(src.param_types[i].shape))
    res += [outs[j] for j in keeping]
    return res


def grad_function(mod: Module, gfn: Function, inputs: Sequence, dot_policy=None) -> List[np.ndarray]:
    """Runs a gradient declaration: inputs are the source's arguments, plus
    the seed last when `seedable` (Fig. 3 `@foo_grad_3`)."""
    cfg = gfn.gradient
    src = mod.functions[cfg.source]
    if not src.has_body:  # higher order: differentiate the generated gradient function
        from .adjoint import canonical
        src = canonical(mod, cfg.source)
    n = len(src.param_types)
    seed = inputs[n] if cfg.seedable else None
    return grad(src, list(inputs[:n]), cfg.wrt, cfg.keeping,
                0 if cfg.from_ is None else cfg.from_, seed, dot_policy)
