"""Oracle interpreter: evaluates each instruction's mathematical definition
in program order, in numpy float64 (test infrastructure only).

Op definitions (Table 1):
  negate/tanh/exp/log/sqrt/abs/sign  pointwise; sign(0) = 0
  add/subtract/multiply/divide/power pointwise after broadcasting (A1)
  lt/le/gt/ge/eq/ne                  pointwise -> bool
  select(c, a, b)                    where(c, a, b) after broadcasting
  dot(a, b)                          a @ b, rank 2
  reduce(a, add|multiply|max, d)     sum / prod / max over axis d (axis removed, A2;
                                     max: extension, reading A26)
  transpose(a)                       all axes reversed (A3)
  shapeCast(a, s)                    row-major reshape
  dataTypeCast(a, t)                 value conversion (floats stay float64)
  slice(a, f, u)                     a[f:u] on axis 0
All floating-point values are float64 regardless of their IR dtype (the
oracle is the exact-arithmetic stand-in; the paper fixes no precision).

dot_policy="bf16" (reading A15 of SURVEY.md §8(c), not from the paper, which
has no bf16): every `dot` operand is first rounded to the nearest bf16 value
(round-to-nearest-even), then multiplied and summed in float64.  This is the
definition of the GPU's bf16-dot execution policy written out; the parity
tests use it for network-level checks where the unrounded comparison is
ill-conditioned (ReLU's derivative jumps at 0).
"""

from __future__ import annotations

from typing import Dict, List, Sequence

import numpy as np

from .ir import FLOAT_DTYPES, Function, Inst, Module, Operand, TensorType


def np_dtype(t: TensorType):
    if t.dtype == "bool":
        return np.bool_
    if t.dtype in FLOAT_DTYPES:
        return np.float64
    return np.int64


def as_value(x, t: TensorType) -> np.ndarray:
    a = np.asarray(x, dtype=np_dtype(t))
    if a.shape != tuple(t.shape):
        raise ValueError(f"input shape {a.shape} does not match type {t}")
    return a


def literal_value(o: Operand) -> np.ndarray:
    return np.full(o.type.shape, o.literal, dtype=np_dtype(o.type))


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Nearest bf16 value of each float (RNE on the float32 bit pattern after
    the float64 -> float32 rounding; NaN/inf pass through)."""
    f = np.asarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    out = r.astype(np.uint32).view(np.float32).astype(np.float64)
    return np.where(np.isfinite(f), out, f.astype(np.float64))


def eval_inst(ins: Inst, args: List[np.ndarray], rt: TensorType, dot_policy=None) -> np.ndarray:
    op = ins.opcode
    if op == "negate":
        r = -args[0]
    elif op == "tanh":
        r = np.tanh(args[0])
    elif op == "exp":
        r = np.exp(args[0])
    elif op == "log":
        r = np.log(args[0])
    elif op == "sqrt":
        r = np.sqrt(args[0])
    elif op == "abs":
        r = np.abs(args[0])
    elif op == "sign":
        r = np.sign(args[0])
    elif op == "add":
        r = args[0] + args[1]
    elif op == "subtract":
        r = args[0] - args[1]
    elif op == "multiply":
        r = args[0] * args[1]
    elif op == "divide":
        r = args[0] / args[1]
    elif op == "power":
        r = np.power(args[0], args[1])
    elif op == "lt":
        r = args[0] < args[1]
    elif op == "le":
        r = args[0] <= args[1]
    elif op == "gt":
        r = args[0] > args[1]
    elif op == "ge":
        r = args[0] >= args[1]
    elif op == "eq":
        r = args[0] == args[1]
    elif op == "ne":
        r = args[0] != args[1]
    elif op == "select":
        r = np.where(args[0], args[1], args[2])
    elif op == "dot":
        if dot_policy == "bf16":
            r = bf16_round(args[0]) @ bf16_round(args[1])
        else:
            r = args[0] @ args[1]
    elif op == "reduce":
        f = {"add": np.sum, "multiply": np.prod, "max": np.max}[ins.attrs["op"]]
        r = f(args[0], axis=ins.attrs["axis"])
    elif op == "transpose":
        r = np.transpose(args[0], tuple(reversed(range(args[0].ndim))))
    elif op == "shapeCast":
        r = np.reshape(args[0], ins.attrs["shape"])
    elif op == "dataTypeCast":
        r = args[0].astype(np_dtype(rt))
    elif op == "slice":
        r = args[0][ins.attrs["from"]:ins.attrs["upto"]]
    else:  # pragma: no cover
        raise NotImplementedError(op)
    r = np.asarray(r, dtype=np_dtype(rt))
    # the inferred static type must equal the runtime shape
    assert r.shape == tuple(rt.shape), (ins.opcode, r.shape, rt)
    return r


def evaluate(fn: Function, inputs: Sequence, dot_policy=None) -> Dict[str, np.ndarray]:
    """All SSA values of one execution of `fn`, keyed by name."""
    if len(inputs) != len(fn.param_types):
        raise ValueError(f"@{fn.name} takes {len(fn.param_types)} inputs, got {len(inputs)}")
    env: Dict[str, np.ndarray] = {}
    for name, t, x in zip(fn.param_names, fn.param_types, inputs):
        env[name] = as_value(x, t)

    def val(o: Operand):
        return literal_value(o) if o.kind == "literal" else env[o.name]

    for ins in fn.insts:
        env[ins.result] = eval_inst(ins, [val(o) for o in ins.operands], fn.types[ins.result], dot_policy)
    return env


def run_function(fn: Function, inputs: Sequence, dot_policy=None) -> List[np.ndarray]:
    env = evaluate(fn, inputs, dot_policy)
    return [literal_value(o) if o.kind == "literal" else env[o.name] for o in fn.ret]


def run(mod: Module, name: str, inputs: Sequence, dot_policy=None) -> List[np.ndarray]:
    """Runs a defined function, or the result a gradient declaration denotes."""
    fn = mod.functions[name]
    if fn.gradient is not None:
        from .vjp import grad_function
        return grad_function(mod, fn, inputs, dot_policy)
    return run_function(fn, inputs, dot_policy)
