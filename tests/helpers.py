"""Shared test helpers: running a program through the C ABI (GPU), running
it through the oracle (CPU, f64), and the tolerances of SURVEY.md §8(c):
  A16  fp32 element-wise outputs: |g - r| <= 1e-5 |r| + 1e-5 * 1e-6 * max|r|
  A17  fp32 dot / reduce outputs: |g - r| <= 1e-5 * sum|terms|
  A18  bf16-dot policy: ||g - r||_F / ||r||_F <= 2e-2 per output tensor
sum|terms| is computed from the oracle's own float64 values of the operands
of the op that produces the output (|A|.|B| for dot, sum|x| for reduce).
"""

from __future__ import annotations

from typing import List, Optional, Sequence

import numpy as np

import oracle


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bf16, returned as float32 (test inputs that
    are exactly representable in bf16)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).reshape(x.shape)


def gpu_run(text: str, fn: str, grad: Optional[str], inputs: Sequence[np.ndarray], seed=None,
            dot_precision: str = "f32", flags: int = 0, which: str = "both", bf16_inputs=()):
    """Runs primal and/or gradient on cuda:0; returns numpy float64 arrays."""
    import torch
    import paper_1711_03016_b200 as P
    f = P.Function(text, fn, grad, dot_precision=dot_precision, flags=flags)
    dev = torch.device("cuda:0")
    ins = []
    for i, x in enumerate(inputs):
        t = torch.from_numpy(np.array(x, copy=True)).to(dev)  # keeps 0-d arrays 0-d (ascontiguousarray does not)
        if i in bf16_inputs:
            t = t.to(torch.bfloat16)
        ins.append(t)
    res = {}
    if which in ("both", "primal"):
        outs = f.run(ins)
        torch.cuda.synchronize()
        res["primal"] = [o.cpu().to(torch.float64).numpy() if o.dtype != torch.bool else o.cpu().numpy()
                         for o in outs]
    if which in ("both", "grad"):
        s = None if seed is None else torch.from_numpy(np.array(seed, dtype=np.float32)).to(dev)
        outs = f.grad_run(ins, seed=s)
        torch.cuda.synchronize()
        res["grad"] = [o.cpu().to(torch.float64).numpy() for o in outs]
    res["fn"] = f
    return res


def oracle_grad_module(mod, name: str):
    """A module-like holder of `name` canonicalised by the oracle's adjoint
    code generation (oracle.canonical: copy of the primal, then the VJP rules
    as IR in reverse order).  Bounds derived from it depend on the
    oracle only."""
    from types import SimpleNamespace
    return SimpleNamespace(functions={name: oracle.canonical(mod, name)})


def term_bound(mod, fname: str, inputs: Sequence[np.ndarray]) -> List[np.ndarray]:
    """sum|terms| of the accumulation producing each output of function
    `fname` in `mod` (an oracle-parsed module, or oracle_grad_module),
    evaluated in float64 by the oracle.  The bound follows the terms through
    the linear ops that carry an accumulation's rounding error unchanged
    (add/subtract/negate, a literal scale, select of one branch, reshapes,
    transposes, reductions); any other op ends it at |value|."""
    fn = mod.functions[fname]
    env = oracle.interp.evaluate(fn, inputs)
    defs = {ins.result: ins for ins in fn.insts}

    def val(o):
        return oracle.interp.literal_value(o) if o.kind == "literal" else env[o.name]

    def bound(o) -> np.ndarray:
        if o.kind == "literal":
            return np.abs(oracle.interp.literal_value(o))
        ins = defs.get(o.name)
        v = env[o.name]
        if ins is None:
            return np.abs(v).astype(np.float64)
        if ins.opcode == "dot":
            a, b = (np.abs(val(x)).astype(np.float64) for x in ins.operands)
            return a @ b
        if ins.opcode == "reduce":
            return np.sum(bound(ins.operands[0]), axis=ins.attrs["axis"])
        if ins.opcode == "shapeCast":
            return np.reshape(bound(ins.operands[0]), v.shape)
        if ins.opcode == "transpose":
            return np.transpose(bound(ins.operands[0]))
        if ins.opcode == "multiply" and any(x.kind == "literal" for x in ins.operands):
            lit = [x for x in ins.operands if x.kind == "literal"][0]
            other = [x for x in ins.operands if x.kind != "literal"][0]
            return np.broadcast_to(abs(lit.literal) * bound(other), v.shape)
        if ins.opcode in ("add", "subtract"):
            return np.broadcast_to(bound(ins.operands[0]) + bound(ins.operands[1]), v.shape)
        if ins.opcode == "negate":
            return bound(ins.operands[0])
        if ins.opcode == "select":
            c = np.broadcast_to(val(ins.operands[0]), v.shape)
            return np.where(c, np.broadcast_to(bound(ins.operands[1]), v.shape),
                            np.broadcast_to(bound(ins.operands[2]), v.shape))
        return np.abs(v).astype(np.float64)

    return [np.asarray(bound(o), dtype=np.float64) for o in fn.ret]


def f32_emulation(mod, fname: str, inputs: Sequence[np.ndarray]) -> List[np.ndarray]:
    """The same function evaluated op by op with every floating operand
    rounded to float32 first (numpy float32 arithmetic, float32 BLAS dot):
    an independent fp32 evaluation whose distance to the float64 oracle
    measures how ill-conditioned each output is in fp32."""
    fn = mod.functions[fname]
    env = {}
    for n, t, x in zip(fn.param_names, fn.param_types, inputs):
        env[n] = oracle.interp.as_value(x, t)

    def f32(a):
        return a.astype(np.float32) if a.dtype == np.float64 else a

    for ins in fn.insts:
        args = [f32(oracle.interp.literal_value(o) if o.kind == "literal" else env[o.name]) for o in ins.operands]
        env[ins.result] = oracle.interp.eval_inst(ins, args, fn.types[ins.result])
    return [oracle.interp.literal_value(o) if o.kind == "literal" else env[o.name] for o in fn.ret]


def assert_f32_parity(got: np.ndarray, ref: np.ndarray, bound: Optional[np.ndarray] = None,
                      rtol: float = 1e-5, what: str = "", extra: float = 0.0):
    """A16/A17 per-element check; `extra` (absolute) adds an allowance for
    programs whose fp32 evaluation is ill-conditioned beyond sum|terms| of
    the last op (random programs only; see f32_emulation)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    scale = np.abs(ref) if bound is None else np.maximum(np.abs(ref), bound)
    floor = rtol * 1e-6 * (np.max(np.abs(ref)) if ref.size else 0.0) + extra
    err = np.abs(got - ref)
    lim = rtol * scale + floor
    bad = ~(err <= lim)
    if bad.any():
        i = np.argmax(err - lim)
        raise AssertionError(f"{what}: {int(bad.sum())}/{bad.size} elements out of tolerance; worst at "
                             f"{np.unravel_index(i, got.shape)}: got {got.flat[i]!r} ref {ref.flat[i]!r} "
                             f"err {err.flat[i]:.3e} lim {lim.flat[i]:.3e}")


def assert_normwise(got: np.ndarray, ref: np.ndarray, tol: float = 2e-2, what: str = ""):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    den = np.linalg.norm(ref)
    num = np.linalg.norm(got - ref)
    rel = num / den if den > 0 else num
    assert rel <= tol, f"{what}: normwise relative error {rel:.3e} > {tol}"
    return rel
