"""Seeded synthetic workloads shared by the tests, the bench and the oracle
legs: IR text emitters and input generators.  Holds none of the method's
arithmetic (no op semantics, no AD, no shape rules) -- only the programs
(as `.dl` text) and their seeded inputs.

Input recipe: every argument is drawn
from numpy `Generator(PCG64(SeedSequence([1711, cfg, arg_index, block])))`
in float64 and rounded (RNE) to float32; those float32 values are canonical
and both the GPU path and the oracle consume exactly them.  Tensors are
generated in row blocks of BLOCK_ROWS rows so any subset of rows can be
regenerated cheaply for sampled full-size parity checks.

Configs (BASELINE.json `configs`):
  c1  MLP 784->128->10 sigmoid, batch 32, fp32 dot, MSE, fwd + adjoint
  c2  tanh(x*w + b) * m, row broadcast, [16384, 16384] f32 (2^28 elems)
  c3  MLP 4096->4096->4096->1000 ReLU, batch 1024, bf16 dot / fp32 acc
  c4  c3 data-parallel, global batch 65536, rows split contiguously
  c5  8 x (8192 -> 8192) tanh MLP, batch 131072 (16384 per rank on 8)
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

BLOCK_ROWS = 256
BASE_SEED = 1711


def _gen(cfg: int, arg: int, block: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([BASE_SEED, cfg, arg, block])))


def _ty(shape: Sequence[int]) -> str:
    if len(shape) == 0:
        return "f32"
    return "<" + " x ".join(str(d) for d in shape) + " x f32>"


@dataclass
class ArgSpec:
    name: str
    shape: Tuple[int, ...]
    dist: Tuple             # ("normal",) | ("uniform", lo, hi) | ("glorot", fan_in, fan_out)
                            # | ("bernoulli", p) | ("onehot",) | ("const", v)
    batched: bool = False   # leading dim is the (data-parallel) batch


def _draw(g: np.random.Generator, dist: Tuple, shape: Tuple[int, ...]) -> np.ndarray:
    kind = dist[0]
    if kind == "normal":
        return g.standard_normal(shape)
    if kind == "uniform":
        return g.uniform(dist[1], dist[2], shape)
    if kind == "glorot":
        lim = math.sqrt(6.0 / (dist[1] + dist[2]))
        return g.uniform(-lim, lim, shape)
    if kind == "bernoulli":
        return (g.random(shape) < dist[1]).astype(np.float64)
    if kind == "onehot":
        rows, cols = shape
        lab = g.integers(0, cols, rows)
        out = np.zeros(shape)
        out[np.arange(rows), lab] = 1.0
        return out
    if kind == "const":
        return np.full(shape, float(dist[1]))
    raise ValueError(kind)


def gen_arg(cfg: int, arg_index: int, spec: ArgSpec, rows: Optional[np.ndarray] = None,
            row_offset: int = 0) -> np.ndarray:
    """float32 values of one argument.  `rows` (sorted global row indices)
    selects a subset; `row_offset` shifts global rows (data-parallel shards
    draw the rows of the global batch they own)."""
    shape = tuple(spec.shape)
    if len(shape) < 2 or spec.dist[0] == "const":
        if rows is not None:
            raise ValueError("row selection needs a rank>=2 argument")
        return _draw(_gen(cfg, arg_index, 0), spec.dist, shape).astype(np.float32)
    R = shape[0]
    rest = shape[1:]
    want = np.arange(row_offset, row_offset + R) if rows is None else np.asarray(rows) + row_offset
    out = np.empty((len(want),) + rest, dtype=np.float32)
    blocks = np.unique(want // BLOCK_ROWS)
    pos = 0
    for b in blocks:
        lo = b * BLOCK_ROWS
        sel = want[(want >= lo) & (want < lo + BLOCK_ROWS)] - lo
        blk = _draw(_gen(cfg, arg_index, int(b)), spec.dist, (BLOCK_ROWS,) + rest)
        out[pos:pos + len(sel)] = blk[sel].astype(np.float32)
        pos += len(sel)
    return out


@dataclass
class Workload:
    cfg: int
    name: str
    text: str
    fn: str
    grad: str
    args: List[ArgSpec]
    seed_value: Optional[float] = None      # scalar seed for seedable grads
    seed_spec: Optional[ArgSpec] = None     # tensor seed (c2)
    dot_precision: str = "f32"              # "f32" | "bf16"
    batch: int = 0
    global_batch: int = 0
    layers: List[Tuple[int, int, Optional[str]]] = field(default_factory=list)

    def inputs(self, row_offset: int = 0) -> List[np.ndarray]:
        """All primal arguments (float32).  Batch-shaped args (leading dim ==
        batch) are drawn from global rows [row_offset, row_offset+batch)."""
        out = []
        for i, a in enumerate(self.args):
            out.append(gen_arg(self.cfg, i, a, row_offset=row_offset if a.batched else 0))
        return out

    def seed(self) -> Optional[np.ndarray]:
        if self.seed_spec is not None:
            return gen_arg(self.cfg, len(self.args), self.seed_spec)
        if self.seed_value is not None:
            return np.float32(self.seed_value)
        return None


# ---------------------------------------------------------------------------
# IR emitters

def _act_lines(act: Optional[str], l: int, a: str, shape) -> Tuple[List[str], str]:
    T = _ty(shape)
    if act is None:
        return [], a
    if act == "tanh":
        return [f"    %h{l} = tanh %{a}: {T}"], f"h{l}"
    if act == "relu":     # select(gt(z, 0), z, 0): "compare and select"; reading A11
        TB = "<" + " x ".join(str(d) for d in shape) + " x bool>"
        return [f"    %c{l} = gt %{a}: {T}, 0: f32",
                f"    %h{l} = select %c{l}: {TB}, %{a}: {T}, 0: f32"], f"h{l}"
    if act == "sigmoid":  # 1 / (1 + exp(-z)): composite; reading A10
        return [f"    %n{l} = negate %{a}: {T}",
                f"    %e{l} = exp %n{l}: {T}",
                f"    %d{l} = add %e{l}: {T}, 1: f32",
                f"    %h{l} = divide 1: f32, %d{l}: {T}"], f"h{l}"
    raise ValueError(act)


def mlp_ir(batch: int, layers: Sequence[Tuple[int, int, Optional[str]]],
           module: str = "mlp", with_grad: bool = True, loss: str = "mse") -> str:
    """Straight-line MLP `@mlp(x, W1, b1, ..., WL, bL, t) -> f32` with MSE
    loss 0.5 * sum((y - t)^2) (reading A9) and the declaration
    `[gradient @mlp wrt 1..2L keeping 0 seedable]` (Appendix A of SURVEY).
    loss="ce": softmax cross-entropy sum_b (logsumexp(y_b) - y_b . t_b),
    the log-sum-exp shifted by the row max (`reduce ... by max`, reading
    A26) and built from the paper's primitives otherwise."""
    L = len(layers)
    params = [(f"x", (batch, layers[0][0]))]
    for l, (i, o, _) in enumerate(layers, 1):
        params += [(f"w{l}", (i, o)), (f"b{l}", (1, o))]
    out_dim = layers[-1][1]
    params.append(("t", (batch, out_dim)))
    sig = ", ".join(_ty(s) for _, s in params)
    lines = [f'module "{module}"', "stage raw", "",
             f"func @mlp: ({sig}) -> f32 {{",
             "'entry(" + ", ".join(f"%{n}: {_ty(s)}" for n, s in params) + "):"]
    h = "x"
    for l, (i, o, act) in enumerate(layers, 1):
        lines.append(f"    %z{l} = dot %{h}: {_ty((batch, i))}, %w{l}: {_ty((i, o))}")
        lines.append(f"    %a{l} = add %z{l}: {_ty((batch, o))}, %b{l}: {_ty((1, o))}")
        more, h = _act_lines(act, l, f"a{l}", (batch, o))
        lines += more
    Y = _ty((batch, out_dim))
    B1 = _ty((batch,))
    if loss == "ce":
        lines += [f"    %mx = reduce %{h}: {Y} by max along 1",
                  f"    %mk = shapeCast %mx: {B1} to {batch} x 1",
                  f"    %zs = subtract %{h}: {Y}, %mk: {_ty((batch, 1))}",
                  f"    %ex = exp %zs: {Y}",
                  f"    %se = reduce %ex: {Y} by add along 1",
                  f"    %ls = log %se: {B1}",
                  f"    %lse = add %ls: {B1}, %mx: {B1}",
                  f"    %zt = multiply %{h}: {Y}, %t: {Y}",
                  f"    %zy = reduce %zt: {Y} by add along 1",
                  f"    %nl = subtract %lse: {B1}, %zy: {B1}",
                  f"    %L = reduce %nl: {B1} by add along 0",
                  "    return %L: f32", "}"]
    else:
        lines += [f"    %r = subtract %{h}: {Y}, %t: {Y}",
                  f"    %s = multiply %r: {Y}, %r: {Y}",
                  f"    %q = reduce %s: {Y} by add along 1",
                  f"    %l = reduce %q: {B1} by add along 0",
                  f"    %L = multiply %l: f32, 0.5: f32",
                  "    return %L: f32", "}"]
    if with_grad:
        wrt = ", ".join(str(k) for k in range(1, 2 * L + 1))
        grads = []
        for (i, o, _) in layers:
            grads += [_ty((i, o)), _ty((1, o))]
        lines += ["", f"[gradient @mlp wrt {wrt} keeping 0 seedable]",
                  f"func @mlp_grad: ({sig}, f32)",
                  f"    -> ({', '.join(grads)}, f32)"]
    return "\n".join(lines) + "\n"


def chain_ir(R: int, C: int, module: str = "chain") -> str:
    """c2: `@chain(x, w, b, m) = tanh(x*w + b) * m` with row-broadcast w, b
    and `[gradient @chain wrt 0, 1, 2 seedable]` (Appendix A of SURVEY)."""
    X, V = _ty((R, C)), _ty((1, C))
    return "\n".join([
        f'module "{module}"', "stage raw", "",
        f"func @chain: ({X}, {V}, {V}, {X}) -> {X} {{",
        f"'entry(%x: {X}, %w: {V}, %b: {V}, %m: {X}):",
        f"    %0 = multiply %x: {X}, %w: {V}",
        f"    %1 = add %0: {X}, %b: {V}",
        f"    %2 = tanh %1: {X}",
        f"    %3 = multiply %2: {X}, %m: {X}",
        f"    return %3: {X}",
        "}", "",
        "[gradient @chain wrt 0, 1, 2 seedable]",
        f"func @chain_grad: ({X}, {V}, {V}, {X}, {X})",
        f"    -> ({X}, {V}, {V})", ""])


def _mlp_workload(cfg: int, name: str, batch: int, layers, x_dist, t_dist, seed_value,
                  dot_precision: str, global_batch: int, loss: str = "mse") -> Workload:
    args = [ArgSpec("x", (batch, layers[0][0]), x_dist, batched=True)]
    for l, (i, o, _) in enumerate(layers, 1):
        args.append(ArgSpec(f"w{l}", (i, o), ("glorot", i, o)))
        args.append(ArgSpec(f"b{l}", (1, o), ("uniform", -0.1, 0.1)))
    args.append(ArgSpec("t", (batch, layers[-1][1]), t_dist, batched=True))
    return Workload(cfg, name, mlp_ir(batch, layers, module=name, loss=loss), "mlp", "mlp_grad", args,
                    seed_value=seed_value, dot_precision=dot_precision, batch=batch,
                    global_batch=global_batch, layers=list(layers))


C1_LAYERS = [(784, 128, "sigmoid"), (128, 10, "sigmoid")]
C3_LAYERS = [(4096, 4096, "relu"), (4096, 4096, "relu"), (4096, 1000, None)]
C5_LAYERS = [(8192, 8192, "tanh")] * 8


def c1(batch: int = 32) -> Workload:
    return _mlp_workload(1, "c1_mlp", batch, C1_LAYERS, ("uniform", 0.0, 1.0), ("onehot",),
                         1.0 / batch, "f32", batch)


def c2(R: int = 16384, C: int = 16384) -> Workload:
    X, V = (R, C), (1, C)
    args = [ArgSpec("x", X, ("normal",), batched=True), ArgSpec("w", V, ("uniform", 0.5, 1.5)),
            ArgSpec("b", V, ("uniform", -0.5, 0.5)),
            ArgSpec("m", X, ("bernoulli", 0.9), batched=True)]
    return Workload(2, "c2_chain", chain_ir(R, C), "chain", "chain_grad", args,
                    seed_spec=ArgSpec("g", X, ("normal",), batched=True), batch=R, global_batch=R)


def c3(batch: int = 1024, global_batch: Optional[int] = None, cfg: int = 3,
       layers=None) -> Workload:
    gb = batch if global_batch is None else global_batch
    return _mlp_workload(cfg, "c3_mlp" if cfg == 3 else "c4_mlp", batch, layers or C3_LAYERS,
                         ("normal",), ("onehot",), 1.0 / gb, "bf16", gb)


def ce_mlp(batch: int = 1024, layers=None, global_batch: Optional[int] = None,
           dot_precision: str = "bf16") -> Workload:
    """The c3 MLP shape with the softmax cross-entropy loss (SURVEY §8(f)
    rank 4): one-hot targets, seed 1/B (mean over the batch)."""
    gb = batch if global_batch is None else global_batch
    return _mlp_workload(8, "ce_mlp", batch, layers or C3_LAYERS, ("normal",), ("onehot",), 1.0 / gb,
                         dot_precision, gb, loss="ce")


def c4(n_ranks: int = 1, global_batch: int = 65536) -> Workload:
    """Per-rank program of c4: the c3 MLP on B_local = global_batch / n_ranks."""
    assert global_batch % n_ranks == 0
    return c3(global_batch // n_ranks, global_batch, cfg=4)


def c5(batch: int = 16384, global_batch: int = 131072) -> Workload:
    return _mlp_workload(5, "c5_mlp", batch, C5_LAYERS, ("normal",), ("uniform", -0.5, 0.5),
                         1.0 / global_batch, "bf16", global_batch)


FIG3 = '''module "my_module"
stage raw

// Representing function foo(x, w, b) = dot(x, w) + b
func @foo: (<1 x 784 x f32>, <784 x 10 x f32>, <1 x 10 x f32>)
          -> <1 x 10 x f32> {
'entry(%x: <1 x 784 x f32>, %w: <784 x 10 x f32>, %b: <1 x 10 x f32>):
    %0 = dot %x: <1 x 784 x f32>, %w: <784 x 10 x f32>
    %1 = add %0: <1 x 10 x f32>, %b: <1 x 10 x f32>
    return %1: <1 x 10 x f32>
}

// Gradient of @foo with respect to all arguments
[gradient @foo]
func @foo_grad: (<1 x 784 x f32>, <784 x 10 x f32>, <1 x 10 x f32>)
           -> (<1 x 784 x f32>, <784 x 10 x f32>, <1 x 10 x f32>)

// Gradient of @foo with respect to arguments 1 and 2
// Keeping original output 0
// Seedable, able to take back-propagated gradient as a seed for AD
[gradient @foo wrt 1, 2 keeping 0 seedable]
func @foo_grad_3:
    (<1 x 784 x f32>, <784 x 10 x f32>, <1 x 10 x f32>, <1 x 10 x f32>)
   -> (<784 x 10 x f32>, <1 x 10 x f32>, <1 x 10 x f32>)
'''
"""Fig. 3 (P:L249-272) with the garbled body read as A4 (P:L252 comment)."""


def fig4_ir(B: int = 4, I: int = 6, O: int = 5) -> str:
    """Fig. 4: g(x, w, b) = tanh(x . w + b),
    dg = gradient(of: g, withRespectTo: (1, 2), keeping: 0)."""
    X, W, V = _ty((B, I)), _ty((I, O)), _ty((B, O))
    Bv = _ty((1, O))
    return "\n".join([
        'module "nnkit_fig4"', "stage raw", "",
        f"func @g: ({X}, {W}, {Bv}) -> {V} {{",
        f"'entry(%x: {X}, %w: {W}, %b: {Bv}):",
        f"    %0 = dot %x: {X}, %w: {W}",
        f"    %1 = add %0: {V}, %b: {Bv}",
        f"    %2 = tanh %1: {V}",
        f"    return %2: {V}", "}", "",
        "[gradient @g wrt 1, 2 keeping 0]",
        f"func @dg: ({X}, {W}, {Bv}) -> ({W}, {Bv}, {V})", ""])


def sgd_ir(shapes: Sequence[Tuple[int, ...]], lr: float = 1e-3, copies: Sequence[bool] = (),
           module: str = "sgd") -> str:
    """The SGD update of SURVEY §8(a) H12 as DLVM IR (P:L213 element-wise
    binary ops): for every parameter p_i with gradient g_i,
    p_i' = subtract(p_i, multiply(g_i, lr)); returned once, and a second
    time when copies[i] (the caller requests that output as the bf16
    operand copy the next step's dots read)."""
    params, body, rets, rtypes = [], [], [], []
    for i, s in enumerate(shapes):
        T = _ty(s)
        params += [(f"p{i}", T), (f"g{i}", T)]
        body += [f"    %u{i} = multiply %g{i}: {T}, {lr!r}: f32", f"    %n{i} = subtract %p{i}: {T}, %u{i}: {T}"]
        rets.append(f"%n{i}: {T}")
        rtypes.append(T)
        if i < len(copies) and copies[i]:
            rets.append(f"%n{i}: {T}")
            rtypes.append(T)
    sig = ", ".join(t for _, t in params)
    return "\n".join([f'module "{module}"', "stage raw", f"func @sgd: ({sig}) -> ({', '.join(rtypes)}) {{",
                      "'entry(" + ", ".join(f"%{n}: {t}" for n, t in params) + "):"] + body +
                     ["    return (" + ", ".join(rets) + ")", "}", ""])


def rnn_ir(T: int, B: int, I: int, H: int, module: str = "rnn") -> str:
    """Unrolled simple RNN (§3.1.2):
    h_t = tanh(x_t W + h_{t-1} U + b), t = 1..T (row-vector convention, x_t
    [B, I], h [B, H]), loss 0.5 * sum((h_T - y)^2), and
    `[gradient @rnn wrt W, U, b keeping 0 seedable]`."""
    xs = [(f"x{t}", (B, I)) for t in range(1, T + 1)]
    params = xs + [("h0", (B, H)), ("W", (I, H)), ("U", (H, H)), ("b", (1, H)), ("y", (B, H))]
    sig = ", ".join(_ty(s) for _, s in params)
    X, Hs = _ty((B, I)), _ty((B, H))
    lines = [f'module "{module}"', "stage raw", "", f"func @rnn: ({sig}) -> f32 {{",
             "'entry(" + ", ".join(f"%{n}: {_ty(s)}" for n, s in params) + "):"]
    for t in range(1, T + 1):
        lines += [f"    %wx{t} = dot %x{t}: {X}, %W: {_ty((I, H))}",
                  f"    %uh{t} = dot %h{t - 1}: {Hs}, %U: {_ty((H, H))}",
                  f"    %s{t} = add %wx{t}: {Hs}, %uh{t}: {Hs}",
                  f"    %z{t} = add %s{t}: {Hs}, %b: {_ty((1, H))}",
                  f"    %h{t} = tanh %z{t}: {Hs}"]
    lines += [f"    %r = subtract %h{T}: {Hs}, %y: {Hs}",
              f"    %e = multiply %r: {Hs}, %r: {Hs}",
              f"    %q = reduce %e: {Hs} by add along 1",
              f"    %l = reduce %q: {_ty((B,))} by add along 0",
              f"    %L = multiply %l: f32, 0.5: f32",
              "    return %L: f32", "}", "",
              f"[gradient @rnn wrt {T + 1}, {T + 2}, {T + 3} keeping 0 seedable]",
              f"func @rnn_grad: ({sig}, f32) -> ({_ty((I, H))}, {_ty((H, H))}, {_ty((1, H))}, f32)"]
    return "\n".join(lines) + "\n"


def rnn(T: int = 8, B: int = 8192, I: int = 2048, H: int = 2048, dot_precision: str = "bf16") -> Workload:
    """Config r (NEXT rank 2): the unrolled RNN above; x_t ~ N(0,1),
    h0 ~ U(-0.5, 0.5), W, U Glorot, b ~ U(+-0.1), y ~ U(-0.5, 0.5), seed 1/B."""
    args = [ArgSpec(f"x{t}", (B, I), ("normal",), batched=True) for t in range(1, T + 1)]
    args += [ArgSpec("h0", (B, H), ("uniform", -0.5, 0.5), batched=True),
             ArgSpec("W", (I, H), ("glorot", I, H)), ArgSpec("U", (H, H), ("glorot", H, H)),
             ArgSpec("b", (1, H), ("uniform", -0.1, 0.1)),
             ArgSpec("y", (B, H), ("uniform", -0.5, 0.5), batched=True)]
    return Workload(6, "rnn", rnn_ir(T, B, I, H), "rnn", "rnn_grad", args, seed_value=1.0 / B,
                    dot_precision=dot_precision, batch=B, global_batch=B)


def mlp_hvp_ir(B: int, I: int, H: int, O: int, module: str = "hvp") -> str:
    """Higher-order AD: a 2-layer
    tanh MLP with MSE loss `@f`, its gradient `@df` w.r.t. W1, b1, W2, and the
    gradient of `@df`'s first output (dL/dW1) w.r.t. W1 and W2, seeded with a
    direction v: a Hessian-vector product `@hvp(x, W1, b1, W2, y, v)`."""
    P = [("x", (B, I)), ("W1", (I, H)), ("b1", (1, H)), ("W2", (H, O)), ("y", (B, O))]
    sig = ", ".join(_ty(s) for _, s in P)
    Hs, Os = _ty((B, H)), _ty((B, O))
    lines = [f'module "{module}"', "stage raw", "", f"func @f: ({sig}) -> f32 {{",
             "'entry(" + ", ".join(f"%{n}: {_ty(s)}" for n, s in P) + "):",
             f"    %z = dot %x: {_ty((B, I))}, %W1: {_ty((I, H))}",
             f"    %a = add %z: {Hs}, %b1: {_ty((1, H))}",
             f"    %h = tanh %a: {Hs}",
             f"    %o = dot %h: {Hs}, %W2: {_ty((H, O))}",
             f"    %r = subtract %o: {Os}, %y: {Os}",
             f"    %e = multiply %r: {Os}, %r: {Os}",
             f"    %q = reduce %e: {Os} by add along 1",
             f"    %l = reduce %q: {_ty((B,))} by add along 0",
             f"    %L = multiply %l: f32, 0.5: f32",
             "    return %L: f32", "}", "",
             "[gradient @f wrt 1, 2, 3]",
             f"func @df: ({sig}) -> ({_ty((I, H))}, {_ty((1, H))}, {_ty((H, O))})", "",
             "[gradient @df from 0 wrt 1, 3 seedable]",
             f"func @hvp: ({sig}, {_ty((I, H))}) -> ({_ty((I, H))}, {_ty((H, O))})"]
    return "\n".join(lines) + "\n"


def mlp_hvp(B: int = 8192, I: int = 4096, H: int = 4096, O: int = 1000) -> Workload:
    """Config h (NEXT rank 3): Hessian-vector product of the MLP above; x ~
    N(0,1), Glorot weights, b ~ U(+-0.1), y one-hot, direction v ~ N(0,1)."""
    args = [ArgSpec("x", (B, I), ("normal",), batched=True), ArgSpec("W1", (I, H), ("glorot", I, H)),
            ArgSpec("b1", (1, H), ("uniform", -0.1, 0.1)), ArgSpec("W2", (H, O), ("glorot", H, O)),
            ArgSpec("y", (B, O), ("onehot",), batched=True)]
    return Workload(7, "mlp_hvp", mlp_hvp_ir(B, I, H, O), "df", "hvp", args,
                    seed_spec=ArgSpec("v", (I, H), ("normal",)), dot_precision="bf16", batch=B, global_batch=B)


CONFIGS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5, "rnn": rnn, "mlp_hvp": mlp_hvp}
