"""Random rank-1..5 straight-line programs (test corpus): NumPy
broadcasting between operands of different ranks and unit dims (reading
A1), full-reversal transposes of rank > 2 (Table 1), reductions along
random axes re-broadcast through shapeCast (L173, L181), compare/select, and
a scalar loss; gradient w.r.t. every argument.  Shared by the CPU (types,
AD, plan) and GPU (parity) tests; holds no arithmetic of the method."""

from __future__ import annotations

import numpy as np


def T(s):
    return "<" + " x ".join(str(d) for d in s) + " x f32>" if s else "f32"


def TB(s):
    return "<" + " x ".join(str(d) for d in s) + " x bool>"


def bcast_shape(rng, S):
    """A shape that broadcasts to S: some dims set to 1, some leading dims dropped."""
    s = [1 if rng.random() < 0.5 else d for d in S]
    drop = int(rng.integers(0, len(S)))
    return tuple(s[drop:])


def nd_program(rng, max_elems=6000, all_values=False, allow_select=True, wide=False):
    """(text, args); with all_values the primal returns every f32 value it
    defines (a tuple, no gradient declaration) instead of the loss; without
    allow_select no compare/select (discrete decisions) is drawn; wide
    programs (rank 2..4, last dim 64..256, >= 128 rows) put their dots on the
    tensor-core path."""
    if wide:
        r = int(rng.integers(2, 5))
        while True:
            S = [int(rng.integers(1, 6)) for _ in range(r - 1)] + [int(rng.choice([64, 96, 128, 200, 256]))]
            S[int(rng.integers(r - 1))] = int(rng.integers(130, 600))
            if int(np.prod(S)) <= 400000:
                break
    else:
        r = int(rng.integers(1, 6))
        while True:
            S = [int(rng.integers(1, 6)) for _ in range(r)]
            S[int(rng.integers(r))] = int(rng.integers(8, 41))  # one long dim: several tiles and a ragged tail
            if int(np.prod(S)) <= max_elems:
                break
    S = tuple(S)
    RS = tuple(reversed(S))
    args = [("x", S), ("b1", bcast_shape(rng, S)), ("b2", bcast_shape(rng, S)), ("y", S), ("w", (S[-1], S[-1]))]
    M2 = (int(np.prod(S[:-1])), S[-1])  # cur viewed as a matrix for dot
    L, vals, cur, k = [], [], "%x", 0

    def d(name, rhs, shape):  # one definition of an f32 value
        L.append(f"    {name} = {rhs}")
        vals.append((name, shape))

    def other():
        c = int(rng.integers(4))
        return [f"%b1: {T(args[1][1])}", f"%b2: {T(args[2][1])}", "0.3: f32", f"%y: {T(S)}"][c]

    for _ in range(int(rng.integers(4, 9))):
        kind = ["bin", "bin_rev", "unary", "transpose", "reduce", "select", "dot", "math"][int(rng.integers(8))]
        if kind == "select" and not allow_select:
            kind = "math"
        if all_values and kind == "reduce" and rng.random() < 0.3:
            kind = "prod"  # forward only (no derivative): all-values programs
        k += 1
        i = k
        if kind in ("bin", "bin_rev"):
            op = ["add", "subtract", "multiply"][int(rng.integers(3))]
            a, b = f"{cur}: {T(S)}", other()
            if kind == "bin_rev":
                a, b = b, a
            d(f"%t{i}", f"{op} {a}, {b}", S)
        elif kind == "unary":
            op = ["tanh", "negate", "sigmoid"][int(rng.integers(3))]
            if op == "sigmoid":
                d(f"%n{i}", f"negate {cur}: {T(S)}", S)
                d(f"%e{i}", f"exp %n{i}: {T(S)}", S)
                d(f"%d{i}", f"add %e{i}: {T(S)}, 1: f32", S)
                d(f"%t{i}", f"divide 1: f32, %d{i}: {T(S)}", S)
            else:
                d(f"%t{i}", f"{op} {cur}: {T(S)}", S)
        elif kind == "transpose":  # (cur^T * y^T)^T: a rank-r reversal and back
            d(f"%p{i}", f"transpose {cur}: {T(S)}", RS)
            d(f"%q{i}", f"transpose %y: {T(S)}", RS)
            d(f"%m{i}", f"multiply %p{i}: {T(RS)}, %q{i}: {T(RS)}", RS)
            d(f"%t{i}", f"transpose %m{i}: {T(RS)}", S)
        elif kind == "reduce":  # cur + 0.1 * shapeCast(sum_a cur) (keepdims broadcast)
            a = int(rng.integers(r))
            RSH = tuple(dd for j, dd in enumerate(S) if j != a)
            KS = tuple(1 if j == a else dd for j, dd in enumerate(S))
            d(f"%r{i}", f"reduce {cur}: {T(S)} by add along {a}", RSH)
            d(f"%k{i}", f"shapeCast %r{i}: {T(RSH)} to {' x '.join(map(str, KS))}", KS)
            d(f"%s{i}", f"multiply %k{i}: {T(KS)}, 0.1: f32", KS)
            d(f"%t{i}", f"add {cur}: {T(S)}, %s{i}: {T(KS)}", S)
        elif kind == "prod":  # cur * shapeCast(prod_a (1 + 0.05 cur)) (factors near 1)
            a = int(rng.integers(r))
            RSH = tuple(dd for j, dd in enumerate(S) if j != a)
            KS = tuple(1 if j == a else dd for j, dd in enumerate(S))
            d(f"%f{i}", f"multiply {cur}: {T(S)}, 0.05: f32", S)
            d(f"%g{i}", f"add %f{i}: {T(S)}, 1: f32", S)
            d(f"%r{i}", f"reduce %g{i}: {T(S)} by multiply along {a}", RSH)
            d(f"%k{i}", f"shapeCast %r{i}: {T(RSH)} to {' x '.join(map(str, KS))}", KS)
            d(f"%t{i}", f"multiply {cur}: {T(S)}, %k{i}: {T(KS)}", S)
        elif kind == "dot":  # shapeCast to [prod(S[:-1]), S[-1]], dot with w, shapeCast back
            d(f"%v{i}", f"shapeCast {cur}: {T(S)} to {M2[0]} x {M2[1]}", M2)
            d(f"%o{i}", f"dot %v{i}: {T(M2)}, %w: {T(args[4][1])}", M2)
            d(f"%t{i}", f"shapeCast %o{i}: {T(M2)} to {' x '.join(map(str, S))}", S)
        elif kind == "math":  # power, divide, log / sqrt of 1 + x^2, abs
            op = ["power2", "power3", "divide", "log", "sqrt", "abs"][int(rng.integers(6))]
            if op.startswith("power"):
                d(f"%t{i}", f"power {cur}: {T(S)}, {op[-1]}: f32", S)
            elif op == "abs":
                d(f"%t{i}", f"abs {cur}: {T(S)}", S)
            else:
                d(f"%u{i}", f"multiply {cur}: {T(S)}, {cur}: {T(S)}", S)
                d(f"%a{i}", f"add %u{i}: {T(S)}, 1: f32", S)
                if op == "divide":
                    d(f"%t{i}", f"divide {cur}: {T(S)}, %a{i}: {T(S)}", S)
                else:
                    d(f"%t{i}", f"{op} %a{i}: {T(S)}", S)
        else:  # relu-like select against a broadcast threshold
            L.append(f"    %c{i} = gt {cur}: {T(S)}, {other()}")
            d(f"%t{i}", f"select %c{i}: {TB(S)}, {cur}: {T(S)}, %b1: {T(args[1][1])}", S)
        cur = f"%t{i}"
    d("%sq", f"multiply {cur}: {T(S)}, {cur}: {T(S)}", S)
    sh, v = list(S), "%sq"
    for j in range(r):
        d(f"%z{j}", f"reduce {v}: {T(tuple(sh))} by add along 0", tuple(sh[1:]))
        v, sh = f"%z{j}", sh[1:]
    sig = ", ".join(T(s) for _, s in args)
    entry = "'entry(" + ", ".join(f"%{n}: {T(s)}" for n, s in args) + "):"
    if all_values:
        rtys = ", ".join(T(s) for _, s in vals)
        rets = ", ".join(f"{n}: {T(s)}" for n, s in vals)
        head = ['module "nd"', "stage raw", f"func @f: ({sig}) -> ({rtys}) {{", entry]
        return "\n".join(head + L + [f"    return ({rets})", "}", ""]), args
    head = ['module "nd"', "stage raw", f"func @f: ({sig}) -> f32 {{", entry]
    tail = [f"    return {v}: f32", "}", "", "[gradient @f]", f"func @g: ({sig}) -> ({sig})", ""]
    return "\n".join(head + L + tail), args


def nd_inputs(rng, args):
    # w scaled so a chain of dots keeps values O(1)
    return [(rng.uniform(-1, 1, s) * (1.0 / np.sqrt(s[0]) if n == "w" else 1.0)).astype(np.float32)
            for n, s in args]


def nd_grad_config(rng, max_elems=6000):
    """A random program whose primal returns a tuple (loss, last tensor
    value) with a random gradient configuration (Fig. 3 / Fig. 4: `wrt` a
    subset, `keeping` some outputs, `from` either output, `seedable` with a
    scalar or tensor seed).  Returns (text, args, cfg)."""
    text, args = nd_program(rng, max_elems)
    S = args[0][1]
    lines = text.split("\n[gradient")[0].splitlines()
    body = [l for l in lines if l.startswith("    %")]
    tail = [l for l in body if l.strip().startswith("%sq =")][0]
    last = tail.split("multiply ")[1].split(":")[0]  # the value squared into the loss
    ret = [l for l in lines if l.strip().startswith("return")][0]
    loss = ret.split("return ")[1].split(":")[0]
    n = len(args)
    wrt = sorted(int(i) for i in rng.choice(n, size=int(rng.integers(1, n + 1)), replace=False))
    frm = int(rng.integers(2))
    keeping = [k for k in range(2) if rng.random() < 0.5]
    seedable = bool(rng.random() < 0.6)
    sig = ", ".join(T(s) for _, s in args)
    rtys = ["f32", T(S)]
    out = [l for l in lines if not l.strip().startswith("return") and not l.startswith("func @f")]
    head = [l for l in lines if l.startswith("func @f")][0]
    head = head.replace("-> f32 {", f"-> (f32, {T(S)}) {{")
    i_entry = [k for k, l in enumerate(out) if l.startswith("'entry")][0]
    out.insert(i_entry, head)
    out = [l for l in out if l != "}"]
    out += [f"    return ({loss}: f32, {last}: {T(S)})", "}", ""]
    gin = sig + (", " + rtys[frm] if seedable else "")
    gout = [T(args[i][1]) for i in wrt] + [rtys[k] for k in keeping]
    attr = f"[gradient @f from {frm} wrt {', '.join(map(str, wrt))}"
    if keeping:
        attr += f" keeping {', '.join(map(str, keeping))}"
    attr += " seedable]" if seedable else "]"
    gsig = gout[0] if len(gout) == 1 else "(" + ", ".join(gout) + ")"
    out += [attr, f"func @g: ({gin}) -> {gsig}", ""]
    cfg = dict(wrt=wrt, frm=frm, keeping=keeping, seedable=seedable, seed_shape=() if frm == 0 else S)
    return "\n".join(out), args, cfg
