"""Pins of the oracle's adjoint code generation (oracle/adjoint.py) and the
higher-order gradients it enables (§3.1.3, Fig. 4
`d2g_dw2` L367-370).  CPU only.

  * first order: the generated adjoint IR, interpreted in float64, equals the
    value-level reverse sweep (vjp.py), a second independent route;
  * second / third order against closed forms: d2/dx2 sum(x^3) = 6x at [1, 2]
    is [6, 12] (F13); d3/dx3 sum(x^4) = 24x; Fig. 4's
    d2g_dw2[k, l] = -2 sum_r x_rk s_r t_rl (1 - t_rl^2), s_r = sum_i x_ri,
    t = tanh(x w + b) (derived by hand from the Fig. 4 program);
  * second order against central finite differences of the first-order
    gradient function.
"""

import numpy as np
import pytest

import oracle
import workloads as W


def _scalar_sum_pow(n, p, orders):
    t = f"<{n} x f32>"
    text = (f'module "h"\nstage raw\nfunc @f: ({t}) -> f32 {{\n\'entry(%x: {t}):\n'
            f"    %p = power %x: {t}, {p}: f32\n    %s = reduce %p: {t} by add along 0\n    return %s: f32\n}}\n"
            f"[gradient @f]\nfunc @d1: ({t}) -> {t}\n")
    for k in range(2, orders + 1):
        text += f"[gradient @d{k - 1}]\nfunc @d{k}: ({t}) -> {t}\n"
    return text


def test_F13_second_derivative_sum_cubes():
    m = oracle.parse(_scalar_sum_pow(2, 3, 2))
    x = np.array([1.0, 2.0])
    np.testing.assert_allclose(oracle.run(m, "d1", [x])[0], 3 * x * x, rtol=1e-15)
    np.testing.assert_allclose(oracle.run(m, "d2", [x])[0], [6.0, 12.0], rtol=1e-15)


def test_third_order_sum_fourth_powers():
    m = oracle.parse(_scalar_sum_pow(3, 4, 3))
    x = np.array([0.5, -1.5, 2.0])
    np.testing.assert_allclose(oracle.run(m, "d2", [x])[0], 12 * x * x, rtol=1e-14)
    np.testing.assert_allclose(oracle.run(m, "d3", [x])[0], 24 * x, rtol=1e-14)


FIG4_D2 = "\n[gradient @dg from 0 wrt 1]\nfunc @d2g_dw2: ({a}, {w}, {b}) -> {w}\n"


def fig4_second_order(B=4, I=6, O=5):
    a, w, b = f"<{B} x {I} x f32>", f"<{I} x {O} x f32>", f"<1 x {O} x f32>"
    return W.fig4_ir(B, I, O) + FIG4_D2.format(a=a, w=w, b=b)


def test_fig4_d2g_dw2_closed_form():
    m = oracle.parse(fig4_second_order())
    assert m.functions["d2g_dw2"].result_types[0].shape == (6, 5)   # Rep<(...) -> Float2D>
    rng = np.random.default_rng(4)
    x, w, b = rng.normal(size=(4, 6)), 0.3 * rng.normal(size=(6, 5)), 0.1 * rng.normal(size=(1, 5))
    (h,) = oracle.run(m, "d2g_dw2", [x, w, b])
    t = np.tanh(x @ w + b)
    want = -2.0 * np.einsum("rk,r,rl->kl", x, x.sum(axis=1), t * (1.0 - t * t))
    np.testing.assert_allclose(h, want, rtol=1e-12, atol=1e-14)


def _mlp2(B, I, H, O, act):
    ty = lambda *s: "<" + " x ".join(map(str, s)) + " x f32>"
    acts = {"tanh": ["    %h = tanh %a: {t}"],
            "sigmoid": ["    %n = negate %a: {t}", "    %e = exp %n: {t}", "    %d = add %e: {t}, 1: f32",
                        "    %h = divide 1: f32, %d: {t}"]}
    body = [f"    %z = dot %x: {ty(B, I)}, %w1: {ty(I, H)}", f"    %a = add %z: {ty(B, H)}, %b1: {ty(1, H)}"]
    body += [l.format(t=ty(B, H)) for l in acts[act]]
    body += [f"    %y = dot %h: {ty(B, H)}, %w2: {ty(H, O)}", f"    %r = subtract %y: {ty(B, O)}, %t: {ty(B, O)}",
             f"    %s = multiply %r: {ty(B, O)}, %r: {ty(B, O)}", f"    %q = reduce %s: {ty(B, O)} by add along 1",
             f"    %l = reduce %q: {ty(B)} by add along 0"]
    P = [("x", (B, I)), ("w1", (I, H)), ("b1", (1, H)), ("w2", (H, O)), ("t", (B, O))]
    sig = ", ".join(ty(*s) for _, s in P)
    text = (f'module "m"\nstage raw\nfunc @f: ({sig}) -> f32 {{\n\'entry(' +
            ", ".join(f"%{n}: {ty(*s)}" for n, s in P) + "):\n" + "\n".join(body) + "\n    return %l: f32\n}\n"
            f"[gradient @f wrt 1, 2, 3]\nfunc @df: ({sig}) -> ({ty(I, H)}, {ty(1, H)}, {ty(H, O)})\n"
            f"[gradient @df from 0 wrt 1, 3 seedable]\nfunc @hvp: ({sig}, {ty(I, H)}) -> ({ty(I, H)}, {ty(H, O)})\n")
    return text, P


@pytest.mark.parametrize("act", ["tanh", "sigmoid"])
def test_second_order_seedable_vs_fd(act):
    """Hessian-vector product of an MLP loss (seed = direction v on dW1):
    d/dW [ <v, dL/dW1> ] from the generated second-order IR equals central
    differences of the generated first-order function."""
    text, P = _mlp2(5, 4, 6, 3, act)
    m = oracle.parse(text)
    rng = np.random.default_rng(7)
    ins = [rng.normal(size=s) * (0.5 if n.startswith("w") else 1.0) for n, s in P]
    v = rng.normal(size=(4, 6))
    got = oracle.run(m, "hvp", ins + [v])
    df = oracle.canonical(m, "df")
    for k, wrt in enumerate((1, 3)):
        fd = oracle.fd_grad(df, ins, wrt, from_=0, seed=v, h=1e-5)
        np.testing.assert_allclose(got[k], fd, rtol=1e-6, atol=1e-8 * np.max(np.abs(fd)))


def _rand_prog(rng):
    n = int(rng.integers(2, 5))
    c = int(rng.integers(2, 5))
    X, V = f"<{n} x {c} x f32>", f"<1 x {c} x f32>"
    lines, cur, k = [], "%x", 0
    for _ in range(int(rng.integers(2, 6))):
        k += 1
        op = ["mulv", "addv", "tanh", "exp", "divv", "sq", "relu", "tt"][int(rng.integers(8))]
        if op == "mulv":
            lines.append(f"    %t{k} = multiply {cur}: {X}, %v: {V}")
        elif op == "addv":
            lines.append(f"    %t{k} = add %v: {V}, {cur}: {X}")
        elif op == "divv":
            lines += [f"    %p{k} = exp %v: {V}", f"    %t{k} = divide {cur}: {X}, %p{k}: {V}"]
        elif op == "sq":
            lines.append(f"    %t{k} = multiply {cur}: {X}, {cur}: {X}")
        elif op == "relu":
            lines += [f"    %c{k} = gt {cur}: {X}, 0: f32", f"    %t{k} = select %c{k}: <{n} x {c} x bool>, {cur}: {X}, 0: f32"]
        elif op == "tt":
            lines += [f"    %u{k} = transpose {cur}: {X}", f"    %t{k} = transpose %u{k}: <{c} x {n} x f32>"]
        else:
            lines.append(f"    %t{k} = {op} {cur}: {X}")
        cur = f"%t{k}"
    lines += [f"    %r0 = reduce {cur}: {X} by add along 1", f"    %r1 = reduce %r0: <{n} x f32> by add along 0"]
    text = (f'module "r"\nstage raw\nfunc @f: ({X}, {V}) -> f32 {{\n\'entry(%x: {X}, %v: {V}):\n' + "\n".join(lines) +
            f"\n    return %r1: f32\n}}\n[gradient @f]\nfunc @g: ({X}, {V}) -> ({X}, {V})\n"
            f"[gradient @g from 1 wrt 1]\nfunc @h: ({X}, {V}) -> {V}\n")
    return text, [(n, c), (1, c)]


@pytest.mark.parametrize("seed", range(12))
def test_random_programs_symbolic_equals_value_vjp_and_fd(seed):
    rng = np.random.default_rng(500 + seed)
    text, shapes = _rand_prog(rng)
    m = oracle.parse(text)
    ins = [rng.uniform(-1, 1, s) for s in shapes]
    g_sym = oracle.run_function(oracle.canonical(m, "g"), ins)
    g_val = oracle.run(m, "g", ins)
    for a, b in zip(g_sym, g_val):
        np.testing.assert_allclose(a, b, rtol=1e-13, atol=1e-13)
    (h,) = oracle.run(m, "h", ins)
    fd = oracle.fd_grad(oracle.canonical(m, "g"), ins, 1, from_=1, h=1e-5)
    np.testing.assert_allclose(h, fd, rtol=1e-5, atol=1e-6 * (np.max(np.abs(fd)) + 1))


def test_first_order_configs_symbolic_equals_value_vjp():
    for w in [W.c1(), W.c2(8, 12), W.c3(16, layers=[(12, 10, "relu"), (10, 6, None)]), W.c5(8)]:
        if w.layers and w.layers[0][0] > 1000:
            w = W._mlp_workload(5, "c5s", 8, [(16, 16, "tanh")] * 3, ("normal",), ("uniform", -0.5, 0.5),
                                1.0 / 8, "bf16", 8)
        m = oracle.parse(w.text)
        ins = [x.astype(np.float64) for x in w.inputs()]
        s = w.seed()
        args = ins + ([np.asarray(s, dtype=np.float64)] if s is not None else [])
        for a, b in zip(oracle.run_function(oracle.canonical(m, w.grad), args), oracle.run(m, w.grad, args)):
            np.testing.assert_allclose(a, b, rtol=1e-13, atol=1e-15)


def test_cyclic_gradient_declarations_rejected():
    t = "<2 x f32>"
    text = (f'module "c"\nstage raw\n[gradient @b]\nfunc @a: ({t}) -> {t}\n'
            f"[gradient @a]\nfunc @b: ({t}) -> {t}\n")
    with pytest.raises(oracle.VerifyError):
        oracle.parse(text)
