"""Pins for the CPU oracle: every check compares the
oracle against something other than itself -- hand-computed values, closed
forms, brute force, finite differences, identities."""

import itertools
import json
import os

import numpy as np
import pytest

import oracle
import workloads as W
from oracle.ir import ParseError, VerifyError

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _pins():
    with open(os.path.join(GOLD, "hand_pins.json")) as f:
        return json.load(f)


def _one_inst_fn(inst_text, result="%r"):
    """Wraps one Table-1 instruction in a function whose args are its operands."""
    import re
    ops = re.findall(r"%(\w+): (<[^>]*>|\w+)", inst_text)
    args = ", ".join(f"%{n}: {t}" for n, t in ops)
    sig = ", ".join(t for _, t in ops)
    return ops, sig, args


def _table1_rows():
    rows = []
    for line in open(os.path.join(GOLD, "table1_types.txt")):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        inst, ty = [s.strip() for s in line.split("|")]
        rows.append((inst, ty))
    return rows


@pytest.mark.parametrize("inst,want", _table1_rows())
def test_F9_table1_types(inst, want):
    ops, sig, args = _one_inst_fn(inst)
    text = (f'module "t"\nstage raw\nfunc @f: ({sig}) -> {want} {{\n'
            f"'entry({args}):\n    %r = {inst}\n    return %r: {want}\n}}\n")
    m = oracle.parse(text)
    assert str(m.functions["f"].types["r"]) == want


def test_F10_fig3_gradient_types():
    m = oracle.parse(W.FIG3)
    g, g3 = m.functions["foo_grad"], m.functions["foo_grad_3"]
    assert [str(t) for t in g.result_types] == ["<1 x 784 x f32>", "<784 x 10 x f32>", "<1 x 10 x f32>"]
    assert [str(t) for t in g3.param_types][-1] == "<1 x 10 x f32>"          # seed last
    assert [str(t) for t in g3.result_types] == ["<784 x 10 x f32>", "<1 x 10 x f32>", "<1 x 10 x f32>"]
    src = m.functions["foo"]
    p, r = oracle.expected_gradient_type(src, g3.gradient)
    assert p == g3.param_types and r == g3.result_types
    # a wrongly declared result arity is a verify error
    bad = W.FIG3.replace("-> (<784 x 10 x f32>, <1 x 10 x f32>, <1 x 10 x f32>)",
                         "-> (<784 x 10 x f32>, <1 x 10 x f32>)")
    with pytest.raises(VerifyError):
        oracle.parse(bad)


def test_F1_fig3_miniature():
    P = _pins()["F1_fig3_miniature"]
    text = W.FIG3.replace("784", "2").replace("10 x", "3 x")
    m = oracle.parse(text)
    x, w, b = (np.array(P[k], dtype=float) for k in ("x", "w", "b"))
    (foo,) = oracle.run(m, "foo", [x, w, b])
    np.testing.assert_array_equal(foo, P["foo"])
    dx, dw, db = oracle.run(m, "foo_grad", [x, w, b])
    np.testing.assert_array_equal(dx, P["dx"])
    np.testing.assert_array_equal(dw, P["dw"])
    np.testing.assert_array_equal(db, P["db"])
    # foo_grad_3 with seed 1: (dw, db, foo) (reading A7: grads then kept outputs)
    dw3, db3, kept = oracle.run(m, "foo_grad_3", [x, w, b, np.ones((1, 3))])
    np.testing.assert_array_equal(dw3, P["dw"])
    np.testing.assert_array_equal(db3, P["db"])
    np.testing.assert_array_equal(kept, P["foo"])


def test_F2_spec_foo_ones():
    m = oracle.parse(W.FIG3)
    (r,) = oracle.run(m, "foo", [np.ones((1, 784)), np.zeros((784, 10)), np.ones((1, 10))])
    np.testing.assert_array_equal(r, np.ones((1, 10)))


def _scalar_fn(body, ty="f32"):
    return (f'module "s"\nstage raw\nfunc @f: ({ty}) -> {ty} {{\n'
            f"'entry(%z: {ty}):\n{body}\n}}\n[gradient @f]\nfunc @df: ({ty}) -> {ty}\n")


SIGMOID = ("    %n = negate %z: f32\n    %e = exp %n: f32\n    %d = add %e: f32, 1: f32\n"
           "    %h = divide 1: f32, %d: f32\n    return %h: f32")


def test_F3_sigmoid_tanh_at_zero():
    m = oracle.parse(_scalar_fn(SIGMOID))
    assert oracle.run(m, "f", [0.0])[0] == 0.5
    assert oracle.run(m, "df", [0.0])[0] == 0.25
    m = oracle.parse(_scalar_fn("    %h = tanh %z: f32\n    return %h: f32"))
    assert oracle.run(m, "f", [0.0])[0] == 0.0
    assert oracle.run(m, "df", [0.0])[0] == 1.0


def test_sigmoid_closed_form_derivative():
    """north_star: sigma' = sigma (1 - sigma); tanh' = 1 - tanh^2, at many z."""
    ms = oracle.parse(_scalar_fn(SIGMOID))
    mt = oracle.parse(_scalar_fn("    %h = tanh %z: f32\n    return %h: f32"))
    for z in np.linspace(-8, 8, 41):
        s = 1.0 / (1.0 + np.exp(-z))
        assert abs(oracle.run(ms, "df", [z])[0] - s * (1 - s)) <= 1e-15
        assert abs(oracle.run(mt, "df", [z])[0] - (1 - np.tanh(z) ** 2)) <= 1e-15


def test_F4_relu():
    T, TB = "<1 x 3 x f32>", "<1 x 3 x bool>"
    text = (f'module "r"\nstage raw\nfunc @f: ({T}) -> {T} {{\n'
            f"'entry(%z: {T}):\n    %c = gt %z: {T}, 0: f32\n"
            f"    %h = select %c: {TB}, %z: {T}, 0: f32\n    return %h: {T}\n}}\n"
            f"[gradient @f]\nfunc @df: ({T}) -> {T}\n")
    m = oracle.parse(text)
    z = np.array([[-1.0, 0.0, 2.0]])
    np.testing.assert_array_equal(oracle.run(m, "f", [z])[0], [[0, 0, 2]])
    np.testing.assert_array_equal(oracle.run(m, "df", [z])[0], [[0, 0, 1]])   # A11: 0 at z=0


def test_F5_broadcast_add_unbroadcast():
    A, V = "<2 x 3 x f32>", "<1 x 3 x f32>"
    text = (f'module "b"\nstage raw\nfunc @f: ({A}, {V}) -> {A} {{\n'
            f"'entry(%a: {A}, %v: {V}):\n    %r = add %a: {A}, %v: {V}\n    return %r: {A}\n}}\n"
            f"[gradient @f]\nfunc @df: ({A}, {V}) -> ({A}, {V})\n")
    m = oracle.parse(text)
    a = np.array([[1.0, 2, 3], [4, 5, 6]])
    v = np.array([[10.0, 20, 30]])
    np.testing.assert_array_equal(oracle.run(m, "f", [a, v])[0], [[11, 22, 33], [14, 25, 36]])
    da, dv = oracle.run(m, "df", [a, v])
    np.testing.assert_array_equal(da, np.ones((2, 3)))
    np.testing.assert_array_equal(dv, [[2, 2, 2]])


def test_F6_reduce():
    A = "<2 x 3 x f32>"
    for axis, want, rt in ((1, [6, 15], "<2 x f32>"), (0, [5, 7, 9], "<3 x f32>")):
        text = (f'module "r"\nstage raw\nfunc @f: ({A}) -> {rt} {{\n'
                f"'entry(%a: {A}):\n    %r = reduce %a: {A} by add along {axis}\n"
                f"    return %r: {rt}\n}}\n[gradient @f seedable]\nfunc @df: ({A}, {rt}) -> {A}\n")
        m = oracle.parse(text)
        a = np.array([[1.0, 2, 3], [4, 5, 6]])
        np.testing.assert_array_equal(oracle.run(m, "f", [a])[0], want)
        seed = np.ones(len(want))
        np.testing.assert_array_equal(oracle.run(m, "df", [a, seed])[0], np.ones((2, 3)))


def _mlp_text(batch, layers):
    return W.mlp_ir(batch, layers)


def test_F7_mse():
    P = _pins()["F7_mse"]
    text = _mlp_text(1, [(1, 1, None)])
    m = oracle.parse(text)
    # identity layer: y = x*1 + 0
    x, w, b, t = np.array(P["y"]), np.ones((1, 1)), np.zeros((1, 1)), np.array(P["t"])
    assert oracle.run(m, "mlp", [x, w, b, t])[0] == P["L"]
    src = m.functions["mlp"]
    (dx,) = oracle.grad(src, [x, w, b, t], wrt=[0])
    np.testing.assert_array_equal(dx, P["dL_dy"])


def test_F8_221_sigmoid_mlp():
    P = _pins()["F8_221_sigmoid_mlp"]
    m = oracle.parse(_mlp_text(1, [(2, 2, "sigmoid"), (2, 1, "sigmoid")]))
    ins = [np.array(P[k], dtype=float) for k in ("x", "w1", "b1", "w2", "b2", "t")]
    L = oracle.run(m, "mlp", ins)[0]
    assert L == P["L"]
    dw1, db1, dw2, db2, kept = oracle.run(m, "mlp_grad", ins + [np.float64(1.0)])
    np.testing.assert_array_equal(dw1, P["dw1"])
    np.testing.assert_array_equal(db1, P["db1"])
    np.testing.assert_array_equal(dw2, P["dw2"])
    np.testing.assert_array_equal(db2, P["db2"])
    assert kept == P["L"]


def test_F11_fig4_fd():
    m = oracle.parse(W.fig4_ir())
    rng = np.random.default_rng(0)
    src = m.functions["g"]
    ins = [rng.uniform(-1, 1, t.shape) for t in src.param_types]
    dw, db, kept = oracle.run(m, "dg", ins)
    np.testing.assert_allclose(dw, oracle.fd_grad(src, ins, 1), rtol=1e-5, atol=1e-8)
    np.testing.assert_allclose(db, oracle.fd_grad(src, ins, 2), rtol=1e-5, atol=1e-8)
    np.testing.assert_array_equal(kept, oracle.run(m, "g", ins)[0])


def test_F12_seed_scaling_bit_exact():
    w = W.c1(4)
    m = oracle.parse(w.text)
    ins = [x.astype(np.float64) for x in w.inputs()]
    g1 = oracle.run(m, "mlp_grad", ins + [np.float64(0.25)])
    for k in (-3, 1, 5):
        gk = oracle.run(m, "mlp_grad", ins + [np.float64(0.25 * 2.0 ** k)])
        for a, b in zip(g1[:-1], gk[:-1]):
            np.testing.assert_array_equal(a * 2.0 ** k, b)


# --- F14: finite differences on every adjoint rule --------

UN = ["negate", "tanh", "exp", "log", "sqrt", "abs"]
BIN = ["add", "subtract", "multiply", "divide", "power"]


def _fd_check(text, fname, ins, wrts):
    m = oracle.parse(text)
    src = m.functions[fname]
    seed = np.random.default_rng(7).uniform(-1, 1, src.result_types[0].shape)
    gs = oracle.grad(src, ins, wrt=wrts, seed=seed)
    for i, g in zip(wrts, gs):
        fd = oracle.fd_grad(src, ins, i, seed=seed)
        np.testing.assert_allclose(g, fd, rtol=1e-5, atol=1e-8)


@pytest.mark.parametrize("op", UN)
def test_F14_fd_unary(op):
    T = "<3 x 4 x f32>"
    text = f'module "u"\nstage raw\nfunc @f: ({T}) -> {T} {{\n\'entry(%a: {T}):\n    %r = {op} %a: {T}\n    return %r: {T}\n}}\n'
    rng = np.random.default_rng(1)
    a = rng.uniform(0.2, 2.0, (3, 4)) * (1 if op in ("log", "sqrt") else rng.choice([-1, 1], (3, 4)))
    _fd_check(text, "f", [a], [0])


@pytest.mark.parametrize("op", BIN)
@pytest.mark.parametrize("sa,sb", [((3, 4), (3, 4)), ((3, 4), (1, 4)), ((3, 1), (1, 4)), ((2, 3, 4), (4,))])
def test_F14_fd_binary_broadcast(op, sa, sb):
    ty = lambda s: "<" + " x ".join(map(str, s)) + " x f32>"
    from oracle.infer import broadcast_shapes
    rs = broadcast_shapes(sa, sb)
    text = (f'module "b"\nstage raw\nfunc @f: ({ty(sa)}, {ty(sb)}) -> {ty(rs)} {{\n'
            f"'entry(%a: {ty(sa)}, %b: {ty(sb)}):\n    %r = {op} %a: {ty(sa)}, %b: {ty(sb)}\n"
            f"    return %r: {ty(rs)}\n}}\n")
    rng = np.random.default_rng(2)
    a = rng.uniform(0.5, 2.0, sa)
    b = rng.uniform(0.5, 2.0, sb) * (1 if op == "power" else rng.choice([-1, 1], sb))
    _fd_check(text, "f", [a, b], [0, 1])


def test_F14_fd_dot_transpose_reduce_shapecast_select():
    text = '''module "m"
stage raw
func @f: (<3 x 5 x f32>, <4 x 5 x f32>, <1 x 4 x f32>) -> <4 x f32> {
'entry(%a: <3 x 5 x f32>, %w: <4 x 5 x f32>, %v: <1 x 4 x f32>):
    %t = transpose %w: <4 x 5 x f32>
    %d = dot %a: <3 x 5 x f32>, %t: <5 x 4 x f32>
    %c = gt %d: <3 x 4 x f32>, %v: <1 x 4 x f32>
    %s = select %c: <3 x 4 x bool>, %d: <3 x 4 x f32>, %v: <1 x 4 x f32>
    %q = multiply %s: <3 x 4 x f32>, %s: <3 x 4 x f32>
    %r = reduce %q: <3 x 4 x f32> by add along 0
    %k = shapeCast %r: <4 x f32> to 2 x 2
    %e = exp %k: <2 x 2 x f32>
    %o = shapeCast %e: <2 x 2 x f32> to 4
    return %o: <4 x f32>
}
'''
    rng = np.random.default_rng(3)
    ins = [rng.uniform(-1, 1, (3, 5)) * 0.5, rng.uniform(-1, 1, (4, 5)) * 0.5, rng.uniform(-1, 1, (1, 4)) * 0.3]
    _fd_check(text, "f", ins, [0, 1, 2])


def test_F14_fd_slice():
    text = '''module "s"
stage raw
func @f: (<5 x 3 x f32>) -> <2 x 3 x f32> {
'entry(%a: <5 x 3 x f32>):
    %s = slice %a: <5 x 3 x f32> from 1 upto 3
    %t = tanh %s: <2 x 3 x f32>
    return %t: <2 x 3 x f32>
}
'''
    _fd_check(text, "f", [np.random.default_rng(4).uniform(-1, 1, (5, 3))], [0])


def test_F14_fd_c1_mlp_all_params():
    w = W.c1(3)
    m = oracle.parse(w.text)
    src = m.functions["mlp"]
    ins = [x.astype(np.float64) for x in w.inputs()]
    # shrink the FD cost: check W2/b2/b1 fully and a slice of W1 via seed-weighted FD
    gs = oracle.grad(src, ins, wrt=[2, 3, 4])
    for i, g in zip([2, 3, 4], gs):
        np.testing.assert_allclose(g, oracle.fd_grad(src, ins, i), rtol=1e-5, atol=1e-8)


def test_F15_dp_semantics():
    """Global-batch gradient == sum over row shards (seed 1/B_global)."""
    wg = W.c3(8, layers=[(6, 5, "relu"), (5, 4, None)])
    m = oracle.parse(wg.text)
    ins = [x.astype(np.float64) for x in wg.inputs()]
    full = oracle.run(m, "mlp_grad", ins + [np.float64(1 / 8)])
    ws = W.c3(4, layers=[(6, 5, "relu"), (5, 4, None)])
    ms = oracle.parse(ws.text)
    parts = []
    for r in range(2):
        si = list(ins)
        si[0] = ins[0][4 * r:4 * r + 4]
        si[-1] = ins[-1][4 * r:4 * r + 4]
        parts.append(oracle.run(ms, "mlp_grad", si + [np.float64(1 / 8)]))
    for k in range(len(full) - 1):
        np.testing.assert_allclose(full[k], parts[0][k] + parts[1][k], rtol=1e-12, atol=1e-15)


# --- shape rules -----------------------------------------------------------

def test_broadcast_rule_examples():
    from oracle.infer import broadcast_shapes
    assert broadcast_shapes((3, 1, 5), (4, 5)) == (3, 4, 5)
    assert broadcast_shapes((10, 20), (1, 20)) == (10, 20)         # Table 1
    assert broadcast_shapes((), (2, 3)) == (2, 3)
    with pytest.raises(ValueError):
        broadcast_shapes((3,), (4,))


def test_broadcast_vs_materialised_expansion():
    """Broadcast coherence: index-broadcast == explicit expansion."""
    rng = np.random.default_rng(5)
    for sa, sb in [((3, 1, 5), (4, 5)), ((2, 1), (1, 3)), ((4,), (2, 3, 4))]:
        from oracle.infer import broadcast_shapes
        rs = broadcast_shapes(sa, sb)
        ty = lambda s: "<" + " x ".join(map(str, s)) + " x f32>"
        text = (f'module "b"\nstage raw\nfunc @f: ({ty(sa)}, {ty(sb)}) -> {ty(rs)} {{\n'
                f"'entry(%a: {ty(sa)}, %b: {ty(sb)}):\n    %r = subtract %a: {ty(sa)}, %b: {ty(sb)}\n"
                f"    return %r: {ty(rs)}\n}}\n")
        a, b = rng.normal(size=sa), rng.normal(size=sb)
        (r,) = oracle.run(oracle.parse(text), "f", [a, b])
        want = np.empty(rs)
        for idx in itertools.product(*[range(d) for d in rs]):
            ia = tuple(i if d > 1 else 0 for i, d in zip(idx[len(rs) - len(sa):], sa))
            ib = tuple(i if d > 1 else 0 for i, d in zip(idx[len(rs) - len(sb):], sb))
            want[idx] = a[ia] - b[ib]
        np.testing.assert_array_equal(r, want)


def test_dot_vs_triple_loop():
    rng = np.random.default_rng(6)
    a, b = rng.normal(size=(3, 7)), rng.normal(size=(7, 2))
    text = ('module "d"\nstage raw\nfunc @f: (<3 x 7 x f32>, <7 x 2 x f32>) -> <3 x 2 x f32> {\n'
            "'entry(%a: <3 x 7 x f32>, %b: <7 x 2 x f32>):\n    %r = dot %a: <3 x 7 x f32>, %b: <7 x 2 x f32>\n"
            "    return %r: <3 x 2 x f32>\n}\n")
    (r,) = oracle.run(oracle.parse(text), "f", [a, b])
    want = np.zeros((3, 2))
    for i in range(3):
        for j in range(2):
            for k in range(7):
                want[i, j] += a[i, k] * b[k, j]
    np.testing.assert_allclose(r, want, rtol=1e-14, atol=1e-14)


BAD_PARSE = [
    'module "m"\nstage raw\nfunc @f: (f32) -> f32 {\n\'entry(%a: f32):\n    %r = frobnicate %a: f32\n    return %r: f32\n}\n',
    'module "m"\nstage raw\nfunc @f: (<2 x f32>) -> <2 x f32> {\n\'entry(%a: <2 x f32>):\n    %r = dot %a: <2 x f32>\n    return %r: <2 x f32>\n}\n',
    'module "m"\nstage cooked\n',
    'module "m"\nstage raw\nfunc @f: (<2 x f32) -> f32\n',
]

BAD_VERIFY = [
    # broadcast mismatch [3] vs [4]
    'module "m"\nstage raw\nfunc @f: (<3 x f32>, <4 x f32>) -> <3 x f32> {\n\'entry(%a: <3 x f32>, %b: <4 x f32>):\n    %r = add %a: <3 x f32>, %b: <4 x f32>\n    return %r: <3 x f32>\n}\n',
    # dot inner mismatch
    'module "m"\nstage raw\nfunc @f: (<2 x 3 x f32>, <4 x 2 x f32>) -> <2 x 2 x f32> {\n\'entry(%a: <2 x 3 x f32>, %b: <4 x 2 x f32>):\n    %r = dot %a: <2 x 3 x f32>, %b: <4 x 2 x f32>\n    return %r: <2 x 2 x f32>\n}\n',
    # annotation mismatch
    'module "m"\nstage raw\nfunc @f: (<2 x f32>) -> <2 x f32> {\n\'entry(%a: <2 x f32>):\n    %r = tanh %a: <3 x f32>\n    return %r: <2 x f32>\n}\n',
    # use before def
    'module "m"\nstage raw\nfunc @f: (<2 x f32>) -> <2 x f32> {\n\'entry(%a: <2 x f32>):\n    %r = tanh %q: <2 x f32>\n    return %r: <2 x f32>\n}\n',
    # wrong return type
    'module "m"\nstage raw\nfunc @f: (<2 x f32>) -> <3 x f32> {\n\'entry(%a: <2 x f32>):\n    %r = tanh %a: <2 x f32>\n    return %r: <2 x f32>\n}\n',
    # shapeCast count
    'module "m"\nstage raw\nfunc @f: (<2 x 3 x f32>) -> <5 x f32> {\n\'entry(%a: <2 x 3 x f32>):\n    %r = shapeCast %a: <2 x 3 x f32> to 5\n    return %r: <5 x f32>\n}\n',
    # reduce axis out of range
    'module "m"\nstage raw\nfunc @f: (<2 x 3 x f32>) -> <2 x f32> {\n\'entry(%a: <2 x 3 x f32>):\n    %r = reduce %a: <2 x 3 x f32> by add along 2\n    return %r: <2 x f32>\n}\n',
    # wrt an integer argument
    'module "m"\nstage raw\nfunc @f: (<2 x i32>) -> <2 x i32> {\n\'entry(%a: <2 x i32>):\n    %r = negate %a: <2 x i32>\n    return %r: <2 x i32>\n}\n[gradient @f]\nfunc @g: (<2 x i32>) -> <2 x i32>\n',
    # reduce-multiply on the active path
    'module "m"\nstage raw\nfunc @f: (<2 x f32>) -> f32 {\n\'entry(%a: <2 x f32>):\n    %r = reduce %a: <2 x f32> by multiply along 0\n    return %r: f32\n}\n[gradient @f]\nfunc @g: (<2 x f32>) -> <2 x f32>\n',
    # wrt index out of range
    'module "m"\nstage raw\nfunc @f: (<2 x f32>) -> <2 x f32> {\n\'entry(%a: <2 x f32>):\n    %r = tanh %a: <2 x f32>\n    return %r: <2 x f32>\n}\n[gradient @f wrt 1]\nfunc @g: (<2 x f32>) -> <2 x f32>\n',
]


@pytest.mark.parametrize("text", BAD_PARSE)
def test_parse_errors(text):
    with pytest.raises(ParseError):
        oracle.parse(text)


@pytest.mark.parametrize("text", BAD_VERIFY)
def test_verify_errors(text):
    with pytest.raises(VerifyError):
        oracle.parse(text)


# --- bf16 policy helper (reading A15) ---------------------------------------

def test_bf16_round_ties_to_even_and_torch():
    from oracle.interp import bf16_round
    one = 1.0
    assert bf16_round(np.array([one]))[0] == 1.0
    assert bf16_round(np.array([1 + 2.0 ** -8]))[0] == 1.0                  # tie -> even (down)
    assert bf16_round(np.array([1 + 3 * 2.0 ** -8]))[0] == 1 + 2.0 ** -6    # tie -> even (up)
    assert bf16_round(np.array([1 + 2.0 ** -8 + 2.0 ** -20]))[0] == 1 + 2.0 ** -7
    import torch
    x = np.random.default_rng(9).standard_normal(10000) * 10.0 ** np.random.default_rng(8).integers(-30, 30, 10000)
    want = torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16).to(torch.float64).numpy()
    np.testing.assert_array_equal(bf16_round(x), want)


def test_bf16_policy_dot_exact_on_bf16_inputs():
    """Under the bf16 policy a dot of bf16-representable operands equals the
    unrounded dot (rounding is then the identity)."""
    from oracle.interp import bf16_round
    rng = np.random.default_rng(10)
    a, b = bf16_round(rng.normal(size=(4, 6))), bf16_round(rng.normal(size=(6, 3)))
    text = ('module "d"\nstage raw\nfunc @f: (<4 x 6 x f32>, <6 x 3 x f32>) -> <4 x 3 x f32> {\n'
            "'entry(%a: <4 x 6 x f32>, %b: <6 x 3 x f32>):\n    %r = dot %a: <4 x 6 x f32>, %b: <6 x 3 x f32>\n"
            "    return %r: <4 x 3 x f32>\n}\n")
    m = oracle.parse(text)
    np.testing.assert_array_equal(oracle.run(m, "f", [a, b], dot_policy="bf16")[0], a @ b)
    c = a + 1e-3  # not bf16-representable: the policy result differs from the exact one
    assert not np.array_equal(oracle.run(m, "f", [c, b], dot_policy="bf16")[0], c @ b)
    np.testing.assert_array_equal(oracle.run(m, "f", [c, b], dot_policy="bf16")[0], bf16_round(c) @ b)


def _prod_module(shape, axis):
    rt = [d for k, d in enumerate(shape) if k != axis]
    T = lambda s: "<" + " x ".join(str(d) for d in s) + " x f32>" if s else "f32"
    return oracle.parse(f'module "m"\nstage raw\nfunc @f: ({T(shape)}) -> {T(rt)} {{\n'
                        f"'entry(%a: {T(shape)}):\n"
                        f"    %r = reduce %a: {T(shape)} by multiply along {axis}\n"
                        f"    return %r: {T(rt)}\n}}\n")


def test_reduce_multiply_forward_pins():
    """`reduce ... by multiply along d` (Table 1): the product
    over axis d, axis removed.  Pinned by hand-computed values, brute force
    over indices, and the identity prod(exp x) = exp(sum x) along the axis."""
    a = np.array([[1.0, 2.0, 3.0], [4.0, 5.0, 6.0]])
    np.testing.assert_array_equal(oracle.run(_prod_module((2, 3), 0), "f", [a])[0], [4.0, 10.0, 18.0])
    np.testing.assert_array_equal(oracle.run(_prod_module((2, 3), 1), "f", [a])[0], [6.0, 120.0])
    assert float(oracle.run(_prod_module((4,), 0), "f", [np.array([1.5, -2.0, 0.5, 4.0])])[0]) == -6.0
    rng = np.random.default_rng(7)
    x = rng.uniform(-1, 1, (3, 4, 5))
    for ax in range(3):
        got = oracle.run(_prod_module(x.shape, ax), "f", [x])[0]
        rest = [d for k, d in enumerate(x.shape) if k != ax]
        for idx in itertools.product(*[range(d) for d in rest]):
            p = 1.0
            for t in range(x.shape[ax]):
                full = list(idx)
                full.insert(ax, t)
                p *= x[tuple(full)]
            assert got[idx] == pytest.approx(p, rel=1e-14, abs=0)
        e = oracle.run(_prod_module(x.shape, ax), "f", [np.exp(x)])[0]
        np.testing.assert_allclose(e, np.exp(x.sum(axis=ax)), rtol=1e-13)
