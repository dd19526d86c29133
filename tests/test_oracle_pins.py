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

UN = ["negate", "tanh", "exp", "log", "sqrt", "abs", "sign"]
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


# --- bf16-policy VJP (reading A15, A18'): pinned by triple loops ---
#
# Under the bf16 dot policy every `dot` -- the forward ones and the two dots of
# each `dot` adjoint (dot(g, transpose b), dot(transpose a, g)) --
# rounds its operands RNE to bf16 (from their f32 value) and accumulates the
# exact products; element-wise math is not rounded.  The expected values below
# are written with torch's bf16 conversion (an implementation independent of
# oracle.interp.bf16_round) and Python triple loops.

def _tbf16(a):
    import torch
    t = torch.from_numpy(np.asarray(a, dtype=np.float64)).to(torch.float32).to(torch.bfloat16)
    return t.to(torch.float64).numpy()


def _loop_matmul(a, b):
    m, k = a.shape
    k2, n = b.shape
    assert k == k2
    out = np.zeros((m, n))
    for i in range(m):
        for j in range(n):
            s = 0.0
            for t in range(k):
                s += a[i, t] * b[t, j]
            out[i, j] = s
    return out


def _dot_grad_text(M, K, N):
    A, B, Y = f"<{M} x {K} x f32>", f"<{K} x {N} x f32>", f"<{M} x {N} x f32>"
    return (f'module "p"\nstage raw\nfunc @f: ({A}, {B}) -> {Y} {{\n'
            f"'entry(%x: {A}, %w: {B}):\n    %y = dot %x: {A}, %w: {B}\n    return %y: {Y}\n}}\n\n"
            f"[gradient @f wrt 0, 1 seedable]\nfunc @g: ({A}, {B}, {Y}) -> ({A}, {B})\n")


def test_bf16_policy_dot_vjp_rounds_operands_and_seed():
    """One `dot` with a seed that is not bf16-representable (1/3 and random
    values): dX = bf16(g)·bf16(W)ᵀ and dW = bf16(x)ᵀ·bf16(g) by triple loops.
    Not rounding g, or rounding the products instead of the operands, moves
    the result by ~1e-3 relative and fails the 1e-12 check."""
    M, K, N = 3, 5, 4
    m = oracle.parse(_dot_grad_text(M, K, N))
    rng = np.random.default_rng(41)
    x, w = rng.normal(size=(M, K)), rng.normal(size=(K, N))
    for g in (np.full((M, N), 1.0 / 3.0), rng.normal(size=(M, N))):
        dx, dw = oracle.run(m, "g", [x, w, g], dot_policy="bf16")
        want_dx = _loop_matmul(_tbf16(g), _tbf16(w).T)
        want_dw = _loop_matmul(_tbf16(x).T, _tbf16(g))
        np.testing.assert_allclose(dx, want_dx, rtol=1e-12, atol=0)
        np.testing.assert_allclose(dw, want_dw, rtol=1e-12, atol=0)
        # the unrounded VJP is measurably different (the policy is not a no-op)
        ux, uw = oracle.run(m, "g", [x, w, g])
        assert np.max(np.abs(uw - want_dw)) > 1e-5 * np.max(np.abs(want_dw))


def test_bf16_policy_two_layer_vjp_by_hand():
    """z = x·W1, h = tanh z, y = h·W2 under the bf16 policy with seed g:
    dW2 = bf16(h)ᵀ·bf16(g), dh = bf16(g)·bf16(W2)ᵀ (not rounded: it is
    element-wise input), dz = dh ⊙ (1 − h²) with h = tanh(bf16(x)·bf16(W1)),
    dW1 = bf16(x)ᵀ·bf16(dz).  Triple loops; the adjoint dZ is rounded where
    it enters the weight-gradient dot, as the GPU stores it (bf16)."""
    B, I, H, O = 4, 6, 5, 3
    X, W1, W2, Z, Y = (f"<{B} x {I} x f32>", f"<{I} x {H} x f32>", f"<{H} x {O} x f32>",
                       f"<{B} x {H} x f32>", f"<{B} x {O} x f32>")
    text = (f'module "p"\nstage raw\nfunc @f: ({X}, {W1}, {W2}) -> {Y} {{\n'
            f"'entry(%x: {X}, %w1: {W1}, %w2: {W2}):\n"
            f"    %z = dot %x: {X}, %w1: {W1}\n    %h = tanh %z: {Z}\n"
            f"    %y = dot %h: {Z}, %w2: {W2}\n    return %y: {Y}\n}}\n\n"
            f"[gradient @f wrt 1, 2 seedable]\nfunc @g: ({X}, {W1}, {W2}, {Y}) -> ({W1}, {W2})\n")
    m = oracle.parse(text)
    rng = np.random.default_rng(43)
    x, w1, w2 = rng.normal(size=(B, I)), rng.normal(size=(I, H)) * 0.5, rng.normal(size=(H, O))
    g = np.full((B, O), 1.0 / 3.0) + rng.normal(size=(B, O)) * 0.1
    dw1, dw2 = oracle.run(m, "g", [x, w1, w2, g], dot_policy="bf16")
    h = np.tanh(_loop_matmul(_tbf16(x), _tbf16(w1)))
    want_dw2 = _loop_matmul(_tbf16(h).T, _tbf16(g))
    dh = _loop_matmul(_tbf16(g), _tbf16(w2).T)
    dz = dh * (1.0 - h * h)
    want_dw1 = _loop_matmul(_tbf16(x).T, _tbf16(dz))
    np.testing.assert_allclose(dw2, want_dw2, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(dw1, want_dw1, rtol=1e-12, atol=1e-15)
    # and its forward loss under the policy
    (y,) = oracle.run(m, "f", [x, w1, w2], dot_policy="bf16")
    np.testing.assert_allclose(y, _loop_matmul(_tbf16(h), _tbf16(w2)), rtol=1e-12, atol=1e-15)


def test_bf16_policy_vjp_equals_plain_vjp_on_dyadic_data():
    """On bf16-exact dyadic inputs and seed every rounding is the identity and
    every product and sum is exact in f64: policy VJP == plain VJP, bit for bit."""
    M, K, N = 4, 6, 3
    m = oracle.parse(_dot_grad_text(M, K, N))
    rng = np.random.default_rng(47)
    vals = np.array([-2.0, -1.0, -0.5, -0.25, 0.0, 0.25, 0.5, 1.0, 1.5, 2.0])
    x, w, g = (rng.choice(vals, size=s) for s in ((M, K), (K, N), (M, N)))
    pol = oracle.run(m, "g", [x, w, g], dot_policy="bf16")
    plain = oracle.run(m, "g", [x, w, g])
    for a, b in zip(pol, plain):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(plain[0], _loop_matmul(g, w.T))
    np.testing.assert_array_equal(plain[1], _loop_matmul(x.T, g))


def test_F14_fd_sign():
    """sign has derivative 0 away from 0 (S:L338 via S:L365): FD of
    sum(seed * sign(a) * a) = sum(seed * |a|) must equal seed * sign(a),
    which needs the sign rule to contribute exactly 0 (a wrong rule that
    passes g through would add seed * a)."""
    T = "<3 x 4 x f32>"
    text = (f'module "s"\nstage raw\nfunc @f: ({T}) -> {T} {{\n\'entry(%a: {T}):\n'
            f"    %s = sign %a: {T}\n    %r = multiply %s: {T}, %a: {T}\n    return %r: {T}\n}}\n")
    rng = np.random.default_rng(5)
    a = rng.uniform(0.2, 2.0, (3, 4)) * rng.choice([-1, 1], (3, 4))
    _fd_check(text, "f", [a], [0])
    src = oracle.parse(text).functions["f"]
    seed = np.random.default_rng(7).uniform(-1, 1, (3, 4))
    (g,) = oracle.grad(src, [a], wrt=[0], seed=seed)
    np.testing.assert_allclose(g, seed * np.sign(a), rtol=1e-14, atol=0)
    # the sign rule alone is zero
    t2 = f'module "s"\nstage raw\nfunc @f: ({T}) -> {T} {{\n\'entry(%a: {T}):\n    %s = sign %a: {T}\n    return %s: {T}\n}}\n'
    (g0,) = oracle.grad(oracle.parse(t2).functions["f"], [a], wrt=[0], seed=seed)
    np.testing.assert_array_equal(g0, np.zeros((3, 4)))
    _fd_check(t2, "f", [a], [0])


def test_F14_fd_dataTypeCast_f32_to_f64():
    """dataTypeCast between float types is the identity on values (the
    oracle evaluates both in float64), so its adjoint passes the incoming
    adjoint through (cast back to the operand type): FD of
    sum(seed * tanh(cast(a))^2)."""
    T, T64 = "<3 x 4 x f32>", "<3 x 4 x f64>"
    text = (f'module "c"\nstage raw\nfunc @f: ({T}) -> {T64} {{\n\'entry(%a: {T}):\n'
            f"    %c = dataTypeCast %a: {T} to f64\n    %t = tanh %c: {T64}\n"
            f"    %r = multiply %t: {T64}, %t: {T64}\n    return %r: {T64}\n}}\n")
    a = np.random.default_rng(6).uniform(-1.5, 1.5, (3, 4))
    _fd_check(text, "f", [a], [0])
    src = oracle.parse(text).functions["f"]
    (g,) = oracle.grad(src, [a], wrt=[0])
    np.testing.assert_allclose(g, 2 * np.tanh(a) * (1 - np.tanh(a) ** 2), rtol=1e-14)


# --- `reduce ... by max` (extension, reading A26) and softmax cross-entropy --

def _max_module(shape, axis, grad=True):
    rt = [d for k, d in enumerate(shape) if k != axis]
    T = lambda s: "<" + " x ".join(str(d) for d in s) + " x f32>" if s else "f32"
    text = (f'module "m"\nstage raw\nfunc @f: ({T(shape)}) -> {T(rt)} {{\n'
            f"'entry(%a: {T(shape)}):\n    %r = reduce %a: {T(shape)} by max along {axis}\n"
            f"    return %r: {T(rt)}\n}}\n")
    if grad:
        text += f"\n[gradient @f wrt 0 seedable]\nfunc @g: ({T(shape)}, {T(rt)}) -> {T(shape)}\n"
    return oracle.parse(text)


def test_reduce_max_forward_pins():
    """max over the axis, axis removed: hand values and brute force."""
    a = np.array([[1.0, -2.0, 3.0], [4.0, 5.0, -6.0]])
    np.testing.assert_array_equal(oracle.run(_max_module((2, 3), 0), "f", [a])[0], [4.0, 5.0, 3.0])
    np.testing.assert_array_equal(oracle.run(_max_module((2, 3), 1), "f", [a])[0], [3.0, 5.0])
    assert float(oracle.run(_max_module((4,), 0), "f", [np.array([-1.5, -2.0, -0.5, -4.0])])[0]) == -0.5
    x = np.random.default_rng(17).uniform(-1, 1, (3, 4, 5))
    for ax in range(3):
        got = oracle.run(_max_module(x.shape, ax), "f", [x])[0]
        rest = [d for k, d in enumerate(x.shape) if k != ax]
        for idx in itertools.product(*[range(d) for d in rest]):
            best = -np.inf
            for t in range(x.shape[ax]):
                full = list(idx)
                full.insert(ax, t)
                best = x[tuple(full)] if x[tuple(full)] > best else best
            assert got[idx] == best


def test_reduce_max_adjoint_ties_split_and_fd():
    """Reading A26: the incoming adjoint goes to the position(s) attaining
    the max, split equally among ties; away from ties it is the derivative
    (central differences)."""
    m = _max_module((2, 3), 1)
    a = np.array([[1.0, 3.0, 3.0], [2.0, 0.0, -1.0]])
    (g,) = oracle.run(m, "g", [a, np.array([1.0, 4.0])])
    np.testing.assert_array_equal(g, [[0.0, 0.5, 0.5], [4.0, 0.0, 0.0]])
    (g2,) = oracle.run(_max_module((2, 3), 0), "g", [a, np.array([1.0, 2.0, 3.0])])
    np.testing.assert_array_equal(g2, [[0.0, 2.0, 3.0], [1.0, 0.0, 0.0]])
    x = np.random.default_rng(19).uniform(-1, 1, (4, 5))
    for ax in (0, 1):
        mm = _max_module((4, 5), ax)
        seed = np.random.default_rng(23).uniform(-1, 1, mm.functions["f"].result_types[0].shape)
        (gx,) = oracle.run(mm, "g", [x, seed])
        np.testing.assert_allclose(gx, oracle.fd_grad(mm.functions["f"], [x], 0, seed=seed), rtol=1e-5, atol=1e-8)
        # the IR adjoint (oracle.canonical) equals the value-level sweep, ties included
        from oracle.interp import run_function
        xt = x.copy()
        xt[1] = xt[0] if ax == 0 else xt[1]
        xt[:, 2] = xt[:, 3] if ax == 1 else xt[:, 2]
        for inp in (x, xt):
            np.testing.assert_allclose(run_function(oracle.canonical(mm, "g"), [inp, seed])[0],
                                       oracle.run(mm, "g", [inp, seed])[0], rtol=1e-15, atol=0)


def test_softmax_cross_entropy_gradient_closed_form():
    """softmax-CE built from primitives with the max shift (workloads.mlp_ir
    loss="ce"): L = sum_b (logsumexp(y_b) - y_b . t_b) and dL/dy = softmax(y)
    - t, so for a linear last layer y = h.W + b: dW = h^T (softmax(y) - t),
    db = sum_b (softmax(y) - t) -- checked against the closed form."""
    w = W.ce_mlp(5, layers=[(6, 4, None)], dot_precision="f32")
    m = oracle.parse(w.text)
    x, W1, b1, t = [a.astype(np.float64) for a in w.inputs()]
    y = x @ W1 + b1
    e = np.exp(y - y.max(axis=1, keepdims=True))
    p = e / e.sum(axis=1, keepdims=True)
    L_ref = float(np.sum(np.log(np.exp(y).sum(axis=1)) - (y * t).sum(axis=1)))
    assert abs(float(oracle.run(m, "mlp", [x, W1, b1, t])[0]) - L_ref) <= 1e-12 * abs(L_ref)
    dW, db, L = oracle.run(m, "mlp_grad", [x, W1, b1, t, np.float64(1.0)])
    np.testing.assert_allclose(dW, x.T @ (p - t), rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(db, (p - t).sum(axis=0, keepdims=True), rtol=1e-12, atol=1e-14)
    # large logits: the max shift keeps the forward finite where exp(y) overflows
    big = [x * 300.0, W1, b1, t]
    assert np.isfinite(oracle.run(m, "mlp", big)[0])
