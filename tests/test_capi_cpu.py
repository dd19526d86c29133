"""CPU checks of the native library (no GPU needed): the C ABI loads and
exports every entry point declared in include/dlvm.h; the C++ front end
(parser, type/broadcast inference, verifier, AD, DCE) agrees with the
oracle -- types bit-exact, error classes equal, and the generated adjoint
IR, interpreted by the oracle in float64, equals the oracle's own
vector-Jacobian product (SURVEY.md §4 tier T1/T6)."""

import ctypes
import os
import re
import subprocess
import sys

import numpy as np
import pytest

import oracle
import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

P = pytest.importorskip("paper_1711_03016_b200")


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "dlvm.h")).read()
    declared = sorted(set(re.findall(r"\b(dlvm_\w+)\s*\(", hdr)))
    assert len(declared) >= 12, declared
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_1711_03016_b200", "libdlvm.so"))
    for name in declared:
        assert hasattr(lib, name), f"libdlvm.so does not export {name}"
    assert sorted(P.dlvm.EXPORTS) == declared
    assert P.dlvm_version().startswith("dlvm-b200")


def _plan_only(text, fn, grad=None, prec="f32"):
    return P.Function(text, fn, grad, dot_precision=prec, flags=P.DLVM_PLAN_ONLY)


def _oracle_sig(mod, name):
    f = mod.functions[name]
    tr = lambda t: (tuple(t.shape), P.DLVM_BOOL if t.dtype == "bool" else P.DLVM_F32)
    return [tr(t) for t in f.param_types], [tr(t) for t in f.result_types]


CONFIGS = [(W.c1(), "f32"), (W.c2(64, 96), "f32"), (W.c3(64), "bf16"), (W.c4(8), "bf16"), (W.c5(32), "bf16")]


@pytest.mark.parametrize("w,prec", CONFIGS, ids=[c[0].name for c in CONFIGS])
def test_signature_and_types_match_oracle(w, prec):
    m = oracle.parse(w.text)
    f = _plan_only(w.text, w.fn, w.grad, prec)
    assert f.signature(0) == _oracle_sig(m, w.fn)
    assert f.signature(1) == _oracle_sig(m, w.grad)
    # the typed primal as printed by C++ re-verifies in the oracle: every
    # operand annotation is the C++-inferred type, checked against the oracle's
    mm = oracle.parse('module "p"\nstage raw\n' + f.print(0))
    assert [str(t) for t in mm.functions[w.fn].param_types] == [str(t) for t in m.functions[w.fn].param_types]
    for name, t in m.functions[w.fn].types.items():
        assert str(mm.functions[w.fn].types[name]) == str(t)


def _ad_cross_check(text, fn, grad, inputs, seed=None, rtol=1e-10):
    m = oracle.parse(text)
    f = _plan_only(text, fn, grad)
    gm = oracle.parse('module "g"\nstage optimizable\n' + f.print(1))
    args = list(inputs) + ([seed] if seed is not None else [])
    ours = oracle.run(gm, grad, args)       # C++-generated adjoint IR, interpreted in f64
    ref = oracle.run(m, grad, args)         # oracle reverse sweep
    assert len(ours) == len(ref)
    for a, b in zip(ours, ref):
        np.testing.assert_allclose(a, b, rtol=rtol, atol=1e-12 * (np.max(np.abs(b)) + 1e-300))
    return f


@pytest.mark.parametrize("w,prec", CONFIGS[:3], ids=[c[0].name for c in CONFIGS[:3]])
def test_cpp_adjoint_equals_oracle_vjp(w, prec):
    ins = [x.astype(np.float64) for x in w.inputs()]
    seed = None if w.seed() is None else np.asarray(w.seed(), dtype=np.float64)
    _ad_cross_check(w.text, w.fn, w.grad, ins, seed)


def test_fig3_fig4_gradients_through_cpp_ad():
    rng = np.random.default_rng(3)
    m = oracle.parse(W.FIG3)
    ins = [rng.normal(size=t.shape) for t in m.functions["foo"].param_types]
    _ad_cross_check(W.FIG3, "foo", "foo_grad", ins)
    _ad_cross_check(W.FIG3, "foo", "foo_grad_3", ins, rng.normal(size=(1, 10)))
    t4 = W.fig4_ir()
    m4 = oracle.parse(t4)
    _ad_cross_check(t4, "g", "dg", [rng.normal(size=t.shape) for t in m4.functions["g"].param_types])


def test_dce_removes_layer1_input_gradient():
    """ADCE: x is not in wrt, so the adjoint never computes
    dot(dZ1, transpose(W1)) -- four dots remain for two layers' dW/dX."""
    f = _plan_only(W.c1().text, "mlp", "mlp_grad")
    g = f.print(1)
    assert g.count(" = dot ") == 2 + 2 + 1  # fwd z1, z2; dW2, dX2(=dH1); dW1
    assert "%w1" in g


def _rand_program(rng):
    """Random straight-line programs over rank-1..3 shapes with numpy-style
    broadcasting, exercising every hot-path op."""
    base = [int(rng.integers(2, 5)) for _ in range(3)]
    rank = int(rng.integers(1, 4))
    S = base[3 - rank:]

    def sub_shape():
        s = [d if rng.random() < 0.6 else 1 for d in S]
        k = int(rng.integers(0, len(s)))
        return s[k:] if rng.random() < 0.3 else s

    ty = lambda s: "<" + " x ".join(map(str, s)) + " x f32>" if s else "f32"
    args = [("a", S), ("b", sub_shape()), ("c", sub_shape())]
    lines, cur, cur_s, n = [], "%a", S, 0
    for _ in range(int(rng.integers(3, 8))):
        n += 1
        op = ["add", "subtract", "multiply", "divide", "tanh", "exp", "negate", "sig", "relu", "shape"][rng.integers(10)]
        if op in ("add", "subtract", "multiply", "divide"):
            o = args[int(rng.integers(1, 3))]
            other = f"%{o[0]}: {ty(o[1])}"
            if op == "divide":
                lines.append(f"    %p{n} = exp %{o[0]}: {ty(o[1])}")
                other = f"%p{n}: {ty(o[1])}"
            lines.append(f"    %t{n} = {op} {cur}: {ty(cur_s)}, {other}")
        elif op == "sig":
            lines += [f"    %n{n} = negate {cur}: {ty(cur_s)}", f"    %e{n} = exp %n{n}: {ty(cur_s)}",
                      f"    %d{n} = add %e{n}: {ty(cur_s)}, 1: f32", f"    %t{n} = divide 1: f32, %d{n}: {ty(cur_s)}"]
        elif op == "relu":
            lines += [f"    %c{n} = gt {cur}: {ty(cur_s)}, 0: f32",
                      f"    %t{n} = select %c{n}: {ty(cur_s)[:-4]}bool>, {cur}: {ty(cur_s)}, 0: f32"
                      if cur_s else f"    %t{n} = select %c{n}: bool, {cur}: f32, 0: f32"]
        elif op == "shape" and len(cur_s) >= 1:
            lines.append(f"    %t{n} = transpose {cur}: {ty(cur_s)}")
            cur_s = list(reversed(cur_s))
            n += 1
            lines.append(f"    %t{n} = transpose %t{n-1}: {ty(cur_s)}")
            cur_s = list(reversed(cur_s))
        else:
            lines.append(f"    %t{n} = {op if op in ('tanh', 'exp', 'negate') else 'tanh'} {cur}: {ty(cur_s)}")
        cur = f"%t{n}"
    while cur_s:
        n += 1
        lines.append(f"    %t{n} = reduce {cur}: {ty(cur_s)} by add along {len(cur_s) - 1}")
        cur_s = cur_s[:-1]
        cur = f"%t{n}"
    lines.append(f"    return {cur}: f32")
    sig = ", ".join(ty(s) for _, s in args)
    head = ['module "r"', "stage raw", f"func @f: ({sig}) -> f32 {{",
            "'entry(" + ", ".join(f"%{a}: {ty(s)}" for a, s in args) + "):"]
    tail = ["}", "", "[gradient @f]", f"func @g: ({sig}) -> ({sig})", ""]
    return "\n".join(head + lines + tail), args


@pytest.mark.parametrize("seed", range(40))
def test_random_programs_types_and_ad(seed):
    rng = np.random.default_rng(1000 + seed)
    text, args = _rand_program(rng)
    ins = [rng.uniform(-1, 1, s) for _, s in args]
    f = _ad_cross_check(text, "f", "g", ins)
    m = oracle.parse(text)
    assert f.signature(1) == _oracle_sig(m, "g")
    assert "unsupported" not in f.print(3), f.print(3)


def _status(text, fn="f", grad=None):
    try:
        P.Function(text, fn, grad, flags=P.DLVM_PLAN_ONLY)
        return 0
    except P.DlvmError as e:
        return e.status


def test_error_classes_match_oracle():
    from test_oracle_pins import BAD_PARSE, BAD_VERIFY
    for t in BAD_PARSE:
        with pytest.raises(oracle.ParseError):
            oracle.parse(t)
        assert _status(t) == 2, t
    for t in BAD_VERIFY:
        with pytest.raises(oracle.VerifyError):
            oracle.parse(t)
        assert _status(t) == 1, t


def test_usage_errors():
    w = W.c1()
    f = _plan_only(w.text, w.fn, w.grad)
    with pytest.raises(P.DlvmError) as e:
        P.dlvm.lib().dlvm_fn_run(f._h, None, 0, None, 0, None, None) and P.dlvm._check(3)
        P.dlvm._check(P.dlvm.lib().dlvm_fn_run(f._h, None, 0, None, 0, None, None))
    assert e.value.status == 3
    with pytest.raises(P.DlvmError) as e:
        P.Function(w.text, "nope", None, flags=P.DLVM_PLAN_ONLY)
    assert e.value.status == 3
    # f64 tensors are valid IR but not executed on the GPU path
    t64 = W.FIG3.replace("f32", "f64")
    with pytest.raises(P.DlvmError) as e:
        P.Function(t64, "foo", "foo_grad")
    assert e.value.status == 6
    assert "unsupported" in P.Function(t64, "foo", "foo_grad", flags=P.DLVM_PLAN_ONLY).print(2)


def test_gradient_ready_events_cover_every_gradient():
    for w, prec in CONFIGS:
        f = _plan_only(w.text, w.fn, w.grad, prec)
        plan = f.print(3)
        n = len(f.signature(1)[1]) - 1  # kept loss output
        for k in range(n):
            assert f"event: gradient {k} ready" in plan, (w.name, k)


def test_specialisation_table_is_current():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "gen_specializations.py"), "--check"],
                       capture_output=True)
    assert r.returncode == 0, "spec_programs.inc is stale: run tools/gen_specializations.py and rebuild"


def test_plan_launch_counts_configs():
    """The fused plans stay small: c3's fwd+adjoint is 8 GEMMs (3 fwd, 3 dW,
    2 dX with fused ReLU'/bias-sum epilogues) + 5 tiny finalize/scalar kernels."""
    f = _plan_only(W.c3().text, "mlp", "mlp_grad", "bf16")
    plan = f.print(3)
    assert plan.count("gemm tcgen05") == 8
    assert f.num_launches(1) <= 14
    f2 = _plan_only(W.c2(64, 128).text, "chain", "chain_grad")
    # one fused fwd+adjoint kernel + ONE finalize for both column sums (dw, db)
    assert f2.num_launches(0) == 1 and f2.num_launches(1) == 2
    assert "finalize %" in f2.print(3) and f2.print(3).count("finalize") == 1


def test_reductions_of_one_producer_share_one_finalize():
    """Column sums (n=1000), row sums (n=3000) and a full sum (n=1) of one
    element-wise kernel are finalized by ONE launch; the c2 adjoint's dw/db
    and c3's loss/db3 likewise."""
    from merged_reductions import merged_reduction_program
    f = _plan_only(merged_reduction_program(3000, 1000), "f")
    plan = f.print(2)
    assert f.num_launches(0) == 2, plan
    assert "finalize %c, %r, %t (250 partials x 1000, 4 partials x 3000, 1000 partials x 1)" in plan, plan
    c3 = _plan_only(W.c3().text, "mlp", "mlp_grad", "bf16").print(3)
    assert "finalize %l, %d8 (" in c3, c3


def test_higher_order_cpp_ad_equals_oracle():
    """Gradient of a gradient function (Fig. 4 d2g_dw2 and an
    MLP Hessian-vector product): the C++-generated second-order IR,
    interpreted by the oracle in float64, equals the oracle's own second-order
    result (its adjoint code generation + reverse sweep)."""
    from test_oracle_higher_order import _mlp2, _scalar_sum_pow, fig4_second_order
    rng = np.random.default_rng(17)
    t = fig4_second_order(8, 12, 6)
    m = oracle.parse(t)
    ins = [rng.normal(size=p.shape) * 0.5 for p in m.functions["g"].param_types]
    f = _plan_only(t, "dg", "d2g_dw2")
    assert f.signature(1) == _oracle_sig(m, "d2g_dw2")
    _ad_cross_check(t, "dg", "d2g_dw2", ins, rtol=1e-10)
    text, P_ = _mlp2(5, 4, 6, 3, "sigmoid")
    ins = [rng.normal(size=s) * 0.5 for _, s in P_]
    _ad_cross_check(text, "df", "hvp", ins, rng.normal(size=(4, 6)), rtol=1e-10)
    t3 = _scalar_sum_pow(3, 4, 3)
    _ad_cross_check(t3, "d2", "d3", [np.array([0.5, -1.5, 2.0])], rtol=1e-12)
    f3 = _plan_only(t3, "d2", "d3")
    assert "unsupported" not in f3.print(3)


def test_cyclic_gradient_declarations_error_class():
    t = "<2 x f32>"
    text = (f'module "c"\nstage raw\n[gradient @b]\nfunc @a: ({t}) -> {t}\n'
            f"[gradient @a]\nfunc @b: ({t}) -> {t}\n")
    with pytest.raises(oracle.VerifyError):
        oracle.parse(text)
    assert _status(text, "a") == 1


def test_linear_algebra_fusion_rnn_plan():
    """W x + U h + b is one matrix multiplication.  The
    RNN's forward cells are single GEMMs with two K segments (bias and tanh
    in the epilogue), and the weight gradients dW = sum_t x_t^T dZ_t,
    dU = sum_t h_{t-1}^T dZ_t are single GEMMs with T K segments."""
    T = 4
    w = W.rnn(T, 256, 128, 192)
    f = _plan_only(w.text, w.fn, w.grad, "bf16")
    fwd, bwd = f.print(2), f.print(3)
    assert fwd.count("gemm tcgen05") == T and fwd.count("(2 K segments: 128 192)") == T
    assert bwd.count(f"({T} K segments: 256 256 256 256)") == 2
    assert bwd.count("gemm tcgen05") == T + (T - 1) + 2
    # the generated adjoint (C++ AD) is still the oracle's VJP
    ws = W.rnn(3, 6, 4, 5, "f32")
    ins = [x.astype(np.float64) for x in ws.inputs()]
    _ad_cross_check(ws.text, ws.fn, ws.grad, ins, np.float64(ws.seed()))


def _opt_equiv(text, fn, grad, ins, seed=None, rtol=1e-11):
    """The optimised IR the plans execute (print modes 6/7), interpreted by
    the oracle in float64, computes what the written program computes."""
    m = oracle.parse(text)
    f = _plan_only(text, fn, grad)
    om = oracle.parse('module "o"\nstage optimizable\n' + f.print(6) + ("\n" + f.print(7) if grad else ""))
    for name, args in [(fn, list(ins))] + ([(grad, list(ins) + ([seed] if seed is not None else []))] if grad else []):
        for a, b in zip(oracle.run(om, name, args), oracle.run(m, name, args)):
            np.testing.assert_allclose(a, b, rtol=rtol, atol=rtol * (np.max(np.abs(b)) + 1e-300))
    return f


OPT_PROGRAM = """module "o"
stage raw
func @f: (<16 x 4 x f32>, <4 x 512 x f32>, <512 x 8 x f32>, <16 x 8 x f32>) -> f32 {
'entry(%x: <16 x 4 x f32>, %w1: <4 x 512 x f32>, %w2: <512 x 8 x f32>, %t: <16 x 8 x f32>):
    %u = dot %x: <16 x 4 x f32>, %w1: <4 x 512 x f32>
    %v = dot %u: <16 x 512 x f32>, %w2: <512 x 8 x f32>
    %p = power %v: <16 x 8 x f32>, 2: f32
    %q = power %t: <16 x 8 x f32>, 1: f32
    %o = power %v: <16 x 8 x f32>, 0: f32
    %a = multiply %p: <16 x 8 x f32>, 1: f32
    %b = add %a: <16 x 8 x f32>, 0: f32
    %c = subtract %b: <16 x 8 x f32>, %q: <16 x 8 x f32>
    %d = multiply %c: <16 x 8 x f32>, %o: <16 x 8 x f32>
    %e = negate %d: <16 x 8 x f32>
    %g = negate %e: <16 x 8 x f32>
    %h = transpose %g: <16 x 8 x f32>
    %k = transpose %h: <8 x 16 x f32>
    %r0 = reduce %k: <16 x 8 x f32> by add along 1
    %r1 = reduce %r0: <16 x f32> by add along 0
    return %r1: f32
}
[gradient @f wrt 1, 2]
func @df: (<16 x 4 x f32>, <4 x 512 x f32>, <512 x 8 x f32>, <16 x 8 x f32>) -> (<4 x 512 x f32>, <512 x 8 x f32>)
"""


def test_optimiser_algebra_cse_and_matrix_chain():
    """Create-time optimiser: x^2 -> x*x, x^1 -> x, x^0 -> 1,
    x*1, x+0, -(-x), transpose(transpose x) removed; (x.W1).W2 with a
    512-wide middle is reassociated to x.(W1.W2) (16*4*8 + 4*512*8
    multiply-adds instead of 16*4*512 + 16*512*8); values unchanged (f64)."""
    rng = np.random.default_rng(5)
    ins = [rng.normal(size=s) for s in [(16, 4), (4, 512), (512, 8), (16, 8)]]
    f = _opt_equiv(OPT_PROGRAM, "f", "df", ins)
    o = f.print(6)
    assert " power " not in o and " negate " not in o and " transpose " not in o, o
    assert "dot %w1: <4 x 512 x f32>, %w2: <512 x 8 x f32>" in o, o
    assert o.count(" = dot ") == 2
    assert "unsupported" not in f.print(3)
    # the written program is planned unchanged with DLVM_NO_OPT
    g = P.Function(OPT_PROGRAM, "f", "df", flags=P.DLVM_PLAN_ONLY | P.DLVM_NO_OPT)
    assert " power " in g.print(6) and g.print(6) == g.print(0)


@pytest.mark.parametrize("seed", range(40))
def test_optimiser_preserves_random_programs(seed):
    rng = np.random.default_rng(1000 + seed)
    text, args = _rand_program(rng)
    ins = [rng.uniform(-1, 1, s) for _, s in args]
    _opt_equiv(text, "f", "g", ins)


def test_optimiser_configs_and_higher_order():
    for w, prec in CONFIGS[:3]:
        ins = [x.astype(np.float64) for x in w.inputs()]
        seed = None if w.seed() is None else np.asarray(w.seed(), dtype=np.float64)
        _opt_equiv(w.text, w.fn, w.grad, ins, seed)
    hv = W.mlp_hvp(8, 4, 6, 3)
    ins = [x.astype(np.float64) for x in hv.inputs()]
    _opt_equiv(hv.text, hv.fn, hv.grad, ins, hv.seed().astype(np.float64))


def test_adjoint_ir_structure_filecheck():
    """FileCheck-style checks (SURVEY §4 T6, P:L92/L340 lit+FileCheck) of the
    generated adjoint IR, written from the adjoint rules: Fig. 4's dg uses
    dot(transpose(x), dZ) for dW, a column reduce for db, the tanh adjoint
    1 - y*y, keeps g's result last; DCE removed the unused dX."""
    f = _plan_only(W.fig4_ir(), "g", "dg")
    g = f.print(1)
    lines = [l.strip() for l in g.splitlines()]
    order = ["= tanh %1", "multiply %2: <4 x 5 x f32>, %2", "subtract 1: f32", "reduce", "by add along 0",
             "shapeCast", "to 1 x 5", "transpose %x", "dot %d", "return (%d"]
    pos = 0
    for pat in order:  # CHECK: in order
        while pos < len(lines) and pat not in lines[pos]:
            pos += 1
        assert pos < len(lines), f"CHECK not found in order: {pat}\n{g}"
    assert "transpose %w" not in g  # CHECK-NOT: dX (x is not in wrt)
    assert lines[-2].endswith("%2: <4 x 5 x f32>)")  # kept g result last (A7)


def test_kernel_templates_compile_under_nvrtc():
    """The create-time JIT (csrc/jit.cpp) compiles the kernel templates with
    NVRTC; a header change that breaks runtime compilation must fail here, on
    the CPU (NVRTC needs no GPU).  One EW, one tcgen05 (CTA pair) and one SIMT
    instantiation with registry programs."""
    nvrtc = pytest.importorskip("cuda.bindings.nvrtc")
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from gen_specializations import prog_type
    kdir = os.path.join(ROOT, "paper_1711_03016_b200", "csrc", "kernels")
    prog = lambda sig: prog_type(sig).replace("spec::", "dlvm::spec::")
    exprs = [f"&dlvm::kern::ew2d_kernel<4, {prog('i4l0|22,0,1,2;1,4,0,0;9,5,3,0|s6|r')}>",
             f"&dlvm::kern::gemm_tc_kernel<256, {prog('i2l0|21,1,0,0;9,0,2,0|s3|r3:0')}, 2>",
             f"&dlvm::kern::simt::gemm_simt_kernel<false, 32, {prog('i2l1|7,0,1,0|s3|r')}>"]
    opts = [b"--gpu-architecture=sm_100a", b"-std=c++17", b"-default-device", ("-I" + kdir).encode(),
            b"-I/usr/local/cuda/include"]
    src = b'#include "gemm_tc_kernel.cuh"\n#include "gemm_simt_kernel.cuh"\n'
    err, p = nvrtc.nvrtcCreateProgram(src, b"t.cu", 0, [], [])
    for e in exprs:
        nvrtc.nvrtcAddNameExpression(p, e.encode())
    (r,) = nvrtc.nvrtcCompileProgram(p, len(opts), opts)
    _, n = nvrtc.nvrtcGetProgramLogSize(p)
    # NVRTC writes into this buffer: it must be a fresh object.  `b" " * n`
    # with n == 1 (an empty log) is CPython's shared one-byte b" ", and
    # overwriting it corrupts every later " " in the process
    log = bytes(n + 8)
    nvrtc.nvrtcGetProgramLog(p, log)
    assert r == nvrtc.nvrtcResult.NVRTC_SUCCESS, log.decode()[:3000]
    for e in exprs:
        _, low = nvrtc.nvrtcGetLoweredName(p, e.encode())
        assert low and low.startswith(b"_ZN4dlvm4kern")


def test_tall_thin_launch_grids_stay_legal():
    """Element-wise groups over very tall, thin spaces ([2^28, 1]) raise rows
    per thread so the grid's y extent stays <= 65535 (CUDA limit)."""
    import re as _re
    for R in (1 << 22, 1 << 26, 1 << 28):
        w = W.c2(R, 1)
        f = _plan_only(w.text, w.fn, w.grad)
        assert "unsupported" not in f.print(3)
    w = W.c2(1 << 28, 1)
    f = _plan_only(w.text, w.fn, w.grad)
    counts = [int(x) for x in _re.findall(r"\((\d+) partials", f.print(3))]
    assert counts and max(counts) <= 65535, counts  # one partial per grid row block


def test_reduce_multiply_plans_one_product_step():
    """`reduce ... by multiply` (Table 1, forward only): its operand is
    materialised and the product is one element-wise step whose input walks
    the reduced axis (chunked load, multiplied in order); the sum over a
    product and later element-wise consumers plan as usual."""
    import prod_programs as PP
    f = _plan_only(PP.prod_chain(40, 24), "f")
    plan = f.print(2)
    assert "unsupported" not in plan, plan
    assert plan.count("product of") == 3, plan
    assert "(40 factors)" in plan and "(24 factors)" in plan and "(3 factors)" in plan, plan
    g = _plan_only(PP.prod_grad(16, 8), "f", "g")
    assert g.print(3).count("product of") == 1, g.print(3)
    # a product of a splat literal folds at create time
    t = ('module "m"\nstage raw\nfunc @f: (<4 x f32>) -> <4 x f32> {\n\'entry(%a: <4 x f32>):\n'
         '    %r = reduce 2: <3 x 4 x f32> by multiply along 0\n    %s = multiply %a: <4 x f32>, %r: <4 x f32>\n'
         '    return %s: <4 x f32>\n}\n')
    assert "product of" not in _plan_only(t, "f").print(2)


@pytest.mark.parametrize("seed", range(60))
def test_random_nd_programs_types_ad_and_plan(seed):
    """Rank-1..5 programs with NumPy broadcasting across ranks, rank>2
    transposes and reductions along random axes: the C++ types match the
    oracle's, the C++ adjoint IR (interpreted in f64) equals the oracle's
    reverse sweep, and both plans (primal, gradient) are supported."""
    import nd_programs as ND
    rng = np.random.default_rng(5000 + seed)
    text, args = ND.nd_program(rng)
    m = oracle.parse(text)
    f = _ad_cross_check(text, "f", "g", [x.astype(np.float64) for x in ND.nd_inputs(rng, args)])
    assert f.signature(0) == _oracle_sig(m, "f")
    assert f.signature(1) == _oracle_sig(m, "g")
    for mode in (2, 3):
        assert "unsupported" not in f.print(mode), text + f.print(mode)
    body, _ = ND.nd_program(np.random.default_rng(5000 + seed), all_values=True)
    fb = _plan_only(body, "f")
    assert fb.signature(0) == _oracle_sig(oracle.parse(body), "f")
    assert "unsupported" not in fb.print(2), body + fb.print(2)


@pytest.mark.parametrize("seed", range(30))
def test_random_gradient_configurations(seed):
    """Random `[gradient @f from F wrt W keeping K seedable]` declarations on
    N-d programs returning (loss, tensor) (Fig. 3, Fig. 4
    P:L358-365): C++ signature and adjoint IR (in f64) equal the oracle's,
    both plans supported."""
    import nd_programs as ND
    rng = np.random.default_rng(300 + seed)
    text, args, cfg = ND.nd_grad_config(rng)
    m = oracle.parse(text)
    ins = [x.astype(np.float64) for x in ND.nd_inputs(rng, args)]
    s = rng.uniform(-1, 1, cfg["seed_shape"]) if cfg["seedable"] else None
    f = _ad_cross_check(text, "f", "g", ins, s)
    assert f.signature(0) == _oracle_sig(m, "f")
    assert f.signature(1) == _oracle_sig(m, "g")
    for mode in (2, 3):
        assert "unsupported" not in f.print(mode), text + f.print(mode)


def test_zero_size_dimensions_are_parse_errors():
    """Reading A25: tensor dimensions are >= 1 (an empty tensor is not an IR
    value); both front ends reject `<0 x 5 x f32>` as a parse error (class 2)."""
    t = ('module "m"\nstage raw\nfunc @f: (<0 x 5 x f32>) -> <0 x 5 x f32> {\n'
         "'entry(%x: <0 x 5 x f32>):\n    %y = tanh %x: <0 x 5 x f32>\n    return %y: <0 x 5 x f32>\n}\n")
    with pytest.raises(oracle.ParseError):
        oracle.parse(t)
    with pytest.raises(P.DlvmError) as e:
        P.Function(t, "f", None, flags=P.DLVM_PLAN_ONLY)
    assert e.value.status == 2


def test_planner_layout_heuristics():
    """Regression guards for plan-time layout choices:
    few-tile GEMMs use 128-wide tiles; weights get row-padded bf16 copies
    only for large-batch dots; reduction results get unpadded homes; row
    splits of a row-padded dot result stay views (no copy launch)."""
    c3 = _plan_only(W.c3().text, W.c3().fn, W.c3().grad, "bf16")
    assert any(l.startswith("GEMM 128") for l in c3.print(4).splitlines())   # %z3: 16 pair tiles -> 128 x 128
    assert "pack %" not in c3.print(3)                                         # batch 1024: no padded weight copy
    c4 = _plan_only(W.c4().text, W.c4().fn, W.c4().grad, "bf16")
    assert "pack %w3 to bf16 rows of 1024" in c4.print(3)                      # batch 65536: padded copy
    # dW GEMMs with K = 65536 split in two: the sum steps are optional (the
    # GEMM adds both splits into an f32-bound home)
    sums = [l for l in c4.print(3).splitlines() if "sum of 2 K-split partials" in l]
    assert len(sums) == 2 and all("skipped when the home is bound as f32" in l for l in sums), sums
    # a [2, 96] reduction result (rank 2, last dim 96 -> would pad to 128): unpadded, 768 bytes
    t = ('module "m"\nstage raw\nfunc @f: (<2 x 50 x 96 x f32>) -> <2 x 96 x f32> {\n'
         "'entry(%x: <2 x 50 x 96 x f32>):\n    %t = tanh %x: <2 x 50 x 96 x f32>\n"
         "    %r = reduce %t: <2 x 50 x 96 x f32> by add along 1\n    %s = multiply %r: <2 x 96 x f32>, %r: <2 x 96 x f32>\n"
         "    return %s: <2 x 96 x f32>\n}\n")
    det = _plan_only(t, "f").print(9)
    assert "work -1 bytes 768 " in det, det
    # dot result [512, 200] (row-padded home, ld 256) split into [4, 128, 200]: a strided view
    t2 = ('module "m"\nstage raw\nfunc @f: (<512 x 64 x f32>, <64 x 200 x f32>) -> <4 x 128 x 200 x f32> {\n'
          "'entry(%a: <512 x 64 x f32>, %b: <64 x 200 x f32>):\n    %d = dot %a: <512 x 64 x f32>, %b: <64 x 200 x f32>\n"
          "    %v = shapeCast %d: <512 x 200 x f32> to 4 x 128 x 200\n    %y = tanh %v: <4 x 128 x 200 x f32>\n"
          "    return %y: <4 x 128 x 200 x f32>\n}\n")
    p2 = _plan_only(t2, "f", None, "bf16")
    assert p2.print(2).count("ew [") == 1, p2.print(2)   # one element-wise launch reads the padded home directly


def test_binding_refuses_host_tensors():
    """The C ABI takes device pointers: the binding refuses CPU tensors (a
    host pointer would fault in the kernels) before anything is launched."""
    import torch
    w = W.c2(8, 16)
    f = _plan_only(w.text, w.fn, w.grad)
    with pytest.raises(ValueError, match="CUDA tensors"):
        f.run([torch.from_numpy(x) for x in w.inputs()])


def test_launch_info_bytes_of_merged_finalize():
    """dlvm_fn_launch_info's minimum bytes for a merged finalize count each
    reduction's partials at its own length: 250x1000 + 4x3000 + 1000x1 f32
    partials read, 1000 + 3000 + 1 f32 results written."""
    from merged_reductions import merged_reduction_program
    f = _plan_only(merged_reduction_program(3000, 1000), "f")
    desc, flops, nbytes = f.launch_info(0, 1)
    assert desc.startswith("finalize"), desc
    assert flops == 0
    assert nbytes == 4 * (250 * 1000 + 4 * 3000 + 1000 * 1) + 4 * (1000 + 3000 + 1)


def test_overflowing_dimensions_are_parse_errors():
    """Shapes whose element count overflows int64 (or exceeds 2^59, so byte
    sizes stay representable) and out-of-range integers are rejected at parse
    time (class 2) instead of wrapping numel / workspace sizes."""
    big = 1 << 31
    for dims in (f"{big} x {big} x {big}", "99999999999999999999999", f"{1 << 30} x {1 << 30}"):
        t = (f'module "m"\nstage raw\nfunc @f: (<{dims} x f32>) -> <{dims} x f32> {{\n'
             f"'entry(%x: <{dims} x f32>):\n    %y = tanh %x: <{dims} x f32>\n    return %y: <{dims} x f32>\n}}\n")
        with pytest.raises(P.DlvmError) as e:
            P.Function(t, "f", None, flags=P.DLVM_PLAN_ONLY)
        assert e.value.status == 2, (dims, e.value)
    X = "<4 x 4 x f32>"
    t = (f'module "m"\nstage raw\nfunc @f: ({X}) -> <{1 << 31} x {1 << 31} x f32> {{\n'
         f"'entry(%x: {X}):\n    %y = shapeCast %x: {X} to {1 << 31} x {1 << 31} x {1 << 31}\n"
         f"    return %y: {X}\n}}\n")
    with pytest.raises(P.DlvmError) as e:
        P.Function(t, "f", None, flags=P.DLVM_PLAN_ONLY)
    assert e.value.status == 2


def test_which_is_range_checked_in_every_entry_point():
    w = W.c1()
    f = _plan_only(w.text, w.fn, w.grad)
    L = P.dlvm.lib()
    n = ctypes.c_size_t(0)
    k = ctypes.c_int(0)
    for which in (-1, 2, 7):
        assert L.dlvm_fn_workspace_bytes(f._h, which, ctypes.byref(n)) == 3
        assert L.dlvm_fn_num_launches(f._h, which, ctypes.byref(k)) == 3
        assert L.dlvm_fn_launch_events(f._h, which, None, 0) == 3
    g = _plan_only(W.FIG3, "foo", None)  # no gradient: which=1 is a usage error
    assert L.dlvm_fn_workspace_bytes(g._h, 1, ctypes.byref(n)) == 3
    assert L.dlvm_fn_num_launches(g._h, 1, ctypes.byref(k)) == 3


def test_device_option_validated():
    o = P.dlvm.dlvm_options(P.dlvm.DLVM_DOT_F32, -2, P.DLVM_PLAN_ONLY)
    h = ctypes.c_void_p()
    b = W.FIG3.encode()
    assert P.dlvm.lib().dlvm_fn_create(b, len(b), b"foo", None, ctypes.byref(o), ctypes.byref(h)) == 3


def test_reduce_max_and_softmax_ce_through_cpp_ad():
    """`reduce ... by max` (reading A26) through the C++ front end: types,
    the generated adjoint (ties split equally) interpreted by the oracle in
    f64 == the oracle's reverse sweep, on a softmax-CE MLP and on a program
    with exact ties; the planner gives each max its own element-wise step."""
    w = W.ce_mlp(6, layers=[(7, 5, "relu"), (5, 4, None)], dot_precision="f32")
    ins = [x.astype(np.float64) for x in w.inputs()]
    f = _ad_cross_check(w.text, w.fn, w.grad, ins, np.float64(w.seed()))
    assert " by max along 1" in f.print(0)
    assert "max of %" in f.print(3), f.print(3)
    T = "<3 x 4 x f32>"
    t = (f'module "m"\nstage raw\nfunc @f: ({T}) -> <3 x f32> {{\n\'entry(%a: {T}):\n'
         f"    %s = multiply %a: {T}, %a: {T}\n    %r = reduce %s: {T} by max along 1\n"
         f"    return %r: <3 x f32>\n}}\n\n[gradient @f wrt 0 seedable]\nfunc @g: ({T}, <3 x f32>) -> {T}\n")
    a = np.array([[1.0, -1.0, 0.5, 0.0], [2.0, 2.0, -2.0, 1.0], [0.0, 0.0, 0.0, 0.0]])
    _ad_cross_check(t, "f", "g", [a], np.array([1.0, 3.0, 4.0]))
    with pytest.raises(P.DlvmError) as e:
        P.Function(t.replace("by max", "by min"), "f", "g", flags=P.DLVM_PLAN_ONLY)
    assert e.value.status == 2


def test_two_stream_schedule_of_c3_gradient():
    """plan_streams (print mode 12): the activation-gradient GEMMs d11 / d18
    run on the auxiliary stream beside the weight-gradient GEMMs they do not
    depend on (d13 / d20), with an event wait for their producers; the next
    weight gradient waits for them; primal plans (a dependent chain) stay on
    one stream."""
    w = W.c3()
    f = _plan_only(w.text, w.fn, w.grad, "bf16")
    s = f.print(12)
    lines = s.splitlines()
    assert lines[0] == "streams: two"
    aux = [l for l in lines if " aux " in l]
    assert any("%d11" in l and "wait[" in l for l in aux), s
    assert any("%d18" in l and "wait[" in l for l in aux), s
    assert any("main" in l and "%d20" in l and "wait[" in l for l in lines), s
    assert f.print(11).startswith("streams: one")


def test_deferred_epilogues_and_split_reduce_add_plans():
    """Plan-time choices of round 2, pinned per benchmarked config: only
    mlp_hvp defers GEMM epilogues (%z: 24 KB of store staging per warp; %o,
    %d9: two and four f32 [M,N] operands; none has reductions), and only the
    K-split-in-two dW GEMMs with store-only epilogues (c4's %d20 / %d25,
    mlp_hvp's %d45) may add into an f32 home instead of running their sum
    step."""
    import re
    expect = {"mlp_hvp": (["%z", "%o", "%d9"], 1), "c4_mlp": ([], 2), "c3_mlp": ([], 0), "c5_mlp": ([], 0),
              "rnn": ([], 0)}
    for w in (W.mlp_hvp(), W.c4(), W.c3(), W.c5(), W.rnn()):
        t = _plan_only(w.text, w.fn, w.grad, "bf16").print(3)
        deferred = [re.search(r"%\w+", l).group(0) for l in t.splitlines() if "raw accumulator" in l]
        assert (deferred, t.count("skipped when the home is bound as f32")) == expect[w.name], (w.name, deferred)
        # every deferred GEMM is followed by its epilogue step, and that step has no reductions
        lines = t.splitlines()
        for i, l in enumerate(lines):
            if "raw accumulator" in l:
                assert "deferred epilogue" in lines[i + 1] and "reductions=0" in lines[i + 1], lines[i + 1]
