"""GPU parity: the C-ABI path (libdlvm.so kernels on cuda:0) against the CPU
float64 oracle, element by element, on seeded inputs."""

import numpy as np
import pytest

import oracle
import workloads as W
from helpers import oracle_grad_module, assert_f32_parity, assert_normwise, bf16_round, f32_emulation, gpu_run, term_bound

pytestmark = pytest.mark.gpu


def _grad_module(m, name):
    """The gradient declaration `name` of the oracle-parsed module `m`,
    canonicalised to IR by the ORACLE's own adjoint code generation
    (oracle.canonical).  Tolerance bounds (sum|terms| of each
    output's last accumulation, the fp32-emulation allowance) are derived
    from it, never from the library's printed adjoint, so a numerically worse
    adjoint from the C++ AD cannot widen its own tolerance."""
    return oracle_grad_module(m, name)


def _check_f32(w, inputs, seed, primal_only=False):
    m = oracle.parse(w.text)
    res = gpu_run(w.text, w.fn, None if primal_only else w.grad, inputs, seed=seed,
                  which="primal" if primal_only else "both")
    ins64 = [x.astype(np.float64) for x in inputs]
    ref_p = oracle.run(m, w.fn, ins64)
    bp = term_bound(m, w.fn, ins64)
    for k, (g, r, b) in enumerate(zip(res["primal"], ref_p, bp)):
        assert_f32_parity(g, r, b, what=f"{w.name} primal out{k}")
    if primal_only:
        return res
    gargs = ins64 + ([np.asarray(seed, dtype=np.float64)] if seed is not None else [])
    ref_g = oracle.run(m, w.grad, gargs)
    gm = _grad_module(m, w.grad)
    bg = term_bound(gm, w.grad, gargs)
    for k, (g, r, b) in enumerate(zip(res["grad"], ref_g, bg)):
        assert_f32_parity(g, r, b, what=f"{w.name} grad out{k}")
    return res


def test_c1_full_parity():
    w = W.c1()
    _check_f32(w, w.inputs(), w.seed())


@pytest.mark.parametrize("R,C", [(64, 128), (37, 1003), (1, 5), (300, 4096)])
def test_c2_chain_parity(R, C):
    w = W.c2(R, C)
    _check_f32(w, w.inputs(), w.seed())


def test_c2_full_size_sampled():
    """c2 at BASELINE size [16384, 16384], the launch configuration bench.py
    times; every element of y, dx, dw and db checked against the oracle."""
    import torch
    import paper_1711_03016_b200 as P
    w = W.c2()
    m = oracle.parse(w.text)
    f = P.Function(w.text, w.fn, w.grad)
    dev = torch.device("cuda:0")
    ins = [torch.from_numpy(x).to(dev) for x in w.inputs()]
    seed = torch.from_numpy(w.seed()).to(dev)
    (y,) = f.run(ins)
    dx, dw, db = f.grad_run(ins, seed=seed)
    torch.cuda.synchronize()
    xs = [a.cpu().numpy() for a in ins]
    g = seed.cpu().numpy()
    yg, dxg, dwg, dbg = y.cpu().numpy(), dx.cpu().numpy(), dw.cpu().numpy(), db.cpu().numpy()
    # every output element: the chain is row-local and column-local, so the
    # oracle runs the same program on [16384, 1024] column blocks (all rows)
    # and compares y and dx element by element (A16) and dw, db (A17)
    B = 1024
    mb = oracle.parse(W.chain_ir(16384, B))
    gb = _grad_module(mb, "chain_grad")
    h = lambda a: np.ascontiguousarray(a, dtype=np.float64)
    for c0 in range(0, 16384, B):
        cs = slice(c0, c0 + B)
        blk = [h(xs[0][:, cs]), h(xs[1][:, cs]), h(xs[2][:, cs]), h(xs[3][:, cs])]
        (ry,) = oracle.run(mb, "chain", blk)
        assert_f32_parity(yg[:, cs], ry, what=f"c2 y cols {c0}+")
        del ry
        blk.append(h(g[:, cs]))
        rdx, rdw, rdb = oracle.run(mb, "chain_grad", blk)
        assert_f32_parity(dxg[:, cs], rdx, what=f"c2 dx cols {c0}+")
        del rdx
        _, bdw, bdb = term_bound(gb, "chain_grad", blk)
        assert_f32_parity(dwg[:, cs], rdw, bdw, what=f"c2 dw cols {c0}+")
        assert_f32_parity(dbg[:, cs], rdb, bdb, what=f"c2 db cols {c0}+")


def test_fig3_fig4_programs():
    m = oracle.parse(W.FIG3)
    rng = np.random.default_rng(11)
    ins = [rng.uniform(-1, 1, t.shape).astype(np.float32) for t in m.functions["foo"].param_types]
    res = gpu_run(W.FIG3, "foo", "foo_grad_3", ins, seed=np.float32(1) * np.ones((1, 10), np.float32))
    ref = oracle.run(m, "foo_grad_3", [x.astype(np.float64) for x in ins] + [np.ones((1, 10))])
    for g, r in zip(res["grad"], ref):
        assert_f32_parity(g, r, np.abs(r) + 1e-3, what="fig3 grad_3")
    text = W.fig4_ir(8, 12, 6)
    m4 = oracle.parse(text)
    ins = [rng.uniform(-1, 1, t.shape).astype(np.float32) for t in m4.functions["g"].param_types]
    res = gpu_run(text, "g", "dg", ins)
    ref = oracle.run(m4, "dg", [x.astype(np.float64) for x in ins])
    bg = term_bound(_grad_module(m4, "dg"), "dg", [x.astype(np.float64) for x in ins])
    for k, (g, r, b) in enumerate(zip(res["grad"], ref, bg)):
        assert_f32_parity(g, r, b, what=f"fig4 out{k}")


@pytest.mark.parametrize("prec", ["f32", "bf16"])
def test_F8_dyadic_bit_exact(prec):
    """F8: every value is dyadic, so f32 and bf16 paths are bit-exact."""
    import json, os
    P = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand_pins.json")))["F8_221_sigmoid_mlp"]
    text = W.mlp_ir(1, [(2, 2, "sigmoid"), (2, 1, "sigmoid")])
    ins = [np.array(P[k], dtype=np.float32) for k in ("x", "w1", "b1", "w2", "b2", "t")]
    res = gpu_run(text, "mlp", "mlp_grad", ins, seed=np.float32(1.0), dot_precision=prec)
    assert res["primal"][0] == P["L"]
    dw1, db1, dw2, db2, L = res["grad"]
    np.testing.assert_array_equal(dw1, P["dw1"])
    np.testing.assert_array_equal(db1, P["db1"])
    np.testing.assert_array_equal(dw2, P["dw2"])
    np.testing.assert_array_equal(db2, P["db2"])
    assert L == P["L"]


def test_F12_seed_scaling_and_determinism():
    w = W.c1()
    ins = w.inputs()
    g1 = gpu_run(w.text, w.fn, w.grad, ins, seed=np.float32(1 / 32), which="grad")["grad"]
    g1b = gpu_run(w.text, w.fn, w.grad, ins, seed=np.float32(1 / 32), which="grad")["grad"]
    g8 = gpu_run(w.text, w.fn, w.grad, ins, seed=np.float32(8 / 32), which="grad")["grad"]
    for a, b, c in zip(g1[:-1], g1b[:-1], g8[:-1]):
        np.testing.assert_array_equal(a, b)          # rerun bit-identical (A14)
        np.testing.assert_array_equal(a * 8.0, c)    # F12
    res = gpu_run(w.text, w.fn, w.grad, ins, seed=np.float32(1 / 32))
    assert res["grad"][-1] == res["primal"][0]       # kept output bit-equal to fn_run (A20)


# --- tcgen05 GEMM: every operand major-ness, ragged tiles ---------------------

def _dot_ir(M, K, N, ta, tb):
    A = f"<{K} x {M} x f32>" if ta else f"<{M} x {K} x f32>"
    B = f"<{N} x {K} x f32>" if tb else f"<{K} x {N} x f32>"
    lines = ['module "d"', "stage raw", f"func @f: ({A}, {B}) -> <{M} x {N} x f32> {{",
             f"'entry(%a: {A}, %b: {B}):"]
    a, b = "%a", "%b"
    if ta:
        lines.append(f"    %at = transpose %a: {A}")
        a = "%at"
    if tb:
        lines.append(f"    %bt = transpose %b: {B}")
        b = "%bt"
    lines += [f"    %r = dot {a}: <{M} x {K} x f32>, {b}: <{K} x {N} x f32>",
              f"    return %r: <{M} x {N} x f32>", "}"]
    return "\n".join(lines) + "\n"


@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False), (True, True)])
@pytest.mark.parametrize("M,K,N", [(256, 128, 256), (200, 72, 136), (384, 1000, 1000), (128, 64, 64)])
def test_tcgen05_dot_majors(M, K, N, ta, tb):
    """bf16-representable inputs: the product is exact in fp32 accumulation up
    to summation error, so compare with the f64 oracle at 1e-5 * sum|terms|."""
    rng = np.random.default_rng(M + K + N)
    a = bf16_round(rng.standard_normal((K, M) if ta else (M, K)))
    b = bf16_round(rng.standard_normal((N, K) if tb else (K, N)))
    text = _dot_ir(M, K, N, ta, tb)
    res = gpu_run(text, "f", None, [a, b], dot_precision="bf16", which="primal")
    assert "tcgen05" in res["fn"].print(2), res["fn"].print(2)
    A = a.astype(np.float64).T if ta else a.astype(np.float64)
    B = b.astype(np.float64).T if tb else b.astype(np.float64)
    ref = A @ B
    assert_f32_parity(res["primal"][0], ref, np.abs(A) @ np.abs(B), what=f"dot {M}x{K}x{N} ta={ta} tb={tb}")


def _check_c3(w, policy_tol=2e-2):
    """bf16 policy (reading A15).  Network-level parity is checked against the
    oracle under the same policy (every dot operand rounded to bf16, float64
    arithmetic): the unrounded comparison is ill-conditioned for gradients
    behind a ReLU, whose derivative jumps at 0 -- bf16 rounding of the forward
    pass moves ~0.2% of pre-activations across 0 (reading A18').
    The outputs whose adjoint crosses no ReLU (last layer dW, db; the loss)
    are also held to A18 (2e-2 normwise) against the unrounded oracle."""
    ins = w.inputs()
    res = gpu_run(w.text, w.fn, w.grad, ins, seed=w.seed(), dot_precision="bf16")
    m = oracle.parse(w.text)
    args = [x.astype(np.float64) for x in ins] + [np.float64(w.seed())]
    ref_pol = oracle.run(m, w.grad, args, dot_policy="bf16")
    ref_raw = oracle.run(m, w.grad, args)
    n = len(w.layers)
    kinked = any(act == "relu" for _, _, act in w.layers)
    rels = []
    for k, (g, rp, rr) in enumerate(zip(res["grad"], ref_pol, ref_raw)):
        rels.append(assert_normwise(g, rp, policy_tol, what=f"{w.name} grad out{k} vs bf16-policy oracle"))
        # A18 against the unrounded oracle: every output of a kink-free
        # (tanh) network; behind a ReLU only the outputs whose adjoint
        # crosses no kink (last layer dW, db and the kept loss)
        if not kinked or k >= 2 * (n - 1):
            assert_normwise(g, rr, 2e-2, what=f"{w.name} grad out{k} vs unrounded oracle")
    assert_normwise(res["primal"][0], oracle.run(m, w.fn, args[:-1], dot_policy="bf16")[0], policy_tol)
    assert_normwise(res["primal"][0], oracle.run(m, w.fn, args[:-1])[0], 2e-2, what=f"{w.name} loss vs unrounded")
    return rels


def test_c3_small_bf16():
    _check_c3(W.c3(128, layers=[(256, 256, "relu"), (256, 256, "relu"), (256, 100, None)]))


def test_c3_full_bf16():
    _check_c3(W.c3())


def test_c5_small_tanh_bf16():
    """c5's program (tanh layers, MSE on a dense target) at reduced width."""
    w = W._mlp_workload(5, "c5_small", 256, [(512, 512, "tanh")] * 4, ("normal",), ("uniform", -0.5, 0.5),
                        1.0 / 256, "bf16", 256)
    _check_c3(w)


@pytest.mark.parametrize("n_ranks", [8, 4])
def test_c4_per_rank_shard_plans(n_ranks):
    """The per-rank program c4 runs at N = 4 and 8 GPUs (global batch 65536
    split in 16384 / 8192 rows, seed 1/65536): other split-K decisions and
    tile counts than N = 1.  One rank's shard gradients against the float64
    oracle on the same rows (A18' vs the bf16-policy oracle; the last layer's
    dW, db and the loss also A18 vs the unrounded one); summing the shards
    over ranks is the linearity F15 pinned on CPU."""
    _check_c3(W.c4(n_ranks))


def test_c5_full_width_reduced_batch():
    """c5 with its full weights (8 tanh layers of 8192 x 8192, SURVEY 8(d):
    "full weights, batch reduced to 256 rows") against the float64 oracle:
    every gradient (A18' vs the bf16-policy oracle, A18 vs the unrounded
    one: a kink-free network) and the loss."""
    _check_c3(W.c5(256, 256))


def test_c3_bf16_inputs_passed_as_bf16():
    """Inputs that feed only dots may be passed as bf16 (dlvm.h): identical
    results to passing f32 (the library's own RNE cast)."""
    layers = [(128, 128, "relu"), (128, 64, None)]
    w = W.c3(128, layers=layers)
    ins = w.inputs()
    a = gpu_run(w.text, w.fn, w.grad, ins, seed=w.seed(), dot_precision="bf16", which="grad")["grad"]
    b = gpu_run(w.text, w.fn, w.grad, ins, seed=w.seed(), dot_precision="bf16", which="grad",
                bf16_inputs=(0, 1, 3))["grad"]
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


def test_no_fusion_matches_fusion():
    """DLVM_NO_FUSION (one launch group per instruction) gives the same
    results within fp32 rounding."""
    import paper_1711_03016_b200 as P
    w = W.c1(8)
    ins = w.inputs()
    a = gpu_run(w.text, w.fn, w.grad, ins, seed=np.float32(0.125))["grad"]
    b = gpu_run(w.text, w.fn, w.grad, ins, seed=np.float32(0.125), flags=P.DLVM_NO_FUSION)["grad"]
    for x, y in zip(a, b):
        assert_f32_parity(x, y, np.abs(y) + 1e-3 * np.max(np.abs(y)), rtol=1e-5)


RANDOM_OPS = ["add", "subtract", "multiply", "tanh", "exp", "negate", "relu", "sigmoid"]


def _random_program(rng, R, C):
    """A straight-line program over [R, C] f32 args with row/col/scalar
    broadcast operands, a dot, and a loss (S:L272 random program corpus)."""
    X = f"<{R} x {C} x f32>"
    lines, cur, k = [], "%x", 0
    args = [("x", (R, C)), ("v", (1, C)), ("u", (R, 1)), ("w", (C, C))]
    for _ in range(rng.integers(3, 8)):
        op = RANDOM_OPS[rng.integers(len(RANDOM_OPS))]
        k += 1
        if op in ("add", "subtract", "multiply"):
            other = [f"%v: <1 x {C} x f32>", f"%u: <{R} x 1 x f32>", "0.5: f32", "%x: " + X][rng.integers(4)]
            lines.append(f"    %t{k} = {op} {cur}: {X}, {other}")
        elif op == "relu":
            lines.append(f"    %c{k} = gt {cur}: {X}, 0: f32")
            lines.append(f"    %t{k} = select %c{k}: <{R} x {C} x bool>, {cur}: {X}, 0: f32")
        elif op == "sigmoid":
            lines += [f"    %n{k} = negate {cur}: {X}", f"    %e{k} = exp %n{k}: {X}",
                      f"    %d{k} = add %e{k}: {X}, 1: f32", f"    %t{k} = divide 1: f32, %d{k}: {X}"]
        else:
            lines.append(f"    %t{k} = {op} {cur}: {X}")
        cur = f"%t{k}"
        if rng.random() < 0.3:
            k += 1
            lines.append(f"    %t{k} = dot {cur}: {X}, %w: <{C} x {C} x f32>")
            cur = f"%t{k}"
    lines += [f"    %s = multiply {cur}: {X}, {cur}: {X}", f"    %q = reduce %s: {X} by add along 1",
              f"    %L = reduce %q: <{R} x f32> by add along 0", "    return %L: f32"]
    sig = ", ".join(f"<{a} x {b} x f32>" for _, (a, b) in args)
    head = ['module "rnd"', "stage raw", f"func @f: ({sig}) -> f32 {{",
            "'entry(" + ", ".join(f"%{n}: <{a} x {b} x f32>" for n, (a, b) in args) + "):"]
    tail = ["}", "", "[gradient @f]", f"func @g: ({sig}) -> ({sig})", ""]
    return "\n".join(head + lines + tail), args


@pytest.mark.parametrize("seed", range(8))
def test_random_programs(seed):
    rng = np.random.default_rng(100 + seed)
    R, C = [(8, 12), (33, 20), (64, 64), (5, 7)][seed % 4]
    text, args = _random_program(rng, R, C)
    m = oracle.parse(text)
    ins = [(rng.uniform(-1, 1, s) * (0.3 if n == "w" else 1.0)).astype(np.float32) for n, s in args]
    res = gpu_run(text, "f", "g", ins)
    ins64 = [x.astype(np.float64) for x in ins]
    rp = oracle.run(m, "f", ins64)[0]
    assert_f32_parity(res["primal"][0], rp, term_bound(m, "f", ins64)[0], what="random primal")
    ref = oracle.run(m, "g", ins64)
    gm = _grad_module(m, "g")
    bg = term_bound(gm, "g", ins64)
    emu = f32_emulation(gm, "g", ins64)   # fp32 conditioning of this random program
    for k, (g, r, b, e) in enumerate(zip(res["grad"], ref, bg, emu)):
        assert_f32_parity(g, r, b, what=f"random grad out{k}\n{text}", extra=4.0 * float(np.max(np.abs(e - r))))


@pytest.mark.parametrize("case", ["c1", "c2", "c3", "c5", "rnn", "hvp"])
def test_specialized_programs_bit_identical_to_interpreter(case):
    """Compile-time specialised programs (spec_programs.inc) and the generic
    interpreter evaluate the same ops in the same order: bit-identical
    (EW kernels, tcgen05 epilogues, SIMT epilogues)."""
    import paper_1711_03016_b200 as P
    if case == "c1":
        w, prec = W.c1(), "f32"
    elif case == "rnn":
        w, prec = W.rnn(8, 256, 128, 192), "bf16"
    elif case == "hvp":
        w, prec = W.mlp_hvp(256, 128, 192, 64), "bf16"
    elif case == "c2":
        w, prec = W.c2(256, 4096), "f32"
    elif case == "c3":
        w, prec = W.c3(256, layers=[(512, 512, "relu"), (512, 256, None)]), "bf16"
    else:
        w, prec = W._mlp_workload(5, "c5s", 256, [(512, 512, "tanh")] * 2, ("normal",), ("uniform", -0.5, 0.5),
                                  1.0 / 256, "bf16", 256), "bf16"
    ins = w.inputs()
    a = gpu_run(w.text, w.fn, w.grad, ins, seed=w.seed(), dot_precision=prec)
    b = gpu_run(w.text, w.fn, w.grad, ins, seed=w.seed(), dot_precision=prec, flags=P.DLVM_NO_SPECIALIZE)
    for x, y in zip(a["primal"] + a["grad"], b["primal"] + b["grad"]):
        np.testing.assert_array_equal(x, y)


def test_sgd_update_two_outputs_one_kernel():
    """H12: W' = W - lr*G (element-wise IR), returned as the fp32 master and
    as a bf16 copy (output dtype policy, dlvm.h) -- one kernel, in place."""
    import torch
    import paper_1711_03016_b200 as P
    shapes = [(300, 520), (1, 520)]
    text = W.sgd_ir(shapes, 1e-3, [True, False])
    f = P.Function(text, "sgd", None)
    assert f.num_launches(0) == 2
    rng = np.random.default_rng(21)
    host = []
    for s in shapes:
        host += [rng.normal(size=s).astype(np.float32), rng.normal(size=s).astype(np.float32)]
    dev = torch.device("cuda:0")
    ins = [torch.from_numpy(x).to(dev) for x in host]
    wb = torch.empty(shapes[0], dtype=torch.bfloat16, device=dev)
    outs = [ins[0], wb, ins[2]]  # in place on the masters
    f.run(ins, outputs=outs)
    torch.cuda.synchronize()
    m = oracle.parse(text)
    ref = oracle.run(m, "sgd", [x.astype(np.float64) for x in host])
    assert_f32_parity(outs[0].cpu().double().numpy(), ref[0], what="W master")
    assert_f32_parity(outs[2].cpu().double().numpy(), ref[2], what="b master")
    got_b = wb.cpu().to(torch.float64).numpy()
    np.testing.assert_array_equal(got_b, oracle.interp.bf16_round(outs[0].cpu().numpy()))


def test_single_partial_reduction_output_bound_as_bf16():
    """c1's db2 / db1 (and the kept loss) come from single-partial epilogue
    reductions, which the GEMM writes straight into an f32 output; bound as
    bf16 (dlvm.h: an f32 output may be requested as bf16) the conditional
    finalize runs instead and must store bf16_round of the same f32 value."""
    import torch
    import paper_1711_03016_b200 as P
    w = W.c1()
    f = P.Function(w.text, w.fn, w.grad)
    dev = torch.device("cuda:0")
    ins = [torch.from_numpy(x).to(dev) for x in w.inputs()]
    seed = torch.tensor(np.float32(w.seed()), device=dev)
    ref = [o.cpu().numpy() for o in f.grad_run(ins, seed=seed)]
    outs = f._outputs(1, dev, None)
    bf = [1, 3, 4]  # db1 [1,128], db2 [1,10], loss
    for k in bf:
        outs[k] = torch.empty(outs[k].shape, dtype=torch.bfloat16, device=dev)
    f.grad_run(ins, seed=seed, outputs=outs)
    torch.cuda.synchronize()
    for k, (o, r) in enumerate(zip(outs, ref)):
        got = o.cpu().to(torch.float32).numpy()
        want = bf16_round(r) if k in bf else r
        assert np.array_equal(got.reshape(-1).view(np.uint32), np.asarray(want, np.float32).reshape(-1).view(np.uint32)), k


def test_simt_split_k_shapes():
    """SIMT dot (fp32 policy) on SM-starved grids, where K is split over a
    thread-block cluster and summed through distributed shared memory, plus a
    ragged tail in every dimension (A17 term bound)."""
    for (M, K, N) in [(7, 1531, 13), (32, 784, 128), (1, 4096, 1), (65, 300, 70)]:
        text = _dot_ir(M, K, N, False, False)
        rng = np.random.default_rng(M * 7 + K)
        a, b = rng.normal(size=(M, K)).astype(np.float32), rng.normal(size=(K, N)).astype(np.float32)
        res = gpu_run(text, "f", None, [a, b], which="primal")
        m = oracle.parse(text)
        ins64 = [a.astype(np.float64), b.astype(np.float64)]
        ref = oracle.run(m, "f", ins64)
        assert_f32_parity(res["primal"][0], ref[0], term_bound(m, "f", ins64)[0], what=f"dot {M}x{K}x{N}")


def test_higher_order_fig4_d2g_dw2_f32():
    """Second-order gradient (Fig. 4 `d2g_dw2`) executed by the
    same kernels: the handle's primal is the canonicalised `dg`, its
    gradient differentiates `dg`'s output 0 w.r.t. w (A17 term bounds)."""
    from test_oracle_higher_order import fig4_second_order
    t = fig4_second_order(64, 96, 80)
    m = oracle.parse(t)
    rng = np.random.default_rng(23)
    ins = [(rng.normal(size=p.shape) * s).astype(np.float32)
           for p, s in zip(m.functions["g"].param_types, (1.0, 0.1, 0.1))]
    res = gpu_run(t, "dg", "d2g_dw2", ins)
    ins64 = [x.astype(np.float64) for x in ins]
    bp = term_bound(_grad_module(m, "dg"), "dg", ins64)
    # out2 = tanh(x.w + b): the dot's accumulation error passes through the
    # 1-Lipschitz tanh, so its bound is the pre-activation's sum|terms|
    bp[2] = np.abs(ins64[0]) @ np.abs(ins64[1]) + np.abs(ins64[2])
    for k, (g, r) in enumerate(zip(res["primal"], oracle.run(m, "dg", ins64))):
        assert_f32_parity(g, r, bp[k], what=f"dg out{k}")
    (ref,) = oracle.run(m, "d2g_dw2", ins64)
    bound = term_bound(_grad_module(m, "d2g_dw2"), "d2g_dw2", ins64)[0]
    assert_f32_parity(res["grad"][0], ref, bound, what="d2g_dw2")


@pytest.mark.parametrize("prec,dims", [("f32", (48, 40, 56, 24)), ("bf16", (512, 256, 384, 128))])
def test_higher_order_mlp_hessian_vector_product(prec, dims):
    """MLP loss Hessian-vector product: [gradient @df from 0 wrt 1, 3
    seedable] with the direction v as seed.  f32: A17 term bounds; bf16
    (tcgen05 GEMMs for every dot of the second-order program): normwise 2e-2
    against the oracle under the bf16 dot policy (A18')."""
    from test_oracle_higher_order import _mlp2
    B, I, H, O = dims
    text, P_ = _mlp2(B, I, H, O, "tanh")
    m = oracle.parse(text)
    rng = np.random.default_rng(29)
    ins = [(rng.normal(size=s) * (1.0 / np.sqrt(s[0]) if n.startswith("w") else 1.0)).astype(np.float32)
           for n, s in P_]
    v = rng.normal(size=(I, H)).astype(np.float32)
    ins64 = [x.astype(np.float64) for x in ins] + [v.astype(np.float64)]
    if prec == "f32":
        res = gpu_run(text, "df", "hvp", ins, seed=v, which="grad")
        ref = oracle.run(m, "hvp", ins64)
        bounds = term_bound(_grad_module(m, "hvp"), "hvp", ins64)
        for k, (g, r, b) in enumerate(zip(res["grad"], ref, bounds)):
            assert_f32_parity(g, r, b, what=f"hvp out{k}")
    else:
        ins = [bf16_round(x) if n in ("x", "w1", "w2") else x for x, (n, _) in zip(ins, P_)]
        ins64 = [x.astype(np.float64) for x in ins] + [v.astype(np.float64)]
        res = gpu_run(text, "df", "hvp", ins, seed=v, dot_precision="bf16", which="grad")
        assert "gemm tcgen05" in res["fn"].print(3)
        ref = oracle.run(m, "hvp", ins64, dot_policy="bf16")
        for k, (g, r) in enumerate(zip(res["grad"], ref)):
            assert_normwise(g, r, 2e-2, what=f"hvp bf16 out{k}")


def test_rnn_two_segment_gemm_f32():
    """Unrolled RNN (linear algebra fusion) under the fp32 dot
    policy: multi-segment SIMT GEMMs, ragged shapes (A17 term bounds)."""
    w = W.rnn(3, 70, 40, 52, "f32")
    _check_f32(w, w.inputs(), w.seed())


def test_rnn_multi_segment_gemm_bf16():
    """Same program at tcgen05 shapes: forward cells with 2 K segments, dW and
    dU with T K segments of mixed operand majors; normwise 2e-2 against the
    oracle under the bf16 dot policy (A18')."""
    w = W.rnn(4, 384, 192, 320)
    m = oracle.parse(w.text)
    ins = [bf16_round(x) if a.name.startswith(("x", "W", "U")) or a.name == "h0" else x
           for x, a in zip(w.inputs(), w.args)]
    res = gpu_run(w.text, w.fn, w.grad, ins, seed=w.seed(), dot_precision="bf16")
    assert res["fn"].print(3).count("K segments") >= 2 + 4
    ins64 = [x.astype(np.float64) for x in ins]
    ref_p = oracle.run(m, w.fn, ins64, dot_policy="bf16")
    assert_normwise(res["primal"][0], ref_p[0], 2e-2, what="rnn loss")
    ref = oracle.run(m, w.grad, ins64 + [np.float64(w.seed())], dot_policy="bf16")
    for k, (g, r) in enumerate(zip(res["grad"], ref)):
        assert_normwise(g, r, 2e-2, what=f"rnn grad out{k}")


def test_optimised_program_parity_f32():
    """The create-time optimiser's output (algebra simplification, CSE,
    matrix-chain reordering) on the GPU against the oracle run on the
    program as written; bounds from the optimised IR's own terms (the
    reassociated chain sums different products)."""
    from test_capi_cpu import OPT_PROGRAM
    rng = np.random.default_rng(41)
    ins = [(rng.normal(size=s) * 0.5).astype(np.float32) for s in [(16, 4), (4, 512), (512, 8), (16, 8)]]
    res = gpu_run(OPT_PROGRAM, "f", "df", ins)
    ins64 = [x.astype(np.float64) for x in ins]
    m = oracle.parse(OPT_PROGRAM)
    om = oracle.parse('module "o"\nstage optimizable\n' + res["fn"].print(6) + "\n" + res["fn"].print(7))
    assert_f32_parity(res["primal"][0], oracle.run(m, "f", ins64)[0], term_bound(om, "f", ins64)[0], what="opt f")
    for k, (g, r, b) in enumerate(zip(res["grad"], oracle.run(m, "df", ins64), term_bound(om, "df", ins64))):
        assert_f32_parity(g, r, b, what=f"opt df out{k}")


@pytest.mark.parametrize("case", ["c1", "c3s", "fig4", "rnn"])
def test_cross_ad_oracle_adjoint_ir_on_gpu(case):
    """SURVEY §4 T6 cross-AD check: the ORACLE's adjoint IR (oracle/adjoint.py,
    generated independently of the C++ AD, no DCE) executed as a plain
    function by the GPU library equals the oracle's value-level gradient."""
    import paper_1711_03016_b200 as P
    if case == "c1":
        w, prec = W.c1(), "f32"
        ins = w.inputs() + [np.float32(w.seed())]
        name, text = w.grad, w.text
    elif case == "c3s":
        w, prec = W.c3(64, layers=[(96, 80, "relu"), (80, 40, None)]), "f32"
        ins = w.inputs() + [np.float32(w.seed())]
        name, text = w.grad, w.text
    elif case == "rnn":
        w, prec = W.rnn(3, 24, 16, 20, "f32"), "f32"
        ins = w.inputs() + [np.float32(w.seed())]
        name, text = w.grad, w.text
    else:
        text, name, prec = W.fig4_ir(8, 12, 6), "dg", "f32"
        m0 = oracle.parse(text)
        rng = np.random.default_rng(2)
        ins = [rng.uniform(-1, 1, t.shape).astype(np.float32) for t in m0.functions["g"].param_types]
    m = oracle.parse(text)
    gtext = 'module "x"\nstage optimizable\n' + oracle.adjoint_text(
        m.functions[m.functions[name].gradient.source], m.functions[name].gradient, name)
    ins = [np.asarray(x, dtype=np.float32) for x in ins]
    res = gpu_run(gtext, name, None, ins, dot_precision=prec, which="primal")
    ins64 = [x.astype(np.float64) for x in ins]
    ref = oracle.run(m, name, ins64)
    bounds = term_bound(oracle.parse(gtext), name, ins64)
    for k, (g, r, b) in enumerate(zip(res["primal"], ref, bounds)):
        assert_f32_parity(g, r, b, what=f"{case} oracle-IR out{k}")


@pytest.mark.parametrize("case", ["c3", "c2"])
def test_bf16_storage_inputs_bit_identical(case):
    """dlvm.h: an f32 argument may be passed as bf16 (bf16 dot policy: any;
    fp32 policy: not feeding a dot).  With bf16-representable values the
    results are bit-identical to passing the same values as f32 (the kernels
    widen on load: EW loads, GEMM epilogue inputs, dot operands)."""
    import torch
    import paper_1711_03016_b200 as P
    dev = torch.device("cuda:0")
    if case == "c3":
        w, prec = W.c3(256, layers=[(512, 512, "relu"), (512, 256, None)]), "bf16"
        as_bf = {"t", "b1", "b2", "x", "w1"}
    else:
        w, prec = W.c2(96, 4096), "f32"
        as_bf = {"x", "w", "b", "m"}
    f = P.Function(w.text, w.fn, w.grad, dot_precision=prec)
    host = [bf16_round(x) for x in w.inputs()]
    ins32 = [torch.from_numpy(x).to(dev) for x in host]
    ins16 = [t.to(torch.bfloat16) if a.name in as_bf else t for t, a in zip(ins32, w.args)]
    sd = w.seed()
    seed = torch.from_numpy(np.array(bf16_round(np.asarray(sd, np.float32)) if np.ndim(sd) else np.float32(sd))).to(dev)
    a = [o.cpu().numpy() for o in f.run(ins32) + f.grad_run(ins32, seed=seed)]
    b = [o.cpu().numpy() for o in f.run(ins16) + f.grad_run(ins16, seed=seed)]
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("case", ["c3", "c2"])
def test_bool_byte_storage_inputs_bit_identical(case):
    """dlvm.h: an f32 argument that feeds no dot may be passed as DLVM_BOOL
    bytes (1.0 where nonzero, else 0.0).  One-hot targets (c3: read by the
    loss in the last GEMM's epilogue) and the c2 mask (EW kernel) as bytes
    give bit-identical results to the same 0/1 values as f32; a dot operand
    passed as bytes is a usage error."""
    import torch
    import paper_1711_03016_b200 as P
    dev = torch.device("cuda:0")
    if case == "c3":
        w, prec, name = W.c3(256, layers=[(512, 512, "relu"), (512, 256, None)]), "bf16", "t"
    else:
        w, prec, name = W.c2(96, 4096), "f32", "m"
    f = P.Function(w.text, w.fn, w.grad, dot_precision=prec)
    host = w.inputs()
    ins32 = [torch.from_numpy(x).to(dev) for x in host]
    insb = [(t != 0) if a.name == name else t for t, a in zip(ins32, w.args)]
    sd = w.seed()
    seed = torch.from_numpy(np.array(np.asarray(sd, np.float32))).to(dev)
    a = [o.cpu().numpy() for o in f.run(ins32) + f.grad_run(ins32, seed=seed)]
    b = [o.cpu().numpy() for o in f.run(insb) + f.grad_run(insb, seed=seed)]
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
    if case == "c3":
        bad = [(t != 0) if a.name == "x" else t for t, a in zip(ins32, w.args)]
        with pytest.raises(P.DlvmError) as e:
            f.run(bad)
        from paper_1711_03016_b200.dlvm import DLVM_ERR_USAGE
        assert e.value.status == DLVM_ERR_USAGE


@pytest.mark.parametrize("case", ["c3", "c5"])
def test_A20_kept_loss_bit_equal_bf16(case):
    """Reading A20: the kept loss of the gradient run equals
    dlvm_fn_run's bit for bit, also when the loss is a full sum fused into a
    tcgen05 epilogue whose program (and chunk width) differs between the
    primal and the gradient plans."""
    if case == "c3":
        w = W.c3(256, layers=[(256, 256, "relu"), (256, 100, None)])
    else:
        w = W._mlp_workload(5, "c5s", 256, [(256, 256, "tanh")] * 2, ("normal",), ("uniform", -0.5, 0.5),
                            1.0 / 256, "bf16", 256)
    res = gpu_run(w.text, w.fn, w.grad, w.inputs(), seed=w.seed(), dot_precision="bf16")
    assert res["grad"][-1] == res["primal"][0]


_JIT_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import paper_1711_03016_b200 as P, workloads as W
from helpers import gpu_run
w = W.c3(256, layers=[(512, 512, "relu"), (512, 256, None)])
r = gpu_run(w.text, w.fn, w.grad, w.inputs(), seed=w.seed(), dot_precision="bf16")
w2 = W.c2(96, 4096)
r2 = gpu_run(w2.text, w2.fn, w2.grad, w2.inputs(), seed=w2.seed())
np.savez({out!r}, *(r["primal"] + r["grad"] + r2["primal"] + r2["grad"]))
print(r["fn"].print(8).count("specialised"))
"""


def test_jit_kernels_bit_identical_to_ahead_of_time(tmp_path):
    """DLVM_FORCE_JIT=1 compiles every EW / tcgen05 program with NVRTC at
    create time instead of using the ahead-of-time registry: same templates,
    same arithmetic -> bit-identical results (c3 bf16 GEMM epilogues, c2 EW)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for force in ("0", "1"):
        out = str(tmp_path / f"r{force}.npz")
        script = _JIT_SCRIPT.format(root=root, tests=os.path.dirname(os.path.abspath(__file__)), out=out)
        env = dict(os.environ, DLVM_FORCE_JIT=force)
        p = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=600)
        assert p.returncode == 0, p.stderr[-3000:]
        if force == "1":
            assert int(p.stdout.strip().splitlines()[-1]) >= 5  # GEMM epilogues really were JIT-compiled
        outs[force] = np.load(out)
    for k in outs["0"].files:
        np.testing.assert_array_equal(outs["0"][k], outs["1"][k])


def test_c2_tall_thin_column():
    """c2 on a [2^27, 1] column: the element-wise grid raises rows per thread
    past 64 to keep gridDim.y <= 65535; sampled rows against the oracle and
    the full column sums dw, db against the oracle over the whole column."""
    import torch
    import paper_1711_03016_b200 as P
    R = 1 << 27
    w = W.c2(R, 1)
    f = P.Function(w.text, w.fn, w.grad)
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(2027)  # c2's distributions, drawn directly (the block generator is slow at 2^27 rows)
    xs = [rng.standard_normal((R, 1)).astype(np.float32), rng.uniform(0.5, 1.5, (1, 1)).astype(np.float32),
          rng.uniform(-0.5, 0.5, (1, 1)).astype(np.float32), (rng.random((R, 1)) < 0.9).astype(np.float32)]
    ins = [torch.from_numpy(x).to(dev) for x in xs]
    g = rng.standard_normal((R, 1)).astype(np.float32)
    seed = torch.from_numpy(g).to(dev)
    (y,) = f.run(ins)
    dx, dw, db = f.grad_run(ins, seed=seed)
    torch.cuda.synchronize()
    rows = np.array([0, 1, 77777, R // 2 + 3, R - 1])
    sub = [xs[0][rows].astype(np.float64), xs[1].astype(np.float64), xs[2].astype(np.float64),
           xs[3][rows].astype(np.float64)]
    mm = oracle.parse(W.chain_ir(len(rows), 1))
    (yr,) = oracle.run(mm, "chain", sub)
    assert_f32_parity(y.cpu().numpy()[rows], yr, what="tall y rows")
    dxr, _, _ = oracle.run(mm, "chain_grad", sub + [g[rows].astype(np.float64)])
    assert_f32_parity(dx.cpu().numpy()[rows], dxr, what="tall dx rows")
    # full column sums: the oracle on the whole column, bounds from the oracle's adjoint IR
    full = [x.astype(np.float64) for x in xs] + [g.astype(np.float64)]
    _, rdw, rdb = oracle.run(oracle.parse(w.text), "chain_grad", full)
    gm = _grad_module(oracle.parse(w.text), "chain_grad")
    _, bdw, bdb = term_bound(gm, "chain_grad", full)
    assert_f32_parity(db.cpu().numpy(), rdb, bdb, what="db")
    assert_f32_parity(dw.cpu().numpy(), rdw, bdw, what="dw")


_TMA_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import workloads as W
from helpers import gpu_run
w = W.c2(300, 4096)
r = gpu_run(w.text, w.fn, w.grad, w.inputs(), seed=w.seed())
np.savez({out!r}, *(r["primal"] + r["grad"]))
"""


def test_tma_staged_ew_kernel_bit_identical(tmp_path):
    """The opt-in TMA-staged element-wise kernel (DLVM_EW_TMA=1: cp.async.bulk
    ring, producer/consumer warps) computes the same program in the same row
    order per column as ew2d_kernel: bit-identical c2 forward and adjoint,
    including the column-sum partials."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for tma in ("0", "1"):
        out = str(tmp_path / f"t{tma}.npz")
        script = _TMA_SCRIPT.format(root=root, tests=os.path.dirname(os.path.abspath(__file__)), out=out)
        p = subprocess.run([sys.executable, "-c", script], env=dict(os.environ, DLVM_EW_TMA=tma),
                           capture_output=True, text=True, timeout=600)
        assert p.returncode == 0, p.stderr[-3000:]
        outs[tma] = np.load(out)
    for k in outs["0"].files:
        np.testing.assert_array_equal(outs["0"][k], outs["1"][k])


def _min_compare_margin(mod, fname, ins64):
    """Smallest |a - b| over the operands of every compare in the function (f64)."""
    fn = mod.functions[fname]
    env = oracle.interp.evaluate(fn, ins64)
    margin = np.inf
    for ins in fn.insts:
        if ins.opcode in ("lt", "le", "gt", "ge", "eq", "ne"):
            a, b = [oracle.interp.literal_value(o) if o.kind == "literal" else env[o.name] for o in ins.operands]
            d = np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64))
            d = d[d > 0]  # exact ties (a value compared with its own copy) decide the same on both sides
            if d.size:
                margin = min(margin, float(np.min(d)))
    return margin


@pytest.mark.parametrize("seed", range(16))
def test_random_nd_programs(seed):
    """Rank-1..5 programs (NumPy broadcasting across ranks, rank>2
    transposes, reductions along random axes, compare/select) run on the GPU
    against the oracle: primal loss and every gradient."""
    import nd_programs as ND
    rng = np.random.default_rng(5000 + seed)
    text, args = ND.nd_program(rng)
    m = oracle.parse(text)
    # a comparison is a discrete decision: inputs whose compares come within
    # 1e-4 of a tie are redrawn (fp32 and f64 may decide a near-tie differently)
    best = None
    for _ in range(50):
        cand = ND.nd_inputs(rng, args)
        mg = _min_compare_margin(m, "f", [x.astype(np.float64) for x in cand])
        if best is None or mg > best[0]:
            best = (mg, cand)
        if mg > 1e-4:
            break
    ins = best[1]
    res = gpu_run(text, "f", "g", ins)
    ins64 = [x.astype(np.float64) for x in ins]
    rp = oracle.run(m, "f", ins64)[0]
    assert_f32_parity(res["primal"][0], rp, term_bound(m, "f", ins64)[0], what="nd primal\n" + text)
    ref = oracle.run(m, "g", ins64)
    gm = _grad_module(m, "g")
    bg = term_bound(gm, "g", ins64)
    emu = f32_emulation(gm, "g", ins64)
    for k, (g, r, b, e) in enumerate(zip(res["grad"], ref, bg, emu)):
        assert_f32_parity(g, r, b, what=f"nd grad out{k}\n{text}", extra=4.0 * float(np.max(np.abs(e - r))))
    # the same program returning every value it defines: returned views
    # (transposes, shapeCasts) and values stored by the kernel that reads them
    body, _ = ND.nd_program(np.random.default_rng(5000 + seed), all_values=True)
    mb = oracle.parse(body)
    gs = gpu_run(body, "f", None, ins, which="primal")["primal"]
    rs = oracle.run(mb, "f", ins64)
    bs = term_bound(mb, "f", ins64)
    es = f32_emulation(mb, "f", ins64)
    for k, (g, r, b, e) in enumerate(zip(gs, rs, bs, es)):
        assert_f32_parity(g, r, b, what=f"nd value {k}\n{body}", extra=4.0 * float(np.max(np.abs(e - r))))


@pytest.mark.parametrize("seed", range(8))
def test_random_nd_programs_bf16(seed):
    """The N-d corpus (without compare/select) under the bf16 dot policy:
    loss and gradients within A18' (2e-2 normwise) of the oracle under the
    same bf16 operand rounding, every intermediate of the all-values
    variant likewise."""
    import nd_programs as ND
    text, args = ND.nd_program(np.random.default_rng(7000 + seed), allow_select=False)
    ins = ND.nd_inputs(np.random.default_rng(17 + seed), args)
    m = oracle.parse(text)
    res = gpu_run(text, "f", "g", ins, dot_precision="bf16")
    ins64 = [x.astype(np.float64) for x in ins]
    assert_normwise(res["primal"][0], oracle.run(m, "f", ins64, dot_policy="bf16")[0], what="nd bf16 loss\n" + text)
    for k, (g, r) in enumerate(zip(res["grad"], oracle.run(m, "g", ins64, dot_policy="bf16"))):
        assert_normwise(g, r, what=f"nd bf16 grad out{k}\n{text}")
    body, _ = ND.nd_program(np.random.default_rng(7000 + seed), all_values=True, allow_select=False)
    mb = oracle.parse(body)
    gs = gpu_run(body, "f", None, ins, dot_precision="bf16", which="primal")["primal"]
    for k, (g, r) in enumerate(zip(gs, oracle.run(mb, "f", ins64, dot_policy="bf16"))):
        assert_normwise(g, r, what=f"nd bf16 value {k}\n{body}")


@pytest.mark.parametrize("seed,prec", [(s, "f32") for s in range(3)] + [(s, "bf16") for s in range(5)])
def test_random_nd_programs_wide(seed, prec):
    """Wide N-d programs (last dim 64..256, >= 128 rows): dots through
    reshapes of padded homes run on tcgen05 (bf16) / SIMT (fp32); the
    all-values variant adds forward products (`reduce ... by multiply`)."""
    import nd_programs as ND
    kw = dict(wide=True, allow_select=prec == "f32")
    text, args = ND.nd_program(np.random.default_rng(9000 + seed), **kw)
    m = oracle.parse(text)
    rng = np.random.default_rng(99 + seed)
    best = None
    for _ in range(20):
        cand = ND.nd_inputs(rng, args)
        mg = _min_compare_margin(m, "f", [x.astype(np.float64) for x in cand])
        if best is None or mg > best[0]:
            best = (mg, cand)
        if mg > 1e-4:
            break
    ins = best[1]
    ins64 = [x.astype(np.float64) for x in ins]
    pol = "bf16" if prec == "bf16" else None
    res = gpu_run(text, "f", "g", ins, dot_precision=prec)
    body, _ = ND.nd_program(np.random.default_rng(9000 + seed), all_values=True, **kw)
    mb = oracle.parse(body)
    gs = gpu_run(body, "f", None, ins, dot_precision=prec, which="primal")["primal"]
    rs = oracle.run(mb, "f", ins64, dot_policy=pol)
    if prec == "bf16":
        assert_normwise(res["primal"][0], oracle.run(m, "f", ins64, dot_policy=pol)[0], what="wide loss\n" + text)
        for k, (g, r) in enumerate(zip(res["grad"], oracle.run(m, "g", ins64, dot_policy=pol))):
            assert_normwise(g, r, what=f"wide grad out{k}\n{text}")
        for k, (g, r) in enumerate(zip(gs, rs)):
            assert_normwise(g, r, what=f"wide value {k}\n{body}")
        return
    assert_f32_parity(res["primal"][0], oracle.run(m, "f", ins64)[0], term_bound(m, "f", ins64)[0], what="wide loss")
    ref = oracle.run(m, "g", ins64)
    gm = _grad_module(m, "g")
    for k, (g, r, b, e) in enumerate(zip(res["grad"], ref, term_bound(gm, "g", ins64), f32_emulation(gm, "g", ins64))):
        assert_f32_parity(g, r, b, what=f"wide grad out{k}\n{text}", extra=4.0 * float(np.max(np.abs(e - r))))
    for k, (g, r, b, e) in enumerate(zip(gs, rs, term_bound(mb, "f", ins64), f32_emulation(mb, "f", ins64))):
        assert_f32_parity(g, r, b, what=f"wide value {k}\n{body}", extra=4.0 * float(np.max(np.abs(e - r))))


@pytest.mark.parametrize("seed", range(10))
def test_random_gradient_configurations(seed):
    """Random gradient declarations (`from` either output of a (loss,
    tensor) tuple, `wrt` subsets, `keeping`, scalar or tensor seeds) run on
    the GPU against the oracle: every gradient and kept output."""
    import nd_programs as ND
    rng = np.random.default_rng(300 + seed)
    text, args, cfg = ND.nd_grad_config(rng)
    m = oracle.parse(text)
    best = None
    for _ in range(20):
        cand = ND.nd_inputs(rng, args)
        mg = _min_compare_margin(m, "f", [x.astype(np.float64) for x in cand])
        if best is None or mg > best[0]:
            best = (mg, cand)
        if mg > 1e-4:
            break
    ins = best[1]
    seed_v = rng.uniform(-1, 1, cfg["seed_shape"]).astype(np.float32) if cfg["seedable"] else None
    res = gpu_run(text, "f", "g", ins, seed=seed_v, which="grad")
    ins64 = [x.astype(np.float64) for x in ins]
    gargs = ins64 + ([seed_v.astype(np.float64)] if seed_v is not None else [])
    ref = oracle.run(m, "g", gargs)
    gm = _grad_module(m, "g")
    for k, (g, r, b, e) in enumerate(zip(res["grad"], ref, term_bound(gm, "g", gargs), f32_emulation(gm, "g", gargs))):
        assert_f32_parity(g, r, b, what=f"grad-config out{k} {cfg}\n{text}", extra=4.0 * float(np.max(np.abs(e - r))))


DEGENERATE = '''module "deg"
stage raw
func @f: (f32, <1 x f32>, <1 x 1 x f32>, <1 x 1 x 1 x 1 x 1 x f32>, <1 x 1 x f32>) -> (f32, <1 x 1 x f32>) {
'entry(%s: f32, %v: <1 x f32>, %m: <1 x 1 x f32>, %q: <1 x 1 x 1 x 1 x 1 x f32>, %w: <1 x 1 x f32>):
    %a = multiply %s: f32, %v: <1 x f32>
    %b = add %a: <1 x f32>, %m: <1 x 1 x f32>
    %c = tanh %b: <1 x 1 x f32>
    %d = dot %c: <1 x 1 x f32>, %w: <1 x 1 x f32>
    %e = transpose %d: <1 x 1 x f32>
    %g = multiply %e: <1 x 1 x f32>, %q: <1 x 1 x 1 x 1 x 1 x f32>
    %h = reduce %g: <1 x 1 x 1 x 1 x 1 x f32> by add along 3
    %pq = reduce %q: <1 x 1 x 1 x 1 x 1 x f32> by multiply along 2
    %hp = multiply %h: <1 x 1 x 1 x 1 x f32>, %pq: <1 x 1 x 1 x 1 x f32>
    %k = reduce %hp: <1 x 1 x 1 x 1 x f32> by add along 0
    %r = shapeCast %k: <1 x 1 x 1 x f32> to 1 x 1
    %t = subtract %r: <1 x 1 x f32>, 0.5: f32
    %l = reduce %t: <1 x 1 x f32> by add along 1
    %z = reduce %l: <1 x f32> by add along 0
    %y = power %z: f32, 2: f32
    return (%y: f32, %c: <1 x 1 x f32>)
}

[gradient @f from 0 wrt 0, 1, 2, 4 keeping 1 seedable]
func @g: (f32, <1 x f32>, <1 x 1 x f32>, <1 x 1 x 1 x 1 x 1 x f32>, <1 x 1 x f32>, f32) -> (f32, <1 x f32>, <1 x 1 x f32>, <1 x 1 x f32>, <1 x 1 x f32>)
'''


@pytest.mark.parametrize("prec", ["f32", "bf16"])
def test_degenerate_unit_and_scalar_shapes(prec):
    """Degenerate shapes (SURVEY §8(c) edge cases): scalars, <1>, <1 x 1>,
    rank-5 all-unit tensors, a 1x1x1 dot, reductions along unit axes
    (add and multiply), transposes of unit matrices; primal and a seeded
    gradient with a kept output (the product sits off the active path of
    %q, which is not in wrt)."""
    m = oracle.parse(DEGENERATE)
    vals = [np.float32(0.7), np.array([0.3], np.float32), np.array([[-0.2]], np.float32),
            np.full((1, 1, 1, 1, 1), 1.5, np.float32), np.array([[0.9]], np.float32)]
    if prec == "bf16":
        vals = [bf16_round(np.asarray(v)).reshape(np.shape(v)) for v in vals]
    seed = np.float32(-1.25)
    res = gpu_run(DEGENERATE, "f", "g", vals, seed=seed, dot_precision=prec)
    pol = "bf16" if prec == "bf16" else None
    ins64 = [np.asarray(v, np.float64) for v in vals]
    for g, r in zip(res["primal"], oracle.run(m, "f", ins64, dot_policy=pol)):
        np.testing.assert_allclose(g, r, rtol=1e-5, atol=1e-7)
    for g, r in zip(res["grad"], oracle.run(m, "g", ins64 + [np.float64(seed)], dot_policy=pol)):
        np.testing.assert_allclose(g, r, rtol=1e-5, atol=1e-7)


def test_c2_beyond_int32_element_count():
    """Maximum sizes: the c2 chain over [2^21, 1025] = 2,149,580,800 elements
    (> 2^31: 64-bit element offsets in the EW kernel, 32768-row column-sum
    partials), mask passed as bool bytes.  Oracle checks: sampled rows of y
    and dx (row-local), and dw/db of sampled columns (the oracle runs the
    same program on each full [R, 1] column)."""
    import torch
    import paper_1711_03016_b200 as P
    R, C = 1 << 21, 1025
    dev = torch.device("cuda:0")
    f = P.Function(W.chain_ir(R, C), "chain", "chain_grad")
    gen = torch.Generator(device=dev).manual_seed(2031)
    u = lambda *s: torch.rand(*s, device=dev, generator=gen) * 2 - 1
    x, w, b = u(R, C), u(1, C), u(1, C)
    m = torch.rand(R, C, device=dev, generator=gen) < 0.5
    s = u(R, C)
    (y,) = f.run([x, w, b, m])
    dx, dw, db = f.grad_run([x, w, b, m], seed=s)
    torch.cuda.synchronize()
    h = lambda t: t.cpu().numpy().astype(np.float64)
    rows = [0, 1, R // 2 + 3, R - 1]
    mr = oracle.parse(W.chain_ir(len(rows), C))
    sub = [h(x[rows]), h(w), h(b), h(m[rows])]
    assert_f32_parity(h(y[rows]), oracle.run(mr, "chain", sub)[0], what="y rows")
    assert_f32_parity(h(dx[rows]), oracle.run(mr, "chain_grad", sub + [h(s[rows])])[0], what="dx rows")
    mc = oracle.parse(W.chain_ir(R, 1))
    gc = _grad_module(mc, "chain_grad")
    for j in (0, 1, 511, C - 1):
        col = [h(x[:, j:j + 1]), h(w[:, j:j + 1]), h(b[:, j:j + 1]), h(m[:, j:j + 1]), h(s[:, j:j + 1])]
        _, rdw, rdb = oracle.run(mc, "chain_grad", col)
        _, bdw, bdb = term_bound(gc, "chain_grad", col)
        assert_f32_parity(h(dw[:, j:j + 1]), rdw, bdw, what=f"dw col {j}")
        assert_f32_parity(h(db[:, j:j + 1]), rdb, bdb, what=f"db col {j}")


@pytest.mark.parametrize("N", [1000, 200, 72])
def test_tcgen05_epilogue_unaligned_byte_rows(N):
    """tcgen05 epilogues with caller-owned byte tensors whose rows are not
    16-byte aligned (N % 16 == 8: odd rows start 8 bytes off): a bool mask
    input, a bool output and a byte-stored f32 input.  Rows whose segments
    are not aligned to the epilogue's vector width take its scalar path
    (this crashed with a misaligned address before)."""
    import torch
    M, K = 1024, 256
    A, Bt, Y, Bl = f"<{M} x {K} x f32>", f"<{K} x {N} x f32>", f"<{M} x {N} x f32>", f"<{M} x {N} x bool>"
    text = (f'module "u"\nstage raw\nfunc @f: ({A}, {Bt}, {Bl}, {Y}) -> ({Y}, {Bl}, <{N} x f32>) {{\n'
            f"'entry(%a: {A}, %b: {Bt}, %c: {Bl}, %t: {Y}):\n"
            f"    %r = dot %a: {A}, %b: {Bt}\n"
            f"    %m = select %c: {Bl}, %r: {Y}, 0: f32\n"
            f"    %d = subtract %m: {Y}, %t: {Y}\n"
            f"    %g = gt %d: {Y}, 0: f32\n"
            f"    %s = reduce %d: {Y} by add along 0\n"
            f"    return (%d: {Y}, %g: {Bl}, %s: <{N} x f32>)\n}}\n")
    rng = np.random.default_rng(N)
    a = bf16_round(rng.uniform(-1, 1, (M, K)).astype(np.float32))
    b = bf16_round(rng.uniform(-1, 1, (K, N)).astype(np.float32))
    c = rng.random((M, N)) < 0.5
    t = (rng.random((M, N)) < 0.3).astype(np.float32)
    m = oracle.parse(text)
    ref = oracle.run(m, "f", [a.astype(np.float64), b.astype(np.float64), c, t.astype(np.float64)], dot_policy="bf16")
    for jit in (0, 1):  # compile-time epilogue program (JIT) and the interpreter
        import paper_1711_03016_b200 as P
        fl = 0 if jit else P.DLVM_NO_JIT | P.DLVM_NO_SPECIALIZE
        dev = torch.device("cuda:0")
        f = P.Function(text, "f", None, dot_precision="bf16", flags=fl)
        ins = [torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev), torch.from_numpy(c).to(dev),
               torch.from_numpy(t != 0).to(dev)]  # t passed as bool bytes
        d, g, s = f.run(ins)
        torch.cuda.synchronize()
        # sum|terms| of d = select(c, a.b, 0) - t is |a|.|b| where c holds, plus |t|
        bnd = term_bound(m, "f", [a.astype(np.float64), b.astype(np.float64), c, t.astype(np.float64)])
        assert_f32_parity(d.cpu().numpy().astype(np.float64), ref[0], bnd[0], what=f"d N={N} jit={jit}")
        gd = d.cpu().numpy()
        np.testing.assert_array_equal(g.cpu().numpy(), gd > 0)  # the stored compare agrees with the stored value
        assert_f32_parity(s.cpu().numpy().astype(np.float64), ref[2], bnd[2], what=f"colsum N={N} jit={jit}")


def test_c4_full_size_in_bench_launch_configuration():
    """c4 at full size (batch 65536 on one GPU) exactly as bench.py times it:
    bench.mlp_setup's storage (x, W as bf16; one-hot t as bool bytes) and
    dp.DataParallelStep, i.e. the same plans (CTA-pair tcgen05 GEMMs, split-K
    dW) and launches.  Every gradient is a sum over all 65536 rows, so the
    oracle runs the whole problem (float64, bf16 operand policy A18')."""
    import os
    import sys
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    from paper_1711_03016_b200.dp import DataParallelStep
    w = W.c4(1)
    dev = torch.device("cuda:0")
    f, dev_in, seed, host, n_grads = bench.mlp_setup(w, dev, 0)
    assert dev_in[-1].dtype == torch.bool  # one-hot targets as bytes, as timed
    dps = DataParallelStep(f, n_grads, dev)
    outs = [o.double().cpu().numpy() for o in dps.step(dev_in, seed)]
    torch.cuda.synchronize()
    m = oracle.parse(w.text)
    ins64 = [x.astype(np.float64) for x in host]
    ref = oracle.run(m, w.grad, ins64 + [np.float64(w.seed())], dot_policy="bf16")
    assert len(outs) == len(ref)
    for k, (g, r) in enumerate(zip(outs, ref)):
        assert_normwise(g, r, what=f"c4 full grad out{k}")


SLICE_CAST = '''module "sc"
stage raw
func @f: (<300 x 96 x f32>, <96 x 64 x f32>, <300 x 96 x f32>) -> (<120 x 96 x f32>, <120 x 64 x f32>, <96 x f32>, <120 x 96 x bool>, <120 x 96 x f32>, <200 x 96 x f32>, <96 x f32>) {
'entry(%x: <300 x 96 x f32>, %w: <96 x 64 x f32>, %y: <300 x 96 x f32>):
    %s = slice %x: <300 x 96 x f32> from 37 upto 157
    %t = tanh %s: <120 x 96 x f32>
    %d = dot %t: <120 x 96 x f32>, %w: <96 x 64 x f32>
    %r = reduce %s: <120 x 96 x f32> by add along 0
    %c = gt %s: <120 x 96 x f32>, 0.25: f32
    %cf = dataTypeCast %c: <120 x 96 x bool> to f32
    %m = multiply %cf: <120 x 96 x f32>, %t: <120 x 96 x f32>
    %b = dataTypeCast %m: <120 x 96 x f32> to bool
    %bf = dataTypeCast %b: <120 x 96 x bool> to f32
    %yt = transpose %y: <300 x 96 x f32>
    %ys = slice %x: <300 x 96 x f32> from 100 upto 300
    %e = add %ys: <200 x 96 x f32>, 1: f32
    %q = multiply %e: <200 x 96 x f32>, 0.001: f32
    %qq = add %q: <200 x 96 x f32>, 1: f32
    %p = reduce %qq: <200 x 96 x f32> by multiply along 0
    return (%t: <120 x 96 x f32>, %d: <120 x 64 x f32>, %r: <96 x f32>, %b: <120 x 96 x bool>, %bf: <120 x 96 x f32>, %ys: <200 x 96 x f32>, %p: <96 x f32>)
}
'''

SLICE_CAST_GRAD = '''module "scg"
stage raw
func @f: (<64 x 32 x f32>, <64 x 32 x f32>) -> f32 {
'entry(%x: <64 x 32 x f32>, %y: <64 x 32 x f32>):
    %c = gt %y: <64 x 32 x f32>, 0: f32
    %cf = dataTypeCast %c: <64 x 32 x bool> to f32
    %t = tanh %x: <64 x 32 x f32>
    %m = multiply %t: <64 x 32 x f32>, %cf: <64 x 32 x f32>
    %s = multiply %m: <64 x 32 x f32>, %m: <64 x 32 x f32>
    %r = reduce %s: <64 x 32 x f32> by add along 1
    %l = reduce %r: <64 x f32> by add along 0
    return %l: f32
}

[gradient @f wrt 0]
func @g: (<64 x 32 x f32>, <64 x 32 x f32>) -> <64 x 32 x f32>
'''


@pytest.mark.parametrize("prec", ["f32", "bf16"])
def test_slice_and_datatypecast(prec):
    """`slice` (Table 1; forward) and `dataTypeCast` (L177) on the GPU:
    a slice feeding element-wise ops, a dot, a column sum and a product,
    returned slices (strided views copied out), bool <-> f32 casts as
    values and outputs; and a gradient through a cast mask."""
    rng = np.random.default_rng(55)
    x = rng.uniform(-1, 1, (300, 96)).astype(np.float32)
    w = rng.uniform(-0.3, 0.3, (96, 64)).astype(np.float32)
    y = rng.uniform(-1, 1, (300, 96)).astype(np.float32)
    if prec == "bf16":
        x, w = bf16_round(x), bf16_round(w)
    m = oracle.parse(SLICE_CAST)
    pol = "bf16" if prec == "bf16" else None
    res = gpu_run(SLICE_CAST, "f", None, [x, w, y], which="primal", dot_precision=prec)["primal"]
    ins64 = [x.astype(np.float64), w.astype(np.float64), y.astype(np.float64)]
    ref = oracle.run(m, "f", ins64, dot_policy=pol)
    bnd = term_bound(m, "f", ins64)
    for k, (g, r, b) in enumerate(zip(res, ref, bnd)):
        if r.dtype == np.bool_:
            np.testing.assert_array_equal(g, r, err_msg=f"out{k}")
        elif k == 6:
            np.testing.assert_allclose(g, r, rtol=(200 + 4) * 2.0 ** -23)  # product of 200 factors (A24)
        else:
            assert_f32_parity(g, r, b * (8 if prec == "bf16" else 1), what=f"slice/cast out{k}")
    mg = oracle.parse(SLICE_CAST_GRAD)
    a = rng.uniform(-1, 1, (64, 32)).astype(np.float32)
    c = rng.uniform(-1, 1, (64, 32)).astype(np.float32)
    rg = gpu_run(SLICE_CAST_GRAD, "f", "g", [a, c], dot_precision=prec)
    a64, c64 = a.astype(np.float64), c.astype(np.float64)
    assert_f32_parity(rg["primal"][0], oracle.run(mg, "f", [a64, c64])[0], term_bound(mg, "f", [a64, c64])[0], what="loss")
    assert_f32_parity(rg["grad"][0], oracle.run(mg, "g", [a64, c64])[0], what="grad through cast mask")


OP_SWEEP = '''module "ops"
stage raw
func @f: (<96 x 80 x f32>, <1 x 80 x f32>, <96 x 1 x f32>, <96 x 80 x f32>) -> (f32, <96 x 80 x f32>, <96 x 80 x f32>, <96 x 80 x bool>, <96 x 80 x bool>) {
'entry(%x: <96 x 80 x f32>, %v: <1 x 80 x f32>, %u: <96 x 1 x f32>, %z: <96 x 80 x f32>):
    %x2 = multiply %x: <96 x 80 x f32>, %x: <96 x 80 x f32>
    %a = add %x2: <96 x 80 x f32>, 1: f32
    %e = multiply %v: <1 x 80 x f32>, 2: f32
    %p = power %a: <96 x 80 x f32>, %e: <1 x 80 x f32>
    %lg = log %a: <96 x 80 x f32>
    %sq = sqrt %a: <96 x 80 x f32>
    %ab = abs %x: <96 x 80 x f32>
    %sg = sign %z: <96 x 80 x f32>
    %ex = exp %u: <96 x 1 x f32>
    %dv = divide %lg: <96 x 80 x f32>, %ex: <96 x 1 x f32>
    %s1 = subtract %p: <96 x 80 x f32>, %sq: <96 x 80 x f32>
    %s2 = add %s1: <96 x 80 x f32>, %dv: <96 x 80 x f32>
    %s3 = multiply %s2: <96 x 80 x f32>, %sg: <96 x 80 x f32>
    %s4 = add %s3: <96 x 80 x f32>, %ab: <96 x 80 x f32>
    %c1 = lt %x: <96 x 80 x f32>, %u: <96 x 1 x f32>
    %c2 = le %z: <96 x 80 x f32>, 0: f32
    %c3 = ge %x: <96 x 80 x f32>, %v: <1 x 80 x f32>
    %c4 = eq %sg: <96 x 80 x f32>, 1: f32
    %c5 = ne %sg: <96 x 80 x f32>, -1: f32
    %n1 = negate %s4: <96 x 80 x f32>
    %k1 = select %c1: <96 x 80 x bool>, %s4: <96 x 80 x f32>, %n1: <96 x 80 x f32>
    %k2 = select %c2: <96 x 80 x bool>, %k1: <96 x 80 x f32>, %x: <96 x 80 x f32>
    %k3 = select %c3: <96 x 80 x bool>, %k2: <96 x 80 x f32>, 0.5: f32
    %k4 = select %c5: <96 x 80 x bool>, %k3: <96 x 80 x f32>, %p: <96 x 80 x f32>
    %q = multiply %k4: <96 x 80 x f32>, %k4: <96 x 80 x f32>
    %r = reduce %q: <96 x 80 x f32> by add along 1
    %l = reduce %r: <96 x f32> by add along 0
    return (%l: f32, %k4: <96 x 80 x f32>, %dv: <96 x 80 x f32>, %c4: <96 x 80 x bool>, %c1: <96 x 80 x bool>)
}

[gradient @f from 0 wrt 0, 1, 2]
func @g: (<96 x 80 x f32>, <1 x 80 x f32>, <96 x 1 x f32>, <96 x 80 x f32>) -> (<96 x 80 x f32>, <1 x 80 x f32>, <96 x 1 x f32>)
'''


def test_op_sweep_every_vm_opcode():
    """Every element-wise opcode of the GPU path with broadcasting (Table 1
    L170-L178): negate, tanh-free transcendental set (exp, log, sqrt, abs,
    sign), add/subtract/multiply/divide/power (tensor exponent), all six
    compares (eq/ne on exact +-1 values from sign), select; primal values,
    bool outputs bit-exact, and the gradient wrt three broadcast arguments."""
    m = oracle.parse(OP_SWEEP)
    rng = np.random.default_rng(808)
    best = None
    for _ in range(30):
        ins = [rng.uniform(-1, 1, (96, 80)).astype(np.float32), rng.uniform(-1, 1, (1, 80)).astype(np.float32),
               rng.uniform(-1, 1, (96, 1)).astype(np.float32), rng.uniform(-1, 1, (96, 80)).astype(np.float32)]
        ins[3][rng.random((96, 80)) < 0.1] = 0.0  # sign(0) = 0 cases
        mg = _min_compare_margin(m, "f", [x.astype(np.float64) for x in ins])
        if best is None or mg > best[0]:
            best = (mg, ins)
        if mg > 1e-4:
            break
    ins = best[1]
    ins64 = [x.astype(np.float64) for x in ins]
    res = gpu_run(OP_SWEEP, "f", "g", ins)
    ref = oracle.run(m, "f", ins64)
    bnd = term_bound(m, "f", ins64)
    emu = f32_emulation(m, "f", ins64)
    for k, (g, r, b, e) in enumerate(zip(res["primal"], ref, bnd, emu)):
        if r.dtype == np.bool_:
            np.testing.assert_array_equal(g, r, err_msg=f"op sweep bool out{k}")
        else:
            assert_f32_parity(g, r, b, what=f"op sweep out{k}", extra=4.0 * float(np.max(np.abs(e - r))))
    refg = oracle.run(m, "g", ins64)
    gm = _grad_module(m, "g")
    bg = term_bound(gm, "g", ins64)
    eg = f32_emulation(gm, "g", ins64)
    for k, (g, r, b, e) in enumerate(zip(res["grad"], refg, bg, eg)):
        assert_f32_parity(g, r, b, what=f"op sweep grad out{k}", extra=4.0 * float(np.max(np.abs(e - r))))


def test_concurrent_runs_on_separate_streams_bit_identical():
    """dlvm_fn_run / dlvm_grad_run keep no mutable state in the handle (the
    caller owns workspace and outputs; the binding keeps one workspace per
    stream): the same handle run concurrently on two streams with DIFFERENT
    input values, and a second handle on a third, give bit-identical results
    to sequential runs of each input set (a shared workspace would mix the
    two runs' intermediates)."""
    import torch
    import paper_1711_03016_b200 as P
    dev = torch.device("cuda:0")
    w3 = W.c3(256, layers=[(512, 512, "relu"), (512, 256, None)])
    f3 = P.Function(w3.text, w3.fn, w3.grad, dot_precision="bf16")
    w2 = W.c2(512, 4096)
    f2 = P.Function(w2.text, w2.fn, w2.grad)
    ins3a = [torch.from_numpy(x).to(dev) for x in w3.inputs()]
    ins3b = [torch.from_numpy(x).to(dev) for x in w3.inputs(row_offset=256)]  # other rows of the batch
    ins3b[1] = ins3b[1] * 0.5  # and other weights
    ins2 = [torch.from_numpy(x).to(dev) for x in w2.inputs()]
    s3 = torch.tensor(np.float32(w3.seed()), device=dev)
    s2 = torch.from_numpy(w2.seed()).to(dev)
    ref3a = [o.cpu() for o in f3.grad_run(ins3a, seed=s3)]
    ref3b = [o.cpu() for o in f3.grad_run(ins3b, seed=s3)]
    ref2 = [o.cpu() for o in f2.grad_run(ins2, seed=s2)]
    torch.cuda.synchronize()
    assert not torch.equal(ref3a[0], ref3b[0])
    streams = [torch.cuda.Stream(device=dev) for _ in range(3)]
    outs = []
    for rep in range(4):
        res = []
        for k, st in enumerate(streams):
            with torch.cuda.stream(st):
                if k < 2:
                    res.append(f3.grad_run(ins3a if k == 0 else ins3b, seed=s3, stream=st.cuda_stream))
                else:
                    res.append(f2.grad_run(ins2, seed=s2, stream=st.cuda_stream))
        torch.cuda.synchronize()
        outs.append(res)
    for res in outs:
        for k, r in enumerate(res):
            ref = (ref3a, ref3b, ref2)[k]
            for a, b in zip(r, ref):
                assert torch.equal(a.cpu(), b), f"stream {k}"


@pytest.mark.parametrize("case", ["c1", "c3", "rnn"])
def test_cuda_graph_capture_and_replay_bit_identical(case):
    """dlvm_grad_run neither allocates nor synchronises, so a whole gradient
    step (SIMT and tcgen05 GEMMs, split K, EW kernels, finalizes, PDL
    launches) can be captured into a CUDA graph; replays with new input
    values give bit-identical results to eager runs on the same values."""
    import torch
    import paper_1711_03016_b200 as P
    dev = torch.device("cuda:0")
    if case == "c1":
        w, prec = W.c1(32), "f32"
    elif case == "c3":
        w, prec = W.c3(256, layers=[(512, 512, "relu"), (512, 256, None)]), "bf16"
    else:
        w, prec = W.rnn(4, 256, 256, 256), "bf16"
    f = P.Function(w.text, w.fn, w.grad, dot_precision=prec)
    ins = [torch.from_numpy(x).to(dev) for x in w.inputs()]
    sd = w.seed()
    seed = torch.from_numpy(np.array(np.asarray(sd, np.float32))).to(dev)
    outs = f._outputs(1, dev, None)
    ws = f._workspace(1, dev)
    st = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(st):
        f.grad_run(ins, seed=seed, outputs=outs, workspace=ws, stream=st.cuda_stream)  # warm-up (JIT, modules)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        f.grad_run(ins, seed=seed, outputs=outs, workspace=ws, stream=st.cuda_stream)
    rng = np.random.default_rng(3)
    for rep in range(2):
        for t in ins:  # new values in the captured buffers
            if t.dtype == torch.float32:
                t.copy_(t * float(rng.uniform(0.5, 1.5)))
        g.replay()
        torch.cuda.synchronize()
        got = [o.clone() for o in outs]
        eager = f.grad_run(ins, seed=seed)
        torch.cuda.synchronize()
        for a, b in zip(got, eager):
            assert torch.equal(a, b), case


def test_gradient_ready_events_fire_after_each_gradient_is_final():
    """dlvm_grad_run records gradient k's event after the last step that
    writes it (incl. split-K sum steps): a second stream that waits on the
    event and copies gradient k while later kernels still run must see the
    final value (the data-parallel all-reduce relies on this)."""
    import torch
    import paper_1711_03016_b200 as P
    dev = torch.device("cuda:0")
    w = W.c3(8192, layers=[(512, 512, "relu"), (512, 256, None)])  # dW GEMMs with K = 8192 split in two
    f = P.Function(w.text, w.fn, w.grad, dot_precision="bf16")
    ins = [torch.from_numpy(x).to(dev) for x in w.inputs()]
    seed = torch.tensor(np.float32(w.seed()), device=dev)
    n_grads = 2 * len(w.layers)
    for rep in range(3):
        events = [torch.cuda.Event() for _ in range(n_grads)]
        for e in events:
            e.record()
        main = torch.cuda.current_stream(dev)
        side = torch.cuda.Stream(device=dev)
        outs = f._outputs(1, dev, None)
        for o in outs:
            o.fill_(float("nan"))  # a copy taken too early shows NaN or a partial sum
        f.grad_run(ins, seed=seed, outputs=outs, stream=main.cuda_stream, events=events)
        copies = []
        with torch.cuda.stream(side):
            for k in reversed(range(n_grads)):
                side.wait_event(events[k])
                copies.append((k, outs[k].clone()))
        torch.cuda.synchronize()
        for k, c in copies:
            assert torch.equal(c, outs[k]), f"gradient {k} copied before it was final"


_PDL_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import workloads as W
from helpers import gpu_run
w = W.c3(8192, layers=[(512, 512, "relu"), (512, 256, None)])
r = gpu_run(w.text, w.fn, w.grad, w.inputs(), seed=w.seed(), dot_precision="bf16")
wr = W.rnn(4, 256, 256, 256)
rr = gpu_run(wr.text, wr.fn, wr.grad, wr.inputs(), seed=wr.seed(), dot_precision="bf16")
w2 = W.c2(300, 4096)
r2 = gpu_run(w2.text, w2.fn, w2.grad, w2.inputs(), seed=w2.seed())
np.savez({out!r}, *(r["primal"] + r["grad"] + rr["grad"] + r2["primal"] + r2["grad"]))
"""


def test_pdl_launches_bit_identical_to_plain_launches(tmp_path):
    """Every kernel waits (griddepcontrol.wait) before touching memory its
    predecessor writes, so programmatic dependent launch changes timing
    only: DLVM_PDL=1 and DLVM_PDL=0 give bit-identical c3 (split-K dW),
    rnn (multi-segment GEMMs) and c2 results."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for pdl in ("1", "0"):
        out = str(tmp_path / f"p{pdl}.npz")
        script = _PDL_SCRIPT.format(root=root, tests=os.path.dirname(os.path.abspath(__file__)), out=out)
        p = subprocess.run([sys.executable, "-c", script], env=dict(os.environ, DLVM_PDL=pdl),
                           capture_output=True, text=True, timeout=600)
        assert p.returncode == 0, p.stderr[-3000:]
        outs[pdl] = np.load(out)
    for k in outs["1"].files:
        np.testing.assert_array_equal(outs["1"][k], outs["0"][k])


def test_merged_finalize_mixed_lengths():
    """ONE finalize launch sums three reductions of one EW kernel with
    different lengths and partial layouts (column sums n=1000 over 250 row
    tiles, row sums n=3000 over 4 column tiles, a full sum n=1 over 1000
    tiles): each vs the float64 oracle within the A16 term bound, and
    bit-identical across runs (fixed summation order)."""
    from merged_reductions import merged_reduction_program
    R, C = 3000, 1000
    text = merged_reduction_program(R, C)
    rng = np.random.default_rng(1711)
    x = rng.uniform(-1, 1, (R, C)).astype(np.float32)
    res = gpu_run(text, "f", None, [x], which="primal")
    assert res["fn"].num_launches(0) == 2
    m = oracle.parse(text)
    x64 = x.astype(np.float64)
    ref = oracle.run(m, "f", [x64])
    bnd = term_bound(m, "f", [x64])
    for k, (g, r, b) in enumerate(zip(res["primal"], ref, bnd)):
        assert_f32_parity(g, r, b, what=f"merged finalize out{k}")
    again = gpu_run(text, "f", None, [x], which="primal")
    for g, h in zip(res["primal"], again["primal"]):
        assert np.array_equal(g, h)


def test_merged_finalize_outputs_bound_as_bf16():
    """Small c3 under the bf16 policy (batch 256; tcgen05 and SIMT GEMMs): the
    last forward GEMM's loss (16 partials) and db2 (8 partials x 100) share one
    finalize launch; with every
    bias gradient bound as bf16 (dlvm.h output dtype policy) that launch
    stores bf16 into some homes and f32 into others, selected per reduction:
    each output equals bf16_round / the f32 value of the all-f32 run."""
    import torch
    import paper_1711_03016_b200 as P
    w = W.c3(256, layers=[(256, 256, "relu"), (256, 100, None)])
    f = P.Function(w.text, w.fn, w.grad, dot_precision="bf16")
    assert "finalize %l, %" in f.print(3)
    dev = torch.device("cuda:0")
    ins = [torch.from_numpy(x).to(dev) for x in w.inputs()]
    seed = torch.tensor(np.float32(w.seed()), device=dev)
    ref = [o.cpu().numpy() for o in f.grad_run(ins, seed=seed)]
    outs = f._outputs(1, dev, None)
    bf = [k for k, o in enumerate(outs) if o.dim() == 2 and o.shape[0] == 1]
    assert len(bf) == 2, [tuple(o.shape) for o in outs]
    for k in bf:
        outs[k] = torch.empty(outs[k].shape, dtype=torch.bfloat16, device=dev)
    f.grad_run(ins, seed=seed, outputs=outs)
    torch.cuda.synchronize()
    for k, (o, r) in enumerate(zip(outs, ref)):
        got = o.cpu().to(torch.float32).numpy()
        want = bf16_round(r) if k in bf else r
        assert np.array_equal(got.reshape(-1).view(np.uint32), np.asarray(want, np.float32).reshape(-1).view(np.uint32)), k


def test_softmax_ce_mlp_f32():
    """Softmax cross-entropy MLP (`reduce ... by max`,
    reading A26) under the fp32 dot policy, ragged shapes: loss and every
    gradient against the oracle (A16/A17 bounds from the oracle's adjoint)."""
    w = W.ce_mlp(37, layers=[(70, 52, "tanh"), (52, 13, None)], dot_precision="f32")
    _check_f32(w, w.inputs(), w.seed())


def test_softmax_ce_mlp_bf16():
    """The same loss on tcgen05 GEMMs (bf16 policy): normwise 2e-2 against the
    oracle under the same operand rounding (A18'), and the loss and
    last-layer gradients against the unrounded oracle."""
    w = W.ce_mlp(256, layers=[(256, 256, "relu"), (256, 100, None)])
    _check_c3(w)


def test_reduce_max_ties_bit_exact():
    """Exact ties (dyadic data): the adjoint splits the seed equally among the
    tied maxima, bit for bit as the oracle (values and counts are exact)."""
    T = "<64 x 40 x f32>"
    text = (f'module "m"\nstage raw\nfunc @f: ({T}) -> <64 x f32> {{\n\'entry(%a: {T}):\n'
            f"    %r = reduce %a: {T} by max along 1\n    return %r: <64 x f32>\n}}\n\n"
            f"[gradient @f wrt 0 seedable]\nfunc @g: ({T}, <64 x f32>) -> {T}\n")
    rng = np.random.default_rng(31)
    a = rng.integers(-3, 4, size=(64, 40)).astype(np.float32)  # many ties
    seed = rng.choice([0.5, 1.0, 2.0, -4.0], size=64).astype(np.float32)
    res = gpu_run(text, "f", "g", [a], seed=seed)
    m = oracle.parse(text)
    np.testing.assert_array_equal(res["primal"][0], oracle.run(m, "f", [a.astype(np.float64)])[0])
    ref = oracle.run(m, "g", [a.astype(np.float64), seed.astype(np.float64)])[0]
    # g / k with k in 1..40: exact only when k is a power of two; otherwise one rounding
    assert_f32_parity(res["grad"][0], ref, what="max ties grad")
    k = (a == a.max(axis=1, keepdims=True)).sum(axis=1)
    pow2 = (k & (k - 1)) == 0
    np.testing.assert_array_equal(res["grad"][0][pow2], ref[pow2])


_STREAMS_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import workloads as W
from helpers import gpu_run
outs = []
for w in (W.c3(256, layers=[(512, 512, "relu"), (512, 512, "relu"), (512, 256, None)]),
          W.c3(8192, layers=[(512, 512, "relu"), (512, 256, None)])):
    r = gpu_run(w.text, w.fn, w.grad, w.inputs(), seed=w.seed(), dot_precision="bf16", which="grad")
    outs += r["grad"]
    r = gpu_run(w.text, w.fn, w.grad, w.inputs(), seed=w.seed(), dot_precision="bf16", which="grad")
    outs += r["grad"]  # a second run on the same handle state
np.savez({out!r}, *outs)
"""


def test_two_stream_schedule_bit_identical(tmp_path):
    """The executor's two-stream schedule (independent dW / dX GEMMs of a
    layer on the handle's auxiliary stream, cross-stream event waits, dynamic
    tile scheduling of the GEMMs; opt-in DLVM_CONCURRENT=1) gives
    bit-identical gradients to one stream with static tile order (the
    default), incl. split-K dW GEMMs."""
    import os
    import subprocess
    import sys
    import paper_1711_03016_b200 as P
    w = W.c3(256, layers=[(512, 512, "relu"), (512, 512, "relu"), (512, 256, None)])
    sched = P.Function(w.text, w.fn, w.grad, dot_precision="bf16", flags=P.DLVM_PLAN_ONLY).print(12)
    assert sched.startswith("streams: two") and " aux " in sched, sched
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for conc in ("1", "0"):
        out = str(tmp_path / f"s{conc}.npz")
        script = _STREAMS_SCRIPT.format(root=root, tests=os.path.dirname(os.path.abspath(__file__)), out=out)
        p = subprocess.run([sys.executable, "-c", script], env=dict(os.environ, DLVM_CONCURRENT=conc),
                           capture_output=True, text=True, timeout=600)
        assert p.returncode == 0, p.stderr[-3000:]
        outs[conc] = np.load(out)
    for k in outs["0"].files:
        np.testing.assert_array_equal(outs["0"][k], outs["1"][k])


_TMA_EPI_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import workloads as W
from helpers import gpu_run
outs = []
cases = [
    (W.c3(200, layers=[(136, 264, "relu"), (264, 72, None)]), "bf16"),      # ragged M and N, mask input
    (W.c3(384, layers=[(256, 1000, "relu"), (1000, 100, None)]), "bf16"),   # N = 1000 (bias N % 4 == 0), 128-wide tiles
    (W._mlp_workload(5, "c5t", 320, [(256, 260, "tanh"), (260, 260, "tanh")], ("normal",), ("uniform", -0.5, 0.5),
                     1.0 / 320, "bf16", 320), "bf16"),                        # f32 saved-activation input, N % 4 == 0
    (W.c3(8192, layers=[(512, 512, "relu"), (512, 256, None)]), "bf16"),    # split-K dW (3-D partial stores)
    (W.ce_mlp(256, layers=[(256, 256, "relu"), (256, 100, None)]), "bf16"),  # softmax-CE loss epilogue
]
for w, prec in cases:
    r = gpu_run(w.text, w.fn, w.grad, w.inputs(), seed=w.seed(), dot_precision=prec)
    outs += r["primal"] + r["grad"]
np.savez({out!r}, *outs)
"""


def test_tma_epilogue_bit_identical_to_direct_stores(tmp_path):
    """The TMA epilogue (staged stores and inputs, 64-column warp groups,
    fast-tile loop) computes the same values in the same summation orders as
    the direct row-per-lane epilogue (DLVM_GEMM_TMA_EPI=0): bit-identical
    losses and gradients over ragged tiles, mask / saved-activation / bias
    inputs, split-K partial stores and the softmax-CE loss."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for on in ("1", "0"):
        out = str(tmp_path / f"e{on}.npz")
        script = _TMA_EPI_SCRIPT.format(root=root, tests=os.path.dirname(os.path.abspath(__file__)), out=out)
        p = subprocess.run([sys.executable, "-c", script], env=dict(os.environ, DLVM_GEMM_TMA_EPI=on),
                           capture_output=True, text=True, timeout=900)
        assert p.returncode == 0, p.stderr[-3000:]
        outs[on] = np.load(out)
    for k in outs["0"].files:
        np.testing.assert_array_equal(outs["0"][k], outs["1"][k], err_msg=k)


_SPLIT_RED_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import workloads as W
from helpers import gpu_run
from torch.profiler import ProfilerActivity, profile
outs, n_ew = [], 0
cases = [
    W.c3(8192, layers=[(512, 512, "relu"), (512, 256, None)]),    # dW GEMMs with K = 8192 split in two
    W.c3(8192, layers=[(264, 520, "relu"), (520, 136, None)]),    # ragged tiles
]
for w in cases:
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        r = gpu_run(w.text, w.fn, w.grad, w.inputs(), seed=w.seed(), dot_precision="bf16", which="grad")
        torch.cuda.synchronize()
    n_ew += sum(1 for e in prof.events() if e.device_type.name == "CUDA" and "ew" in e.name and "gemm" not in e.name)
    outs += r["grad"]
# gradients bound as bf16: the sum step runs (the GEMM cannot add into a
# bf16 home) and stores the bf16 rounding of the same f32 sums
import paper_1711_03016_b200 as P
w = cases[0]
f = P.Function(w.text, w.fn, w.grad, dot_precision="bf16")
dev = torch.device("cuda:0")
ins = [torch.from_numpy(x).to(dev) for x in w.inputs()]
seed = torch.tensor(np.float32(w.seed()), device=dev)
o32 = f.grad_run(ins, seed=seed)
o16 = [torch.empty(o.shape, dtype=torch.bfloat16, device=dev) for o in o32]
f.grad_run(ins, seed=seed, outputs=o16)
torch.cuda.synchronize()
bf16_same = all(torch.equal(a.to(torch.bfloat16), b) for a, b in zip(o32, o16))
np.savez({out!r}, *outs, n_ew=np.int64(n_ew), bf16_same=np.int64(bf16_same))
"""


def test_split_k_reduce_add_bit_identical_to_partials(tmp_path):
    """A GEMM whose K is split in two and whose output is bound as f32 adds
    both splits into the zeroed output (TMA reduce-add; red.global.add with
    the direct epilogue) instead of storing partials for a sum step: 0 + a + b
    rounds to fl(a + b) in either order, so the gradients are bit-identical
    to the partials + sum-step path (DLVM_GEMM_SPLITRED=0), and the sum
    steps' EW launches are gone.  With the gradients bound as bf16 the sum
    step runs and stores exactly the bf16 rounding of the f32 results."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for red, tma in (("0", "1"), ("1", "1"), ("1", "0")):
        out = str(tmp_path / f"r{red}{tma}.npz")
        script = _SPLIT_RED_SCRIPT.format(root=root, tests=os.path.dirname(os.path.abspath(__file__)), out=out)
        p = subprocess.run([sys.executable, "-c", script],
                           env=dict(os.environ, DLVM_GEMM_SPLITRED=red, DLVM_GEMM_TMA_EPI=tma),
                           capture_output=True, text=True, timeout=600)
        assert p.returncode == 0, p.stderr[-3000:]
        outs[red + tma] = np.load(out)
    ref = outs["01"]
    for key in ("11", "10"):
        for k in ref.files:
            if k not in ("n_ew", "bf16_same"):
                np.testing.assert_array_equal(outs[key][k], ref[k], err_msg=f"{key} {k}")
        assert int(outs[key]["n_ew"]) < int(ref["n_ew"]), (key, int(outs[key]["n_ew"]), int(ref["n_ew"]))
        assert int(outs[key]["bf16_same"]) == 1, key


_MC_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import workloads as W
from helpers import gpu_run
outs = []
cases = [
    W.c3(1024),                                                      # c3: pair tiles, 4 pair rows
    W.c3(1000, layers=[(520, 1000, "relu"), (1000, 136, None)]),    # ragged: last pair half out of range
    W.c3(8192, layers=[(512, 512, "relu"), (512, 256, None)]),      # split-K dW
    W.c3(8192, layers=[(2048, 4096, "relu"), (4096, 264, None)]),   # hybrid-sized (>= 66 super tiles)
    W.c3(16384, layers=[(2048, 4096, "relu"), (4096, 264, None)]),  # hybrid + split-K dW1 (K = 16384)
]
for w in cases:
    r = gpu_run(w.text, w.fn, w.grad, w.inputs(), seed=w.seed(), dot_precision="bf16")
    outs += r["primal"] + r["grad"]
np.savez({out!r}, *outs)
"""


def test_multicast_clusters_bit_identical_to_pairs(tmp_path):
    """CTA pairs in 4-CTA clusters (two pair tiles stacked in M share their B
    tile through TMA multicast) move operands differently but compute the
    same MMAs in the same order: losses and gradients are bit-identical to
    plain CTA pairs (DLVM_GEMM_MC=0) both for multicast launches alone
    (DLVM_GEMM_MC=2) and for the default hybrid (DLVM_GEMM_MC=1: a
    multicast launch beside a pair launch on super tiles, both fed by one
    counter), incl. a ragged M whose last super tile is half out of range,
    N-major and K-major B and split K (alone and in a hybrid launch); each
    path was really taken
    (DLVM_EPI_VERBOSE)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for mc in ("0", "1", "2"):
        out = str(tmp_path / f"m{mc}.npz")
        script = _MC_SCRIPT.format(root=root, tests=os.path.dirname(os.path.abspath(__file__)), out=out)
        p = subprocess.run([sys.executable, "-c", script], env=dict(os.environ, DLVM_GEMM_MC=mc, DLVM_EPI_VERBOSE="1"),
                           capture_output=True, text=True, timeout=600)
        assert p.returncode == 0, p.stderr[-3000:]
        n_mc = sum(1 for line in p.stderr.splitlines() if "ctas=2 mc=1" in line)
        n_sup = sum(1 for line in p.stderr.splitlines() if "sup=1" in line)
        assert (n_mc > 0) == (mc != "0") and (n_sup > 0) == (mc == "1"), (mc, n_mc, n_sup)
        outs[mc] = np.load(out)
    for mc in ("1", "2"):
        for k in outs["0"].files:
            np.testing.assert_array_equal(outs[mc][k], outs["0"][k], err_msg=f"DLVM_GEMM_MC={mc} {k}")


_DEFER_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import workloads as W
from helpers import gpu_run
outs, plans = [], []
for w in (W.mlp_hvp(256, 128, 192, 64), W.mlp_hvp(1000, 512, 520, 136)):   # the second ragged
    r = gpu_run(w.text, w.fn, w.grad, w.inputs(), seed=w.seed(), dot_precision="bf16")
    outs += r["primal"] + r["grad"]
    plans.append(r["fn"].print(3))
np.savez({out!r}, *outs, deferred=np.int64(sum(p.count("deferred epilogue") for p in plans)))
"""


def test_deferred_epilogue_bit_identical_to_fused():
    """A GEMM epilogue with two or more f32 [M, N] operands (mlp_hvp) runs as
    an EW step after the GEMM stores its raw accumulator: the same program on
    the same f32 values, so losses and Hessian-vector products are
    bit-identical to the fused epilogue (DLVM_EPI_DEFER=0), incl. ragged tiles."""
    import os
    import subprocess
    import sys
    import tempfile
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    with tempfile.TemporaryDirectory() as tmp:
        for d in ("0", "2"):
            out = os.path.join(tmp, f"d{d}.npz")
            script = _DEFER_SCRIPT.format(root=root, tests=os.path.dirname(os.path.abspath(__file__)), out=out)
            p = subprocess.run([sys.executable, "-c", script], env=dict(os.environ, DLVM_EPI_DEFER=d),
                               capture_output=True, text=True, timeout=600)
            assert p.returncode == 0, p.stderr[-3000:]
            outs[d] = dict(np.load(out))
    assert outs["0"]["deferred"] == 0 and outs["2"]["deferred"] >= 4, (outs["0"]["deferred"], outs["2"]["deferred"])
    for k in outs["0"]:
        if k != "deferred":
            np.testing.assert_array_equal(outs["2"][k], outs["0"][k], err_msg=k)
