#!/usr/bin/env python
"""Steady-state time of single small programs (one or two launches each),
replayed REPS times inside one CUDA graph: isolates the SIMT GEMM's K loop,
epilogue and split-K cost from host launch gaps.  GPU only.

  python tools/simt_probe.py [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1711_03016_b200 as P  # noqa: E402


def ty(*s):
    return "<" + " x ".join(map(str, s)) + " x f32>" if s else "f32"


def dot_prog(M, K, N, epi: str):
    args = [("x", (M, K)), ("w", (K, N)), ("b", (1, N)), ("t", (M, N))]
    body = [f"    %z = dot %x: {ty(M, K)}, %w: {ty(K, N)}"]
    if epi == "none":
        ret, rt = "%z", ty(M, N)
    elif epi == "bias":
        body.append(f"    %a = add %z: {ty(M, N)}, %b: {ty(1, N)}")
        ret, rt = "%a", ty(M, N)
    else:  # c1's layer-2 epilogue: sigmoid, squared error, loss reduction
        body += [f"    %a = add %z: {ty(M, N)}, %b: {ty(1, N)}",
                 f"    %n = negate %a: {ty(M, N)}", f"    %e = exp %n: {ty(M, N)}",
                 f"    %d = add %e: {ty(M, N)}, 1: f32", f"    %h = divide 1: f32, %d: {ty(M, N)}",
                 f"    %r = subtract %h: {ty(M, N)}, %t: {ty(M, N)}",
                 f"    %s = multiply %r: {ty(M, N)}, %r: {ty(M, N)}",
                 f"    %q = reduce %s: {ty(M, N)} by add along 1", f"    %l = reduce %q: {ty(M)} by add along 0"]
        ret, rt = "%l", "f32"
    sig = ", ".join(ty(*s) for _, s in args)
    head = f"func @f: ({sig}) -> {rt} {{\n'entry(" + ", ".join(f"%{a}: {ty(*s)}" for a, s in args) + "):"
    return 'module "p"\nstage raw\n\n' + head + "\n" + "\n".join(body) + f"\n    return {ret}: {rt}\n}}\n", args


def time_fn(text, args, reps, env_split=None):
    dev = torch.device("cuda:0")
    f = P.Function(text, "f", None)
    rng = np.random.default_rng(0)
    ins = [torch.from_numpy(rng.uniform(-1, 1, s).astype(np.float32)).to(dev) for _, s in args]
    outs = f._outputs(0, dev, None)
    ws = f._workspace(0, dev)
    run = lambda: f.run(ins, outputs=outs, workspace=ws)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            run()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (5 * reps), f.num_launches(0)


if __name__ == "__main__":
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    cases = [("z1 32x784x128 none", (32, 784, 128, "none")), ("z1 32x784x128 bias", (32, 784, 128, "bias")),
             ("z2 32x128x10 none", (32, 128, 10, "none")), ("z2 32x128x10 loss", (32, 128, 10, "loss")),
             ("d31 784x32x128 none", (784, 32, 128, "none")), ("tiny 32x16x16 none", (32, 16, 16, "none"))]
    for name, (M, K, N, epi) in cases:
        text, args = dot_prog(M, K, N, epi)
        us, nl = time_fn(text, args, reps)
        print(f"{name:24s} launches={nl}  {us:7.2f} us/run (graph, {reps} reps)")
