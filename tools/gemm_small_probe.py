#!/usr/bin/env python
"""Fixed cost of single-wave tcgen05 GEMMs (the c3 shapes): M=1024, N=4096
at several K, with no store (fused full sum), a bf16 store, and the dX
epilogue (mask select + bf16 store + column sums).  Each line: ms per launch
over back-to-back launches (PDL overlap included) and TFLOP/s.
usage: gemm_small_probe.py [M N]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1711_03016_b200 as P  # noqa: E402
from ew_probe import time_fn  # noqa: E402

M, N = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (1024, 4096)


def progs(K):
    A, B, Bt, Y = f"<{M} x {K} x f32>", f"<{N} x {K} x f32>", f"<{K} x {N} x f32>", f"<{M} x {N} x f32>"
    body = f"'entry(%a: {A}, %b: {B}):\n    %bt = transpose %b: {B}\n    %r = dot %a: {A}, %bt: {Bt}\n"
    return {
        "no store": (f"func @f: ({A}, {B}) -> f32 {{\n" + body + f"    %s0 = reduce %r: {Y} by add along 1\n"
                     f"    %s1 = reduce %s0: <{M} x f32> by add along 0\n    return %s1: f32\n}}\n", False),
        "bf16 store": (f"func @f: ({A}, {B}) -> {Y} {{\n" + body + f"    return %r: {Y}\n}}\n", False),
        "mask+bf16+colsum": (f"func @f: ({A}, {B}, <{M} x {N} x bool>) -> ({Y}, <{N} x f32>) {{\n"
                             f"'entry(%a: {A}, %b: {B}, %c: <{M} x {N} x bool>):\n"
                             f"    %bt = transpose %b: {B}\n    %r = dot %a: {A}, %bt: {Bt}\n"
                             f"    %m = select %c: <{M} x {N} x bool>, %r: {Y}, 0: f32\n"
                             f"    %s = reduce %m: {Y} by add along 0\n    return (%m: {Y}, %s: <{N} x f32>)\n}}\n", True),
    }


dev = torch.device("cuda:0")
for K in [64, 256, 1024, 4096]:
    a = torch.randn(M, K, device=dev).to(torch.bfloat16)
    b = torch.randn(N, K, device=dev).to(torch.bfloat16)
    c = torch.rand(M, N, device=dev) < 0.5
    for name, (text, mask) in progs(K).items():
        f = P.Function('module "k"\nstage raw\n' + text, "f", None, dot_precision="bf16")
        ins = [a, b, c] if mask else [a, b]
        outs = f.run(ins)
        bf = [o.to(torch.bfloat16) if o.dim() == 2 else o for o in outs]
        ws = f._workspace(0, dev)
        ms = time_fn(lambda: f.run(ins, outputs=bf, workspace=ws), reps=50)
        print(f"M={M} N={N} K={K:5d} {name:18s} {ms * 1000:7.1f} us  {2 * M * N * K / ms / 1e9:7.1f} TFLOP/s", flush=True)
