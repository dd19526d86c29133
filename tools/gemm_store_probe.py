#!/usr/bin/env python
"""Epilogue store cost of the tcgen05 GEMM at [65536, 1024] x [1024, 4096]:
the same dot with no store (fused full reduction), a u8 store (gt mask),
a bf16 store and an f32 store of the [M, N] result (informational)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1711_03016_b200 as P  # noqa: E402
from ew_probe import time_fn  # noqa: E402

M, K, N = 65536, 1024, 4096
A, B, Bt, Y = f"<{M} x {K} x f32>", f"<{N} x {K} x f32>", f"<{K} x {N} x f32>", f"<{M} x {N} x f32>"
HEAD = f'module "k"\nstage raw\n'
BODY = f"'entry(%a: {A}, %b: {B}):\n    %bt = transpose %b: {B}\n    %r = dot %a: {A}, %bt: {Bt}\n"
PROGS = {
    "no store": f"func @f: ({A}, {B}) -> f32 {{\n" + BODY + f"    %s0 = reduce %r: {Y} by add along 1\n    %s1 = reduce %s0: <{M} x f32> by add along 0\n    return %s1: f32\n}}\n",
    "u8 store": f"func @f: ({A}, {B}) -> <{M} x {N} x bool> {{\n" + BODY + f"    %c = gt %r: {Y}, 0: f32\n    return %c: <{M} x {N} x bool>\n}}\n",
    "bf16 store": f"func @f: ({A}, {B}) -> {Y} {{\n" + BODY + f"    return %r: {Y}\n}}\n",
    "f32 store": f"func @f: ({A}, {B}) -> {Y} {{\n" + BODY + f"    return %r: {Y}\n}}\n",
    "mask+bf16": (f"func @f: ({A}, {B}, <{M} x {N} x bool>) -> {Y} {{\n'entry(%a: {A}, %b: {B}, %c: <{M} x {N} x bool>):\n"
                  f"    %bt = transpose %b: {B}\n    %r = dot %a: {A}, %bt: {Bt}\n"
                  f"    %m = select %c: <{M} x {N} x bool>, %r: {Y}, 0: f32\n    return %m: {Y}\n}}\n"),
    "mask+bf16+colsum": (f"func @f: ({A}, {B}, <{M} x {N} x bool>) -> ({Y}, <{N} x f32>) {{\n'entry(%a: {A}, %b: {B}, %c: <{M} x {N} x bool>):\n"
                         f"    %bt = transpose %b: {B}\n    %r = dot %a: {A}, %bt: {Bt}\n"
                         f"    %m = select %c: <{M} x {N} x bool>, %r: {Y}, 0: f32\n"
                         f"    %s = reduce %m: {Y} by add along 0\n    return (%m: {Y}, %s: <{N} x f32>)\n}}\n"),
}
if __name__ == "__main__":
    dev = torch.device("cuda:0")
    a = torch.randn(M, K, device=dev).to(torch.bfloat16)
    b = torch.randn(N, K, device=dev).to(torch.bfloat16)
    for name, body in PROGS.items():
        f = P.Function(HEAD + body, "f", None, dot_precision="bf16")
        outs, ws = f._outputs(0, dev, None), f._workspace(0, dev)
        ins = [a, b]
        if name.startswith("mask"):
            ins.append(torch.rand(M, N, device=dev) > 0.5)
        if name.startswith("bf16") or name.startswith("mask"):
            outs[0] = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        ms = time_fn(lambda: f.run(ins, outputs=outs, workspace=ws))
        print(f"{name:10s}: {ms:.4f} ms  {2 * M * N * K / ms / 1e9:.1f} TFLOP/s")
