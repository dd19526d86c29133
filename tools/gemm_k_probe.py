#!/usr/bin/env python
"""tcgen05 mainloop cost vs K: sum(A.B) with the full reduction fused into
the GEMM epilogue (no [M, N] store), bf16 operands, B K-major (informational)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1711_03016_b200 as P  # noqa: E402
from ew_probe import time_fn  # noqa: E402


def prog(M, K, N):
    A, B, Bt = f"<{M} x {K} x f32>", f"<{N} x {K} x f32>", f"<{K} x {N} x f32>"
    return (f'module "k"\nstage raw\nfunc @f: ({A}, {B}) -> f32 {{\n\'entry(%a: {A}, %b: {B}):\n'
            f"    %bt = transpose %b: {B}\n    %r = dot %a: {A}, %bt: {Bt}\n"
            f"    %s0 = reduce %r: <{M} x {N} x f32> by add along 1\n    %s1 = reduce %s0: <{M} x f32> by add along 0\n"
            f"    return %s1: f32\n}}\n")


if __name__ == "__main__":
    dev = torch.device("cuda:0")
    M, N = 65536, 4096
    for K in [int(k) for k in sys.argv[1:]] or [512, 1024, 2048, 4096]:
        f = P.Function(prog(M, K, N), "f", None, dot_precision="bf16")
        a = torch.randn(M, K, device=dev).to(torch.bfloat16)
        b = torch.randn(N, K, device=dev).to(torch.bfloat16)
        outs, ws = f._outputs(0, dev, None), f._workspace(0, dev)
        ms = time_fn(lambda: f.run([a, b], outputs=outs, workspace=ws))
        print(f"K={K}: {ms:.4f} ms  {2 * M * N * K / ms / 1e9:.1f} TFLOP/s   {f.print(2).splitlines()[1].strip()[:70]}")
