#!/usr/bin/env python
"""tcgen05 mainloop throughput by operand major-ness at the dW shape
(M = N = 4096, K = 65536; A = transpose of a [K, M] tensor when ta, B given
as [K, N] (N-major) or [N, K] (K-major)); the result is fully reduced in the
epilogue so nothing is stored (informational)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1711_03016_b200 as P  # noqa: E402
from ew_probe import time_fn  # noqa: E402


def prog(M, K, N, ta, tb):
    A = f"<{K} x {M} x f32>" if ta else f"<{M} x {K} x f32>"
    B = f"<{N} x {K} x f32>" if tb else f"<{K} x {N} x f32>"
    lines = [f"func @f: ({A}, {B}) -> f32 {{", f"'entry(%a: {A}, %b: {B}):"]
    a, b = "%a", "%b"
    if ta:
        lines.append(f"    %at = transpose %a: {A}")
        a = "%at"
    if tb:
        lines.append(f"    %bt = transpose %b: {B}")
        b = "%bt"
    lines += [f"    %r = dot {a}: <{M} x {K} x f32>, {b}: <{K} x {N} x f32>",
              f"    %s0 = reduce %r: <{M} x {N} x f32> by add along 1",
              f"    %s1 = reduce %s0: <{M} x f32> by add along 0", "    return %s1: f32", "}"]
    return 'module "m"\nstage raw\n' + "\n".join(lines) + "\n"


if __name__ == "__main__":
    dev = torch.device("cuda:0")
    M, K, N = 4096, 65536, 4096
    for ta, tb in [(0, 1), (1, 0), (1, 1), (0, 0)]:
        f = P.Function(prog(M, K, N, ta, tb), "f", None, dot_precision="bf16")
        a = torch.randn((K, M) if ta else (M, K), device=dev).to(torch.bfloat16)
        b = torch.randn((N, K) if tb else (K, N), device=dev).to(torch.bfloat16)
        outs, ws = f._outputs(0, dev, None), f._workspace(0, dev)
        ms = time_fn(lambda: f.run([a, b], outputs=outs, workspace=ws))
        print(f"A {'M' if ta else 'K'}-major, B {'K' if tb else 'N'}-major: {ms:.3f} ms {2*M*N*K/ms/1e9:.0f} TFLOP/s")
