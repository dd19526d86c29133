#!/usr/bin/env python
"""Times single bf16 dots through the C ABI: python tools/gemm_probe.py M K N [ta] [tb] ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1711_03016_b200 as P  # noqa: E402


def dot_ir(M, K, N, ta, tb):
    A = f"<{K} x {M} x f32>" if ta else f"<{M} x {K} x f32>"
    B = f"<{N} x {K} x f32>" if tb else f"<{K} x {N} x f32>"
    lines = ['module "d"', "stage raw", f"func @f: ({A}, {B}) -> <{M} x {N} x f32> {{", f"'entry(%a: {A}, %b: {B}):"]
    a, b = "%a", "%b"
    if ta:
        lines.append(f"    %at = transpose %a: {A}")
        a = "%at"
    if tb:
        lines.append(f"    %bt = transpose %b: {B}")
        b = "%bt"
    lines += [f"    %r = dot {a}: <{M} x {K} x f32>, {b}: <{K} x {N} x f32>", f"    return %r: <{M} x {N} x f32>", "}"]
    return "\n".join(lines) + "\n"


def probe(M, K, N, ta, tb, reps=10):
    f = P.Function(dot_ir(M, K, N, ta, tb), "f", None, dot_precision="bf16")
    dev = torch.device("cuda:0")
    a = torch.randn((K, M) if ta else (M, K), device=dev).to(torch.bfloat16)
    b = torch.randn((N, K) if tb else (K, N), device=dev).to(torch.bfloat16)
    out = [torch.empty(M, N, device=dev)]
    ws = f._workspace(0, dev)
    for _ in range(3):
        f.run([a, b], outputs=out, workspace=ws)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        f.run([a, b], outputs=out, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"M={M} K={K} N={N} ta={ta} tb={tb}: {ms:.4f} ms  {2*M*N*K/ms/1e9:.1f} TFLOP/s")


if __name__ == "__main__":
    args = sys.argv[1:]
    cases = [args[i:i + 5] for i in range(0, len(args), 5)]
    for c in cases:
        probe(int(c[0]), int(c[1]), int(c[2]), int(c[3]), int(c[4]))
