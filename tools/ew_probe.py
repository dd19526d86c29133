#!/usr/bin/env python
"""Element-wise bandwidth probe: the library on simple programs over c2's
2^28 elements in two layouts vs torch's 1-D kernels (informational)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1711_03016_b200 as P  # noqa: E402


def ty(R, C):
    return f"<{R} x {C} x f32>"


def prog(R, C, body, nin):
    X = ty(R, C)
    args = ", ".join(f"%a{i}: {X}" for i in range(nin))
    sig = ", ".join([X] * nin)
    return f'module "p"\nstage raw\nfunc @f: ({sig}) -> {X} {{\n\'entry({args}):\n{body}\n    return %y: {X}\n}}\n'


def time_fn(fn, reps=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


if __name__ == "__main__":
    dev = torch.device("cuda:0")
    n = 1 << 28
    for R, C in [(16384, 16384), (262144, 1024), (4096, 65536)]:
        X = ty(R, C)
        for name, body, nin, nb in [
                ("add 2R1W", f"    %y = add %a0: {X}, %a1: {X}", 2, 12),
                ("fma 3R1W", f"    %t = multiply %a0: {X}, %a1: {X}\n    %y = add %t: {X}, %a2: {X}", 3, 16),
                ("tanh 1R1W", f"    %y = tanh %a0: {X}", 1, 8)]:
            f = P.Function(prog(R, C, body, nin), "f", None)
            ins = [torch.randn(R, C, device=dev) for _ in range(nin)]
            outs = f._outputs(0, dev, None)
            ws = f._workspace(0, dev)
            ms = time_fn(lambda: f.run(ins, outputs=outs, workspace=ws))
            print(f"[{R}x{C}] {name:10s} {nb * n / (ms * 1e-3) / 1e9:7.0f} GB/s  {ms:.3f} ms")
