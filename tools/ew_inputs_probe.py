#!/usr/bin/env python
"""HBM throughput of an element-wise program against its number of f32
[R, C] operands: y = sum_i (a_i * a_{i+1}) over n inputs, stored as f32 or
bf16 (R=8192, C=4096 by default).  Prints algorithmic GB/s (each operand
read once, the result written once) and the plan's launch shape.
usage: ew_inputs_probe.py [R C]"""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1711_03016_b200 as P  # noqa: E402


def program(n, R, C):
    T = f"<{R} x {C} x f32>"
    args = ", ".join(f"%a{i}: {T}" for i in range(n))
    lines = [f'module "e"\nstage raw\nfunc @f: ({", ".join([T] * n)}) -> {T} {{', f"'entry({args}):"]
    acc = "%a0"
    for i in range(1, n):
        lines.append(f"    %p{i} = multiply {acc}: {T}, %a{i}: {T}")
        lines.append(f"    %s{i} = add %p{i}: {T}, %a{i}: {T}")
        acc = f"%s{i}"
    if n == 1:
        lines.append(f"    %s0 = multiply %a0: {T}, 2: f32")
        acc = "%s0"
    lines.append(f"    return {acc}: {T}")
    lines.append("}")
    return "\n".join(lines) + "\n"


def main():
    R, C = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (8192, 4096)
    dev = torch.device("cuda:0")
    for n in (1, 2, 3, 4, 5, 6):
        f = P.Function(program(n, R, C), "f", None)
        ins = [torch.randn(R, C, device=dev) for _ in range(n)]
        for odt in (torch.float32, torch.bfloat16):
            out = [torch.empty(R, C, device=dev, dtype=odt)]
            ws = f._workspace(0, dev)
            for _ in range(3):
                f.run(ins, outputs=out, workspace=ws)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ts = []
            for _ in range(5):
                torch.cuda.synchronize()
                time.sleep(0.1)
                e0.record()
                for _ in range(10):
                    f.run(ins, outputs=out, workspace=ws)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) / 10)
            ms = statistics.median(ts)
            nbytes = R * C * (4 * n + (4 if odt == torch.float32 else 2))
            shape = [l for l in f.print(9).splitlines() if "space" in l][:1]
            print(f"n={n} out={str(odt)[6:]:9s} {ms * 1e3:8.1f} us {nbytes / ms / 1e6:7.0f} GB/s  "
                  f"{shape[0].strip()[:80] if shape else ''}", flush=True)


if __name__ == "__main__":
    main()
