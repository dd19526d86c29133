#!/usr/bin/env python
"""Informational yardstick (not the path): HBM bandwidth torch's own
element-wise kernels reach on c2's shapes (2^28 f32) for the read/write
mixes of the c2 kernels: 1R1W (copy), 2R1W (c2 forward: x, m -> y), 3R1W
(c2 adjoint: x, m, g -> dx).  Compare with bench.py fused_elementwise."""
import torch


def t(fn, nbytes, reps=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return nbytes / (ms * 1e-3) / 1e9, ms


if __name__ == "__main__":
    n = 1 << 28
    dev = torch.device("cuda:0")
    x, m, g, y = (torch.randn(n, device=dev) for _ in range(4))
    print("1R1W copy   GB/s %.0f (%.3f ms)" % t(lambda: y.copy_(x), 8 * n))
    print("2R1W add    GB/s %.0f (%.3f ms)" % t(lambda: torch.add(x, m, out=y), 12 * n))
    print("3R1W addcmul GB/s %.0f (%.3f ms)" % t(lambda: torch.addcmul(x, m, g, out=y), 16 * n))
