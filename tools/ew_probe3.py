#!/usr/bin/env python
"""The c2 program (forward and adjoint) on 2^28 elements in three row shapes
(informational): shows how the row length / column-strip count changes
bandwidth.  GB/s algorithmic: fwd 12 B/elem, fwd+adj 16 B/elem."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1711_03016_b200 as P  # noqa: E402
import workloads as W  # noqa: E402
from ew_probe import time_fn  # noqa: E402

if __name__ == "__main__":
    dev = torch.device("cuda:0")
    for R, C in [(16384, 16384), (65536, 4096), (262144, 1024), (4096, 65536)]:
        w = W.c2(R, C)
        f = P.Function(w.text, w.fn, w.grad)
        ins = [torch.randn(R, C, device=dev), torch.rand(1, C, device=dev) + 0.5, torch.rand(1, C, device=dev) - 0.5,
               (torch.rand(R, C, device=dev) < 0.9).float()]
        seed = torch.randn(R, C, device=dev)
        o0, o1 = f._outputs(0, dev, None), f._outputs(1, dev, None)
        w0, w1 = f._workspace(0, dev), f._workspace(1, dev)
        ms0 = time_fn(lambda: f.run(ins, outputs=o0, workspace=w0))
        ms1 = time_fn(lambda: f.grad_run(ins, seed=seed, outputs=o1, workspace=w1))
        n = R * C
        print(f"[{R}x{C}] fwd {12 * n / (ms0 * 1e-3) / 1e9:6.0f} GB/s   fwd+adj {16 * n / (ms1 * 1e-3) / 1e9:6.0f} GB/s")
        del ins, seed, o0, o1
