#!/usr/bin/env python
"""Quick per-kernel timing of one MLP workload's fwd+adjoint step (no oracle,
no e2e): python tools/bench_mlp.py [c4|c4xN|c3|c5] [steps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import workloads as W  # noqa: E402
from paper_1711_03016_b200.dp import DataParallelStep  # noqa: E402

if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    # c4xN: one rank's share of c4 at N GPUs (global batch 65536 / N rows)
    w = W.c4(int(name[3:])) if name.startswith("c4x") else {"c4": lambda: W.c4(1), "c3": W.c3, "c5": W.c5}[name]()
    dev = torch.device("cuda:0")
    f, dev_in, seed, host, n_grads = bench.mlp_setup(w, dev, 0)
    dps = DataParallelStep(f, n_grads, dev)
    step = lambda: dps.step(dev_in, seed)
    for _ in range(3):
        step()
    ms = bench.time_steps(step, K, dev, 1)
    kb = bench.kernel_breakdown(f, 1, step, 3, dev)
    gm = sum(r["ms"] for r in kb if r["flops"] > 0)
    gf = sum(r["flops"] for r in kb)
    print(json.dumps({"workload": w.name, "ms_per_step": ms, "samples_per_s": w.global_batch / ms * 1e3,
                      "gemm_tflops": gf / gm / 1e9 if gm else None}))
    for r in kb:
        t = r["flops"] / r["ms"] / 1e9 if r["flops"] else 0
        print(f"{r['ms']:8.4f} ms {t:7.1f} TF/s  {r['desc'][:110]}")
