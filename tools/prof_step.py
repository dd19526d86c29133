#!/usr/bin/env python
"""Runs a few fwd+adjoint steps of a workload through the C ABI (no timing);
the target for ncu captures:  ncu -k regex:gemm_tc -s S -c 1 python tools/prof_step.py c4 2"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import workloads as W
import paper_1711_03016_b200 as P


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    dev = torch.device("cuda:0")
    if name == "c2":
        w = W.c2()
        f = P.Function(w.text, w.fn, w.grad)
        ins = [torch.from_numpy(x).to(dev) for x in w.inputs()]
        seed = torch.from_numpy(w.seed()).to(dev)
        for _ in range(steps):
            f.run(ins)
            f.grad_run(ins, seed=seed)
    else:
        w = {"c4": lambda: W.c4(1), "c3": W.c3, "c5": W.c5, "c1": W.c1}[name]()
        f = P.Function(w.text, w.fn, w.grad, dot_precision=w.dot_precision)
        ins = []
        for a, x in zip(w.args, w.inputs()):
            t = torch.from_numpy(x).to(dev)
            if w.dot_precision == "bf16" and (a.name == "x" or a.name.startswith("w")):
                t = t.to(torch.bfloat16)
            ins.append(t)
        seed = torch.tensor(np.float32(w.seed()), device=dev)
        for _ in range(steps):
            f.grad_run(ins, seed=seed)
    torch.cuda.synchronize()
    print(f.print(3))


if __name__ == "__main__":
    main()
