#!/usr/bin/env python
"""Small fwd+adjoint cases for compute-sanitizer (memcheck / racecheck):
c1 (SIMT GEMMs), c2 (EW kernels), small bf16 MLPs (tcgen05 GEMMs with
fused epilogues and reductions, CTA pairs, split-K dW with its sum step),
and an RNN (multi-K-segment GEMMs).  Run under
`compute-sanitizer --tool memcheck|racecheck|synccheck`; summaries in
profiles/r2_sanitizer.txt."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_1711_03016_b200 as P  # noqa: E402


def run(w, prec):
    dev = torch.device("cuda:0")
    f = P.Function(w.text, w.fn, w.grad, dot_precision=prec)
    ins = [torch.from_numpy(x).to(dev) for x in w.inputs()]
    s = w.seed()
    seed = torch.from_numpy(np.array(s, dtype=np.float32)).to(dev)
    f.run(ins)
    f.grad_run(ins, seed=seed)
    torch.cuda.synchronize()


if __name__ == "__main__":
    run(W.c1(), "f32")
    run(W.c2(200, 1030), "f32")
    run(W.c3(256, layers=[(256, 256, "relu"), (256, 200, None)]), "bf16")
    run(W._mlp_workload(5, "c5s", 128, [(256, 256, "tanh")] * 2, ("normal",), ("uniform", -0.5, 0.5),
                        1.0 / 128, "bf16", 128), "bf16")
    # split-K dW GEMMs (K = batch 8192 split 2) with CTA pairs, and the
    # deferred-epilogue sum step
    w = W.c3(8192, layers=[(512, 512, "relu"), (512, 256, None)])
    f = P.Function(w.text, w.fn, w.grad, dot_precision="bf16", flags=P.DLVM_PLAN_ONLY)
    assert "K split" in f.print(3), f.print(3)
    run(w, "bf16")
    # rnn: multi-segment GEMMs
    run(W.rnn(3, 256, 128, 128), "bf16")
    print("sanitize cases done")
