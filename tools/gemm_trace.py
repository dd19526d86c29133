#!/usr/bin/env python
"""Phase breakdown of the tcgen05 GEMM launches of one gradient step (trace
build: `DLVM_BUILD_VARIANT=trace python -m paper_1711_03016_b200.build`;
this tool loads libdlvm_trace.so through DLVM_LIBRARY).  Each CTA of each
GEMM writes %globaltimer stamps: entry, after the PDL wait, first TMA
issued, first stage landed (MMA issuer), last MMA committed, first
accumulator ready and last epilogue tile done (epilogue warp 4), exit.
Prints per GEMM the median over CTAs of each stamp relative to that GEMM's
earliest entry, the latest exit, and the gap to the previous GEMM's last
exit (us).
Then, per GEMM, where the time goes in the persistent loop (clock64
cycles, median over CTAs): the MMA issuer's share waiting for an empty
accumulator (the epilogue is behind) and for a full operand stage (the
loads are behind), and the first epilogue warp's share waiting for a full
accumulator (the MMAs are behind).
usage: gemm_trace.py [c3|c4|c4x8]   (c4x8: one rank's c4 shard at N=8)"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("DLVM_LIBRARY", os.path.join(ROOT, "paper_1711_03016_b200", "libdlvm_trace.so"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_1711_03016_b200 as P  # noqa: E402

NAMES = ["entry", "pdl_done", "tma0", "stage0", "mma_end", "acc0", "epi_end", "exit"]


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
    w = W.c3() if cfg == "c3" else W.c4(8) if cfg == "c4x8" else W.c4()
    dev = torch.device("cuda:0")
    f = P.Function(w.text, w.fn, w.grad, dot_precision="bf16")
    ins = [torch.from_numpy(x).to(dev) for x in w.inputs()]
    for i, a in enumerate(w.args):
        if a.name == "x" or a.name.startswith("w"):
            ins[i] = ins[i].to(torch.bfloat16)
    seed = torch.tensor(np.float32(w.seed()), device=dev)
    outs = f._outputs(1, dev, None)
    ws = f._workspace(1, dev)
    n = f.num_launches(1)
    gemms = [f.launch_info(1, i)[0] for i in range(n) if f.launch_info(1, i)[1] > 0]
    G = len(gemms)
    L = P.dlvm.lib()
    L.dlvm_debug_gemm_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
    buf = torch.zeros(G * 148 * 32, dtype=torch.int64, device=dev)
    for _ in range(5):
        f.grad_run(ins, seed=seed, outputs=outs, workspace=ws)
    torch.cuda.synchronize()
    for rep in range(3):
        buf.zero_()
        L.dlvm_debug_gemm_trace(buf.data_ptr(), G)
        f.grad_run(ins, seed=seed, outputs=outs, workspace=ws)
        torch.cuda.synchronize()
        L.dlvm_debug_gemm_trace(None, 1)
    t = buf.cpu().numpy().reshape(G, 148, 32).astype(np.float64)
    t0 = t[t > 0].min()
    prev_exit = None
    print(f"{'gemm':60s} " + " ".join(f"{n:>8s}" for n in NAMES) + f" {'last_exit':>9s} {'gap':>6s}")
    for g in range(G):
        live = t[g][t[g][:, 0] > 0]
        start = live[:, 0].min()
        med = [np.median(live[:, k][live[:, k] > 0] - start) / 1e3 if (live[:, k] > 0).any() else float("nan")
               for k in range(8)]
        last = (live[:, 7].max() - start) / 1e3
        gap = (start - prev_exit) / 1e3 if prev_exit is not None else float("nan")
        prev_exit = live[:, 7].max()
        print(f"{gemms[g][:60]:60s} " + " ".join(f"{m:8.2f}" for m in med) + f" {last:9.2f} {gap:6.2f}"
              f"  ctas={len(live)} t={(start - t0) / 1e3:.1f}")
    print(f"\n{'gemm':60s} {'tiles':>6s} {'mma_wait_acc%':>14s} {'mma_wait_stage%':>16s} {'epi_wait_acc%':>14s}")
    for g in range(G):
        mma = t[g][t[g][:, 18] > 0]
        epi = t[g][t[g][:, 21] > 0]
        med = lambda a: float(np.median(a)) if len(a) else float("nan")
        print(f"{gemms[g][:60]:60s} {med(mma[:, 19]):6.1f} {100 * med(mma[:, 16] / mma[:, 18]):14.1f} "
              f"{100 * med(mma[:, 17] / mma[:, 18]):16.1f} {100 * med(epi[:, 20] / epi[:, 21]):14.1f}")


if __name__ == "__main__":
    main()
