#!/usr/bin/env python
"""Is a persistent tcgen05 GEMM epilogue-bound?  Times M x N x K GEMMs
(default c4's d11: 65536 x 4096 x 1000) with the epilogue programs of
tools/epi_trace.py through the normal build (CUDA events; median of 7 bursts of 8 runs,
each after a 0.3 s cool-down) and prints ms and TFLOP/s per program: when the mainloop hides the
epilogue, every program runs at the plain-store time.
usage: EPI_M=65536 EPI_K=1000 epi_bound.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
os.environ.setdefault("EPI_M", "65536")
os.environ.setdefault("EPI_K", "1000")
# the normal build (epi_trace defaults DLVM_LIBRARY to the trace build)
os.environ.setdefault("DLVM_LIBRARY", os.path.join(ROOT, "paper_1711_03016_b200", "libdlvm.so"))
import torch  # noqa: E402

import epi_trace as T  # noqa: E402
import paper_1711_03016_b200 as P  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    M, N, K = T.M, T.N, T.K
    a = torch.randn(M, K, device=dev).to(torch.bfloat16)
    b = torch.randn(N, K, device=dev).to(torch.bfloat16)
    m = torch.rand(M, N, device=dev) < 0.5
    v = torch.randn(1, N, device=dev)
    try:
        import pynvml
        pynvml.nvmlInit()
        nv = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    except Exception:  # noqa: BLE001
        nv = None
    only = os.environ.get("EPI_ONLY")
    for name, (extra, body, rtypes, odt) in T.PROGS.items():
        if only and not any(o in name for o in only.split(",")):
            continue
        rt = rtypes[0] if len(rtypes) == 1 else "(" + ", ".join(rtypes) + ")"
        params = f"{T.A}, {T.B}" + (f", {T.V}" if "%v" in extra else "") + (f", {T.BL}" if "%m" in extra else "")
        text = f'module "e"\nstage raw\nfunc @f: ({params}) -> {rt} {{\n' + T.HEAD.replace("%EXTRA", extra) + body + "}\n"
        f = P.Function(text, "f", None, dot_precision="bf16")
        ins = [a, b] + ([v] if "%v" in extra else []) + ([m] if "%m" in extra else [])
        outs = f.run(ins)
        outs = [o.to(torch.bfloat16) if (k < len(odt) and odt[k] == "bf16") else o for k, o in enumerate(outs)]
        ws = f._workspace(0, dev)
        for _ in range(5):
            f.run(ins, outputs=outs, workspace=ws)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        # short bursts after a cool-down, median over trials: long runs are
        # power-capped (SM clock 1300-1600 MHz at ~1 kW) and would measure
        # the power limit, not the kernel
        import statistics
        import time
        reps, trials = int(os.environ.get("EPI_REPS", 8)), int(os.environ.get("EPI_TRIALS", 7))
        times, clks = [], []
        for _ in range(trials):
            torch.cuda.synchronize()
            time.sleep(0.3)
            e0.record()
            for _ in range(reps):
                f.run(ins, outputs=outs, workspace=ws)
            e1.record()
            if nv is not None:
                clks.append(pynvml.nvmlDeviceGetClockInfo(nv, pynvml.NVML_CLOCK_SM))
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / reps)
        ms = statistics.median(times)
        clk = f" sm {statistics.median(clks):.0f} MHz (min {min(clks)})" if clks else ""
        print(f"{name:28s} {ms:7.4f} ms/run ({f.num_launches(0)} launches)  {2.0 * M * N * K / ms / 1e9:7.1f} TFLOP/s{clk}",
              flush=True)


if __name__ == "__main__":
    main()
