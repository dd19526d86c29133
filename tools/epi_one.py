#!/usr/bin/env python
"""Runs one epilogue program of tools/epi_trace.py (by name prefix) a few
times with the product library: a target for `ncu -k regex:gemm_tc`.
usage: epi_one.py <name prefix> [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
os.environ["DLVM_LIBRARY"] = os.path.join(ROOT, "paper_1711_03016_b200", "libdlvm.so")
import torch  # noqa: E402

import epi_trace as E  # noqa: E402
import paper_1711_03016_b200 as P  # noqa: E402

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
dev = torch.device("cuda:0")
a = torch.randn(E.M, E.K, device=dev).to(torch.bfloat16)
b = torch.randn(E.N, E.K, device=dev).to(torch.bfloat16)
m = torch.rand(E.M, E.N, device=dev) < 0.5
v = torch.randn(1, E.N, device=dev)
for key, (extra, body, rtypes, odt) in E.PROGS.items():
    if not key.startswith(name):
        continue
    rt = rtypes[0] if len(rtypes) == 1 else "(" + ", ".join(rtypes) + ")"
    params = f"{E.A}, {E.B}" + (f", {E.V}" if "%v" in extra else "") + (f", {E.BL}" if "%m" in extra else "")
    text = f'module "e"\nstage raw\nfunc @f: ({params}) -> {rt} {{\n' + E.HEAD.replace("%EXTRA", extra) + body + "}\n"
    f = P.Function(text, "f", None, dot_precision="bf16")
    ins = [a, b] + ([v] if "%v" in extra else []) + ([m] if "%m" in extra else [])
    outs = f.run(ins)
    outs = [o.to(torch.bfloat16) if (k < len(odt) and odt[k] == "bf16") else o for k, o in enumerate(outs)]
    for _ in range(reps):
        f.run(ins, outputs=outs)
    torch.cuda.synchronize()
    print("ran", key)
    break
