#!/usr/bin/env python
"""Epilogue cost of single-tile tcgen05 GEMMs (trace build, see
tools/gemm_trace.py): M=1024, N=4096, K=64 (one 256x256 pair tile per CTA,
negligible mainloop) with several epilogue programs; prints the median over
CTAs of (last epilogue tile done - first accumulator ready) in us.
usage: epi_trace.py"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("DLVM_LIBRARY", os.path.join(ROOT, "paper_1711_03016_b200", "libdlvm_trace.so"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1711_03016_b200 as P  # noqa: E402

M, N, K = int(os.environ.get("EPI_M", 1024)), 4096, int(os.environ.get("EPI_K", 64))
A, B, Bt, Y = f"<{M} x {K} x f32>", f"<{N} x {K} x f32>", f"<{K} x {N} x f32>", f"<{M} x {N} x f32>"
BL, V = f"<{M} x {N} x bool>", f"<1 x {N} x f32>"
HEAD = f"'entry(%a: {A}, %b: {B}%EXTRA):\n    %bt = transpose %b: {B}\n    %r = dot %a: {A}, %bt: {Bt}\n"
PROGS = {
    "f32 store": ("", f"    return %r: {Y}\n", [Y], ()),
    "bf16 store": ("", f"    return %r: {Y}\n", [Y], ("bf16",)),
    "u8 store (gt)": ("", f"    %g = gt %r: {Y}, 0: f32\n    return %g: {BL}\n", [BL], ()),
    "bias+relu bf16+u8 (z)": (f", %v: {V}", f"    %s = add %r: {Y}, %v: {V}\n    %c = gt %s: {Y}, 0: f32\n"
                              f"    %h = select %c: {BL}, %s: {Y}, 0: f32\n    return (%c: {BL}, %h: {Y})\n", [BL, Y], ("", "bf16")),
    "mask in, bf16, colsum (d)": (f", %m: {BL}", f"    %s = select %m: {BL}, %r: {Y}, 0: f32\n"
                                  f"    %q = reduce %s: {Y} by add along 0\n    return (%s: {Y}, %q: <{N} x f32>)\n",
                                  [Y, f"<{N} x f32>"], ("bf16", "")),
    "colsum only": ("", f"    %q = reduce %r: {Y} by add along 0\n    return %q: <{N} x f32>\n", [f"<{N} x f32>"], ()),
}


def main():
    dev = torch.device("cuda:0")
    L = P.dlvm.lib()
    L.dlvm_debug_gemm_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
    a = torch.randn(M, K, device=dev).to(torch.bfloat16)
    b = torch.randn(N, K, device=dev).to(torch.bfloat16)
    m = torch.rand(M, N, device=dev) < 0.5
    v = torch.randn(1, N, device=dev)
    buf = torch.zeros(148 * 32, dtype=torch.int64, device=dev)
    for name, (extra, body, rtypes, odt) in PROGS.items():
        rt = rtypes[0] if len(rtypes) == 1 else "(" + ", ".join(rtypes) + ")"
        params = f"{A}, {B}" + (f", {V}" if "%v" in extra else "") + (f", {BL}" if "%m" in extra else "")
        text = f'module "e"\nstage raw\nfunc @f: ({params}) -> {rt} {{\n' + HEAD.replace("%EXTRA", extra) + body + "}\n"
        f = P.Function(text, "f", None, dot_precision="bf16")
        ins = [a, b] + ([v] if "%v" in extra else []) + ([m] if "%m" in extra else [])
        outs = f.run(ins)
        outs = [o.to(torch.bfloat16) if (k < len(odt) and odt[k] == "bf16") else o for k, o in enumerate(outs)]
        ws = f._workspace(0, dev)
        for _ in range(3):
            f.run(ins, outputs=outs, workspace=ws)
        torch.cuda.synchronize()
        res = []
        for rep in range(5):
            buf.zero_()
            L.dlvm_debug_gemm_trace(buf.data_ptr(), 1)
            f.run(ins, outputs=outs, workspace=ws)
            torch.cuda.synchronize()
            L.dlvm_debug_gemm_trace(None, 1)
            t = buf.cpu().numpy().reshape(148, 32).astype(np.float64)
            live = t[t[:, 5] > 0]
            res.append(np.median(live[:, 6] - live[:, 5]) / 1e3)
            if int(os.environ.get("DLVM_EPI_DBG", "0")) & 8:  # section cycles of epilogue warp 4
                sec = [int(np.median(live[:, 8 + k])) for k in range(7)]
        extra = ""
        if int(os.environ.get("DLVM_EPI_DBG", "0")) & 8:
            extra = " cycles: loop %d tmem %d in %d prog %d st %d red %d stwait %d" % tuple(sec)
        print(f"{name:28s} epilogue {np.median(res):6.2f} us{extra}", flush=True)


if __name__ == "__main__":
    main()
