"""Debug aid: run random N-d programs (tests/nd_programs.py) on the GPU under
each subsystem switch and report the loss error vs the oracle, plus the
error of every intermediate (the all-values variant).
usage: nd_bisect.py [--wide] [--bf16] [--base B] seed..."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import nd_programs as ND  # noqa: E402
import oracle  # noqa: E402
import paper_1711_03016_b200 as P  # noqa: E402
from helpers import gpu_run  # noqa: E402

argv = sys.argv[1:]
wide = "--wide" in argv
prec = "bf16" if "--bf16" in argv else "f32"
base = 9000 if wide else 5000
if "--base" in argv:
    base = int(argv[argv.index("--base") + 1])
seeds = [int(s) for s in argv if s.isdigit() and str(base) != s] or [0]
kw = dict(wide=wide, allow_select=prec == "f32")
pol = "bf16" if prec == "bf16" else None
for seed in seeds:
    text, args = ND.nd_program(np.random.default_rng(base + seed), **kw)
    ins = ND.nd_inputs(np.random.default_rng(99 + seed), args)
    ins64 = [x.astype(np.float64) for x in ins]
    ref = oracle.run(oracle.parse(text), "f", ins64, dot_policy=pol)[0]
    line = [f"seed {seed} {prec}:"]
    for name, fl in [("default", 0), ("no_fusion", P.DLVM_NO_FUSION), ("no_spec", P.DLVM_NO_SPECIALIZE),
                     ("no_opt", P.DLVM_NO_OPT), ("no_jit", P.DLVM_NO_JIT)]:
        g = gpu_run(text, "f", None, ins, flags=fl, which="primal", dot_precision=prec)["primal"][0]
        line.append(f"{name} {float(abs(g - ref) / (abs(ref) + 1e-30)):.1e}")
    print(" ".join(line), flush=True)
    body, _ = ND.nd_program(np.random.default_rng(base + seed), all_values=True, **kw)
    refs = oracle.run(oracle.parse(body), "f", ins64, dot_policy=pol)
    gs = gpu_run(body, "f", None, ins, which="primal", dot_precision=prec)["primal"]
    for v, (g, r) in enumerate(zip(gs, refs)):
        e = float(np.max(np.abs(g - r)) / (np.max(np.abs(r)) + 1e-30))
        if e > 1e-4:
            print(f"   value {v} {r.shape} rel err {e:.2e}")
    print(P.Function(text, "f", None, dot_precision=prec).print(2))
