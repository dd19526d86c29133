"""Debug aid: run random N-d programs (tests/nd_programs.py) on the GPU under
each subsystem switch and report the primal error vs the oracle, plus the
per-value error of every intermediate (the program rewritten to return all
its f32 values)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import nd_programs as ND  # noqa: E402
import oracle  # noqa: E402
import paper_1711_03016_b200 as P  # noqa: E402
from helpers import gpu_run  # noqa: E402


seeds = [int(s) for s in sys.argv[1:]] or [22]
for seed in seeds:
    rng = np.random.default_rng(5000 + seed)
    text, args = ND.nd_program(rng)
    ins = ND.nd_inputs(rng, args)
    ref = oracle.run(oracle.parse(text), "f", [x.astype(np.float64) for x in ins])[0]
    line = [f"seed {seed}:"]
    for name, fl in [("default", 0), ("no_fusion", P.DLVM_NO_FUSION), ("no_spec", P.DLVM_NO_SPECIALIZE),
                     ("no_opt", P.DLVM_NO_OPT), ("no_jit", P.DLVM_NO_JIT)]:
        g = gpu_run(text, "f", None, ins, flags=fl, which="primal")["primal"][0]
        line.append(f"{name} {float(abs(g - ref) / (abs(ref) + 1e-30)):.1e}")
    print(" ".join(line), flush=True)
    body, _ = ND.nd_program(np.random.default_rng(5000 + seed), all_values=True)
    refs = oracle.run(oracle.parse(body), "f", [x.astype(np.float64) for x in ins])
    gs = gpu_run(body, "f", None, ins, which="primal")["primal"]
    for v, g, r in zip(range(len(refs)), gs, refs):
        e = float(np.max(np.abs(g - r)) / (np.max(np.abs(r)) + 1e-30))
        if e > 1e-5:
            print(f"   {v} {r.shape} rel err {e:.2e}")
    if seed == seeds[0]:
        print(P.Function(text, "f", None).print(2))
