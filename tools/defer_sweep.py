#!/usr/bin/env python
"""Stress sweep of planner paths on random wide N-d programs (tests/nd_programs.py,
bf16 policy): for seeds [a, b) runs every program's primal + gradient under
two settings of an environment switch (default DLVM_EPI_DEFER=0 vs 2) in
separate processes and checks the outputs bit for bit; prints how many plans
took the path (the count of `marker` in the printed plans).
usage: [SWEEP_PREC=f32] defer_sweep.py a b [VAR v0 v1 marker]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {root!r} + "/tests")
import nd_programs as ND
from helpers import gpu_run
outs, n, owner = [], 0, []
for seed in range({a}, {b}):
    kw = dict(wide=True, allow_select={prec!r} == "f32")
    text, args = ND.nd_program(np.random.default_rng(9000 + seed), **kw)
    ins = ND.nd_inputs(np.random.default_rng(99 + seed), args)
    try:
        r = gpu_run(text, "f", "g", ins, dot_precision={prec!r})
    except Exception as ex:
        outs.append(np.array([float(seed)])); owner.append(seed); print("seed", seed, "error", repr(ex)[:120]); continue
    outs += r["primal"] + r["grad"]
    owner += [seed] * (len(r["primal"]) + len(r["grad"]))
    n += r["fn"].print(2).count({marker!r}) + r["fn"].print(3).count({marker!r})
np.savez({out!r}, *outs, n=np.int64(n), owner=np.array(owner, dtype=np.int64))
"""


def main():
    a, b = int(sys.argv[1]), int(sys.argv[2])
    var, v0, v1, marker = (sys.argv[3:7] if len(sys.argv) > 6 else ("DLVM_EPI_DEFER", "0", "2", "deferred epilogue"))
    import numpy as np
    res = {}
    for v in (v0, v1):
        out = f"/tmp/sweep_{v}.npz"
        prec = os.environ.get("SWEEP_PREC", "bf16")  # f32: the SIMT dot path (and selects in the programs)
        p = subprocess.run([sys.executable, "-c", CHILD.format(root=ROOT, a=a, b=b, out=out, marker=marker, prec=prec)],
                           env=dict(os.environ, **{var: v}), capture_output=True, text=True, timeout=3000)
        if p.returncode:
            print(p.stderr[-2000:])
            sys.exit(1)
        res[v] = dict(np.load(out))
    keys = [k for k in res[v0] if k not in ("n", "owner")]
    # NaN == NaN here: programs whose inputs overflow (exp of a large
    # argument) have NaN gradients, identical on both sides
    bad = [k for k in keys if not np.array_equal(res[v0][k], res[v1][k], equal_nan=True)]
    own = res[v0]["owner"]
    seeds = sorted({int(own[int(k[4:])]) for k in bad})
    print(f"seeds {a}..{b}: {len(keys)} outputs, {var}={v1} path taken {int(res[v1]['n'])} times "
          f"({int(res[v0]['n'])} at {v0}); mismatches: {bad[:10]} (seeds {seeds})")


if __name__ == "__main__":
    main()
