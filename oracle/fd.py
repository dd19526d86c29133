"""Central finite differences, the independent pin for the oracle's
reverse sweep (test infrastructure only).

fd_grad returns d/dx_i of sum(seed * f_o(x)) by
    (F(x + h e_k) - F(x - h e_k)) / (2 h)
for every element k of argument i, in float64 (default h = 1e-6).
"""

from __future__ import annotations

from typing import Sequence

import numpy as np

from .interp import run_function
from .ir import Function


def fd_grad(src: Function, inputs: Sequence, wrt: int, from_: int = 0,
            seed=None, h: float = 1e-6) -> np.ndarray:
    xs = [np.array(x, dtype=np.float64) if t.dtype.startswith("f") else np.array(x)
          for x, t in zip(inputs, src.param_types)]
    shape = src.result_types[from_].shape
    s = np.ones(shape) if seed is None else np.asarray(seed, dtype=np.float64).reshape(shape)

    def F(vals):
        y = run_function(src, vals)[from_]
        return float(np.sum(s * y))

    x = xs[wrt]
    g = np.zeros(x.shape, dtype=np.float64)
    flat = x.reshape(-1)
    gf = g.reshape(-1)
    for k in range(flat.size):
        orig = flat[k]
        flat[k] = orig + h
        fp = F(xs)
        flat[k] = orig - h
        fm = F(xs)
        flat[k] = orig
        gf[k] = (fp - fm) / (2.0 * h)
    return g
