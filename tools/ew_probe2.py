#!/usr/bin/env python
"""c2-forward variants on [16384, 16384] f32: isolates tanh and the
row-broadcast operands (informational; GB/s = 12 B/elem: x, m read, y written)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1711_03016_b200 as P  # noqa: E402
from ew_probe import time_fn  # noqa: E402

R = C = 16384
X, V = f"<{R} x {C} x f32>", f"<1 x {C} x f32>"
HEAD = f'module "p"\nstage raw\nfunc @f: ({X}, {V}, {V}, {X}) -> {X} {{\n\'entry(%x: {X}, %w: {V}, %b: {V}, %m: {X}):\n'
BODIES = {
    "c2 fwd tanh(x*w+b)*m": f"    %a = multiply %x: {X}, %w: {V}\n    %z = add %a: {X}, %b: {V}\n    %t = tanh %z: {X}\n    %y = multiply %t: {X}, %m: {X}",
    "no tanh (x*w+b)*m": f"    %a = multiply %x: {X}, %w: {V}\n    %z = add %a: {X}, %b: {V}\n    %y = multiply %z: {X}, %m: {X}",
    "no bcast tanh(x)*m": f"    %t = tanh %x: {X}\n    %y = multiply %t: {X}, %m: {X}",
    "x*m": f"    %y = multiply %x: {X}, %m: {X}",
}
if __name__ == "__main__":
    dev = torch.device("cuda:0")
    ins = [torch.randn(R, C, device=dev), torch.rand(1, C, device=dev) + 0.5, torch.rand(1, C, device=dev) - 0.5,
           (torch.rand(R, C, device=dev) < 0.9).float()]
    for name, body in BODIES.items():
        f = P.Function(HEAD + body + f"\n    return %y: {X}\n}}\n", "f", None)
        outs = f._outputs(0, dev, None)
        ws = f._workspace(0, dev)
        ms = time_fn(lambda: f.run(ins, outputs=outs, workspace=ws))
        print(f"{name:24s} {12 * R * C / (ms * 1e-3) / 1e9:7.0f} GB/s {ms:.3f} ms  {f.print(2).splitlines()[1].strip()[:60]}")
