#!/usr/bin/env python
"""Quick timing of the c2 element-wise chain (fwd and fwd+adjoint) alone."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

if __name__ == "__main__":
    r, _ = bench.bench_chain(torch.device("cuda:0"), int(sys.argv[1]) if len(sys.argv) > 1 else 20, 3)
    print(json.dumps({k: r[k] for k in ("fwd_gbs", "fwd_adj_gbs")}))
