#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
launches and total time per kernel class.  python tools/launch_summary.py list.csv"""
import csv
import re
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"]
        m = re.search(r"(gemm_tc_kernel|gemm_simt_kernel|ew2d_kernel|ew_kernel|finalize_kernel|cast_bf16_kernel|pack_bf16_kernel)", name)
        key = m.group(1) if m else name[:60]
        if m and m.group(1) == "gemm_tc_kernel":
            c = re.search(r", (\d)>\([^()]*TcParams\)", name)
            key += " (CTA pair)" if c and c.group(1) == "2" else " (1 CTA)"
        us = float(d["Metric Value"]) / (1000.0 if d["Metric Unit"] == "ns" else 1.0)
        if d["Metric Unit"] == "ms":
            us = float(d["Metric Value"]) * 1000.0
        tot[key] += us
        cnt[key] += 1
    s = sum(tot.values())
    print(f"{'kernel class':60s} {'launches':>9s} {'total us':>12s} {'share':>7s}")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{k:60s} {cnt[k]:9d} {tot[k]:12.1f} {100 * tot[k] / s:6.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
