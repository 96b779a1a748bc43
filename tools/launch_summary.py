#!/usr/bin/env python3
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch count, total and average duration (serialised, cold-cache
ncu timings: use for shares, not absolute step times)."""
import collections
import csv
import sys


def summarise(path):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, collections.defaultdict(list)
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            agg[d["Kernel Name"][:70]].append(float(d["Metric Value"]))
    tot = sum(sum(v) for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:70s} n={len(v):4d} tot={sum(v) / 1e3:9.1f}us avg={sum(v) / len(v) / 1e3:8.1f}us "
              f"share={sum(v) / tot:6.3f}")


if __name__ == "__main__":
    summarise(sys.argv[1])
