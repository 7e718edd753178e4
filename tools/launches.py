#!/usr/bin/env python3
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel shares.

usage: python tools/launches.py gpurun_out/launches_fast.csv [--md]
"""
import collections
import csv
import sys

UNIT = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}


def load(path):
    hdr, rows = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                rows.append(d)
    return rows


def summarise(rows):
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in rows:
        name = d["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "")
        us = float(d["Metric Value"].replace(",", "")) * UNIT[d["Metric Unit"]]
        agg[name][0] += 1
        agg[name][1] += us
    total = sum(v[1] for v in agg.values())
    return sorted(((k, n, us, us / total) for k, (n, us) in agg.items()), key=lambda x: -x[2]), total


if __name__ == "__main__":
    rows, total = summarise(load(sys.argv[1]))
    md = "--md" in sys.argv
    if md:
        print("| kernel | launches | total us | mean us | share |\n|---|---:|---:|---:|---:|")
    for k, n, us, sh in rows:
        if md:
            print(f"| `{k}` | {n} | {us:.1f} | {us / n:.1f} | {sh * 100:.1f}% |")
        else:
            print(f"{k:55s} n={n:4d} total={us:10.1f}us mean={us / n:9.1f}us share={sh * 100:5.1f}%")
    print(f"total {total:.1f} us over {sum(r[1] for r in rows)} launches")
