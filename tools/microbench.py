#!/usr/bin/env python3
"""Runs the scaled-size HBM microbenchmarks (flw_microbench) and prints GB/s vs the measured peak.

usage: python tools/microbench.py [env_step|gae|adam ...]   (default: all three)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2210_00882_b200.api import microbench  # noqa: E402

SIZES = {"env_step": 1 << 21, "gae": 1 << 26, "adam": 1 << 27}

if __name__ == "__main__":
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    for name in sys.argv[1:] or list(SIZES):
        ms, nbytes = microbench(name, SIZES[name], 10)
        gbs = nbytes / (ms * 1e-3) / 1e9
        print(json.dumps({"kernel": name, "n": SIZES[name], "ms": ms, "bytes": nbytes, "GB/s": gbs,
                          "frac_of_peak": gbs / peak}))
