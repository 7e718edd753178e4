#!/usr/bin/env python3
"""Condenses an ncu --set full report into a JSON summary per kernel launch: duration, DRAM
traffic, pipe utilisation, occupancy and the top warp-stall reasons.

usage: python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/<name>.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_MB": "dram__bytes_read.sum",
    "dram_write_MB": "dram__bytes_write.sum",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pipe_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "fma_pipe_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
}


def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        k = {"kernel": d["Kernel Name"].split("(")[0]}
        for name, m in KEYS.items():
            v = d.get(m)
            if v in (None, ""):
                continue
            v = float(v.replace(",", ""))
            unit = u.get(m, "")
            if name.endswith("_MB"):
                v = v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1.0)
            if name == "duration_us":
                v = v * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(unit, 1.0)
            k[name] = v
        st = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(d[h].replace(",", "") or 0)) for h in hdr
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
        tot = sum(v for _, v in st) or 1.0
        k["top_stalls_pct"] = {n: round(v / tot * 100, 1) for n, v in sorted(st, key=lambda x: -x[1])[:5]}
        out.append(k)
    return out


if __name__ == "__main__":
    print(json.dumps({"report": sys.argv[1], "launches": summarise(sys.argv[1])}, indent=1))
