#!/usr/bin/env python3
"""Warp-stall samples per CUDA source line (file, line) from
`ncu -i REP --page source --csv --print-source cuda,sass --launch-skip K --launch-count 1`.
usage: python tools/ncu_lines.py src.csv [N]"""
import csv
import os
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg, fname, last, seen, hdr = {}, '?', None, set(), None
for r in rows:
    if len(r) >= 2 and r[0] == 'File Path':
        fname = os.path.basename(r[1])
        continue
    if len(r) >= 5 and r[0] == 'Line No':
        hdr = r
        continue
    if hdr is None or len(r) < 5:
        continue
    if r[0] != '':
        last = (fname, r[0], r[1].strip()[:80])
        continue
    if r[2] in seen:
        continue
    seen.add(r[2])
    try:
        s = float(r[4])
    except ValueError:
        continue
    agg[last] = agg.get(last, 0) + s
tot = sum(agg.values())
print('total samples', tot)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:n]:
    print(f"{v / tot * 100:5.1f}% {k[0][:18]:18s} {k[1]:>5} {k[2]}")


def reasons(path, keys):
    """stall-reason breakdown of the given (file, line) keys"""
    rows = list(csv.reader(open(path)))
    fname, last, seen, hdr, out = '?', None, set(), None, {}
    for r in rows:
        if len(r) >= 2 and r[0] == 'File Path':
            fname = os.path.basename(r[1])
            continue
        if len(r) >= 5 and r[0] == 'Line No':
            hdr = r
            continue
        if hdr is None or len(r) < 5:
            continue
        if r[0] != '':
            last = (fname, r[0])
            continue
        if r[2] in seen or last not in keys:
            continue
        seen.add(r[2])
        d = out.setdefault(last, {})
        for i, c in enumerate(hdr):
            if c.startswith('stall_') and 'Not Issued' not in c:
                try:
                    d[c[6:]] = d.get(c[6:], 0) + float(r[i])
                except ValueError:
                    pass
    return out


if len(sys.argv) > 3:
    keys = set()
    for spec in sys.argv[3].split(','):
        f, l = spec.split(':')
        keys.add((f, l))
    for k, d in reasons(sys.argv[1], keys).items():
        print(k, sorted(((round(v), nm) for nm, v in d.items() if v > 0), reverse=True)[:5])
