#!/usr/bin/env python3
"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`.
usage: python tools/ncu_src_top.py src.csv [N]"""
import csv
import sys


def fnum(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 45
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h) and r[0] != 'Address']
ai, si, ns = h.index('Address'), h.index('Source'), h.index('Warp Stall Sampling (All Samples)')
stall = [i for i, c in enumerate(h) if c.startswith('stall_') and 'Not Issued' not in c]
tot = sum(fnum(r[ns]) for r in data)
print('total samples', tot, 'instructions', len(data))
agg = {}
for r in data:
    for i in stall:
        agg[h[i]] = agg.get(h[i], 0) + fnum(r[i])
print('by reason:', ', '.join(f"{k[6:]} {v / tot * 100:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:10]))
for r in sorted(data, key=lambda r: -fnum(r[ns]))[:n]:
    s = fnum(r[ns])
    reasons = sorted(((fnum(r[i]), h[i][6:]) for i in stall), reverse=True)[:3]
    print(f"{r[ai]:>6} {s / tot * 100:5.1f}% {r[si][:64]:64s} " + ' '.join(f"{nm}:{v / max(s, 1) * 100:.0f}" for v, nm in reasons))
