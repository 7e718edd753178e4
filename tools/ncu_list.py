"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-launch or per-kernel."""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("(anonymous namespace)::", "")
    m = re.search(r"k_tgemm<[^>]*>", r[ki])
    if m:
        name = m.group(0)
    us = float(r[vi].replace(",", "")) / 1e3
    if len(sys.argv) > 2:
        print(r[ii], name[:70], f"{us:.1f}")
    agg[name][0] += 1
    agg[name][1] += us
for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{us:10.1f} us  {n:4d}x  {k[:90]}")
