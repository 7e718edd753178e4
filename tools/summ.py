"""Prints the episode time and per-phase shares of bench.py JSON lines (scratch helper)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["ms_per_step"], 4), {k: round(v["ms_per_episode"], 4) for k, v in d.get("kernel_shares", {}).items()})
    except Exception as ex:  # noqa: BLE001
        print(f, "unreadable:", ex)
