"""Per-phase time of one exact MAPPO episode (C3 shape) from the in-graph CUDA-event probes."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_00882_b200 import DpdEngine

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
E = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
numerics = sys.argv[3] if len(sys.argv) > 3 else "exact"
algo = {"algorithm": "mappo", "agent": {"num": n}, "env": {"type": "spread_lite", "num": E, "params": {"accel": 1}},
        "policy_net": {"hidden": [64] * 6}, "loop": {"episodes": 4, "steps_per_episode": 32}}
eng = DpdEngine(algo, seed=7, env_lo=0, env_hi=E, env_total=E, numerics=numerics)
eng.enable_probes(True)
eng.run_episodes(0, 2)
ms = eng.run_episodes(2, 1)
pt = eng.probe_times()
print(json.dumps({"agents": n, "envs": E, "numerics": numerics, "episode_ms": ms, "probes_ms": {k: round(sum(v), 3) for k, v in pt.items()}}))
