"""One fast-numerics C3 (MAPPO spread_lite, 2048 envs) episode on cuda:0 for an ncu launch list
(scratch: where the C3 episode time goes). usage: python tools/c3_probe.py N"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_00882_b200 import DpdEngine

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
algo = {"algorithm": "mappo", "agent": {"num": n}, "env": {"type": "spread_lite", "num": 2048, "params": {"accel": 1}},
        "policy_net": {"hidden": [64] * 6}, "loop": {"episodes": 2, "steps_per_episode": 32}}
eng = DpdEngine(algo, device=0, seed=7, numerics="fast")
eng.run_episodes(0, 2)
