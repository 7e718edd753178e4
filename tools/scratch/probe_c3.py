import json, sys
sys.path.insert(0, '.')
from paper_2210_00882_b200 import DpdEngine
for n in (int(x) for x in sys.argv[1].split(',')):
    algo = {"algorithm": "mappo", "agent": {"num": n}, "env": {"type": "spread_lite", "num": 2048, "params": {"accel": 1}},
            "policy_net": {"hidden": [64] * 6}, "loop": {"episodes": 8, "steps_per_episode": 32}}
    e = DpdEngine(algo, seed=7, numerics="fast")
    e.run_episode(0)
    e.enable_probes(True)
    e.run_episode(1); r, ms = e.run_episode(2)
    p = e.probe_times()
    print(n, round(ms, 2), {k: round(sum(v), 3) for k, v in p.items()}, flush=True)
