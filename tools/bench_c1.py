#!/usr/bin/env python3
"""BASELINE configs[0] (C1): PPO, 7-layer MLP policy (hidden [64]*6), 200 vectorised envs of the
reference's built-in env (gridline, length 16), T=32, train_iters=4. The reference runs DP-A with
a single learner on the CPU (its "oracle run", plan.cpp DP-A) and DP-D with one unit (== the
unpartitioned interpreter); this repository runs the fused DP-D loop on one B200
(exact numerics: bit-exact with the reference's DP-D; fast numerics: tensor cores).
Episode time = the driver's wall_ms (local_run.cpp:540-551), median over the timed episodes
(the first is a warm-up); env-steps/s = 200 * 32 / episode time. One JSON line per arm.

usage: python tools/bench_c1.py [--episodes 4] [--no-ref]
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ENVS = 200


def algo(episodes: int) -> dict:
    return {"algorithm": "ppo", "env": {"type": "gridline", "num": ENVS, "params": {"length": 16}},
            "policy_net": {"hidden": [64] * 6}, "loop": {"episodes": episodes, "steps_per_episode": 32}}


def line(arm: str, ms: list, rewards: list) -> dict:
    med = statistics.median(ms)
    return {"config": "C1", "arm": arm, "envs": ENVS, "episode_ms": med, "env_steps_per_s": ENVS * 32 / (med * 1e-3),
            "episodes_timed": len(ms), "final_reward": rewards[-1]}


def ref_arm(policy: str, episodes: int, seed: int) -> dict:
    tool = os.path.join(ROOT, "oracle", "_ref", "ref_tool")
    with tempfile.TemporaryDirectory() as tmp:
        ap, dp = os.path.join(tmp, "a.json"), os.path.join(tmp, "d.json")
        json.dump(algo(episodes), open(ap, "w"))
        json.dump({"workers": ["local"], "slots_per_worker": {"cpu": 4, "accel": 4}, "distribution_policy": policy},
                  open(dp, "w"))
        r = json.loads(subprocess.run([tool, "run", ap, dp, str(seed)], check=True, capture_output=True,
                                      text=True).stdout)
    eps = r["episodes"]
    return line(f"reference {policy} (CPU, single learner / unit)", [e["wall_ms"] for e in eps][1:],
                [e["reward"] for e in eps])


def ours(numerics: str, episodes: int, seed: int) -> dict:
    from paper_2210_00882_b200 import Program

    prog = Program(algo(episodes), {"workers": ["local"], "slots_per_worker": {"cpu": 1, "accel": 1},
                                    "distribution_policy": "dp-d", "numerics": numerics})
    prog.run_local(seed=seed, episodes=2)  # engine build + graph capture
    csv, _ = prog.run_local(seed=seed)
    rows = [l.split(",") for l in csv.strip().split("\n")[1:]]
    return line(f"ours dp-d fused, 1 x B200, numerics={numerics}", [float(r[1]) for r in rows][1:],
                [float(r[2]) for r in rows])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--episodes", type=int, default=4)
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--no-ref", action="store_true")
    a = ap.parse_args()
    if not a.no_ref:
        for pol in ("dp-a", "dp-d"):
            print(json.dumps(ref_arm(pol, a.episodes, a.seed)), flush=True)
    for num in ("exact", "fast"):
        print(json.dumps(ours(num, a.episodes, a.seed)), flush=True)


if __name__ == "__main__":
    main()
