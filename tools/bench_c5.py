#!/usr/bin/env python3
"""BASELINE configs[4] (C5): A3C with 24 actors (= 24 gridline envs, length 16, 7-layer MLP
H=64, T=32) - the reference's DP-A (asynchronous actors, CPU) and DP-D (24 replica threads, CPU)
against this repository's fused DP-D with the 24 units folded onto N GPUs (R = 24 / N units per
GPU, flw_run_local). Episode time = the driver's wall_ms (local_run.cpp:540-551), median over
the timed episodes. Prints one JSON line per arm.

usage: python tools/bench_c5.py [--episodes 8] [--gpus 1] [--no-ref]
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

ALGO = {"algorithm": "a3c", "actor": {"num": 24}, "env": {"type": "gridline", "num": 24, "params": {"length": 16}},
        "policy_net": {"hidden": [64] * 6}, "loop": {"episodes": 8, "steps_per_episode": 32}}


def ref_arm(policy: str, episodes: int, seed: int) -> dict:
    tool = os.path.join(ROOT, "oracle", "_ref", "ref_tool")
    algo = dict(ALGO, loop={"episodes": episodes, "steps_per_episode": 32})
    with tempfile.TemporaryDirectory() as tmp:
        ap, dp = os.path.join(tmp, "a.json"), os.path.join(tmp, "d.json")
        json.dump(algo, open(ap, "w"))
        json.dump({"workers": ["local"], "slots_per_worker": {"cpu": 32, "accel": 32},
                   "distribution_policy": policy}, open(dp, "w"))
        out = subprocess.run([tool, "run", ap, dp, str(seed)], check=True, capture_output=True, text=True).stdout
    r = json.loads(out)
    ms = [e["wall_ms"] for e in r["episodes"]][1:]  # first episode = warm-up
    return {"arm": f"reference {policy} (CPU, {os.cpu_count()} cores)", "episode_ms": statistics.median(ms),
            "episodes": len(ms), "final_reward": r["episodes"][-1]["reward"], "grad_messages": r["grad_messages"]}


def ours(numerics: str, gpus: int, episodes: int, seed: int) -> dict:
    from paper_2210_00882_b200 import Program

    algo = dict(ALGO, loop={"episodes": episodes, "steps_per_episode": 32})
    prog = Program(algo, {"workers": ["local"], "slots_per_worker": {"cpu": 32, "accel": 32},
                          "distribution_policy": "dp-d", "numerics": numerics, "replicas_per_gpu": 24 // gpus})
    prog.run_local(seed=seed, episodes=2)  # build engines + capture graphs
    csv, s = prog.run_local(seed=seed)
    ms = [float(l.split(",")[1]) for l in csv.strip().split("\n")[1:]][1:]
    return {"arm": f"ours dp-d fused, {gpus} x B200, {24 // gpus} units/GPU, numerics={numerics}",
            "episode_ms": statistics.median(ms), "episodes": len(ms),
            "final_reward": float(csv.strip().split("\n")[-1].split(",")[2]), "grad_messages": s["grad_messages"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--episodes", type=int, default=8)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--no-ref", action="store_true")
    a = ap.parse_args()
    if not a.no_ref:
        for pol in ("dp-a", "dp-d"):
            print(json.dumps({"config": "C5", **ref_arm(pol, a.episodes, a.seed)}), flush=True)
    for num in ("exact", "fast"):
        print(json.dumps({"config": "C5", **ours(num, a.gpus, a.episodes, a.seed)}), flush=True)


if __name__ == "__main__":
    main()
