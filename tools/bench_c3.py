#!/usr/bin/env python3
"""BASELINE configs[2] (C3): MAPPO on spread_lite, agents swept 3 -> 64, 2048 envs, dp-d on one
B200 (exact numerics = bit-exact with the reference; compact critic: the [joint | one-hot] rows
of programs.cpp:390-402 are never materialised). The reference side (oracle/_ref on the host CPU,
one replica thread) is timed where SURVEY §8 quotes it: n=3 at E=2048 and n=8 at E=256.
Episode time = median driver wall_ms over the timed episodes; one JSON line per point.

usage: python tools/bench_c3.py [--agents 3,4,8,16,32,64] [--envs 2048] [--episodes 3] [--no-ref]
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


def algo(n: int, envs: int, episodes: int) -> dict:
    return {"algorithm": "mappo", "agent": {"num": n}, "env": {"type": "spread_lite", "num": envs, "params": {"accel": 1}},
            "policy_net": {"hidden": [64] * 6}, "loop": {"episodes": episodes, "steps_per_episode": 32}}


def ref_point(n: int, envs: int, seed: int) -> dict:
    tool = os.path.join(ROOT, "oracle", "_ref", "ref_tool")
    with tempfile.TemporaryDirectory() as tmp:
        ap, dp = os.path.join(tmp, "a.json"), os.path.join(tmp, "d.json")
        json.dump(algo(n, envs, 1), open(ap, "w"))
        json.dump({"workers": ["local"], "slots_per_worker": {"cpu": 1, "accel": 1}, "distribution_policy": "dp-d"},
                  open(dp, "w"))
        out = subprocess.run([tool, "run", ap, dp, str(seed)], check=True, capture_output=True, text=True).stdout
    r = json.loads(out)
    ms = r["episodes"][0]["wall_ms"]
    return {"arm": "reference dp-d (CPU, 1 replica thread)", "agents": n, "envs": envs, "episode_ms": ms,
            "env_steps_per_s": envs * 32 / (ms * 1e-3)}


def ours_point(n: int, envs: int, episodes: int, seed: int, numerics: str = "exact") -> dict:
    from paper_2210_00882_b200 import Program

    prog = Program(algo(n, envs, episodes), {"workers": ["local"], "slots_per_worker": {"cpu": 1, "accel": 1},
                                             "distribution_policy": "dp-d", "numerics": numerics})
    prog.run_local(seed=seed, episodes=1)  # engine build + graph capture
    csv, _ = prog.run_local(seed=seed)
    ms = statistics.median(float(l.split(",")[1]) for l in csv.strip().split("\n")[1:])
    if numerics == "exact":
        arm = "ours dp-d fused, 1 x B200, numerics=exact (compact critic)"
    else:
        roll = "fused tensor-core rollout" if n <= 16 else "split-f16 tcgen05 GEMM rollout"
        pol = "fused tcgen05 policy learn" if 2 + 2 * n <= 64 else "layer-wise tcgen05 policy learn"
        cri = ", compact critic: tcgen05 joint GEMMs" if 2 * n * n + 3 * n > 64 else ""
        arm = f"ours dp-d fused, 1 x B200, numerics=fast ({roll}, {pol}{cri})"
    return {"arm": arm, "agents": n, "envs": envs,
            "episode_ms": ms, "env_steps_per_s": envs * 32 / (ms * 1e-3)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--agents", default="3,4,8,16,32,64")
    ap.add_argument("--envs", type=int, default=2048)
    ap.add_argument("--episodes", type=int, default=3)
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--no-ref", action="store_true")
    ap.add_argument("--fast-only", action="store_true")
    a = ap.parse_args()
    if not a.no_ref:
        for n, envs in ((3, 2048), (8, 256)):
            print(json.dumps({"config": "C3", **ref_point(n, envs, a.seed)}), flush=True)
            print(json.dumps({"config": "C3", **ours_point(n, envs, a.episodes, a.seed)}), flush=True)
    for n in (int(x) for x in a.agents.split(",")):
        if not a.fast_only:
            print(json.dumps({"config": "C3", **ours_point(n, a.envs, a.episodes, a.seed)}), flush=True)
        if True:  # fast numerics: every n (wide policies on the layer-wise path)
            print(json.dumps({"config": "C3", **ours_point(n, a.envs, a.episodes, a.seed, "fast")}), flush=True)


if __name__ == "__main__":
    main()
