"""Generates the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
It builds oracle/_ref/ref_tool (oracle/Makefile `ref`: reference sources compiled where they lie,
plus the builder env synth17x6 registered by link-time wrapping) and records, per case:
  trace_<case>.npz : Interp::whole phase-by-phase tensors (the DP-D k=1 unit)
  run_<case>.npz   : run_plan_local under dp-d with k replicas (episode rewards, final params)
The fixtures are small enough to commit; the GPU box never needs /root/reference.
"""
from __future__ import annotations

import json
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle import pyoracle  # noqa: E402

# name -> (algo config, seed)
TRACE_CASES = {
    "ppo_gridline": ({"algorithm": "ppo", "env": {"type": "gridline", "num": 6, "params": {"length": 8}},
                      "policy_net": {"hidden": [8, 8]}, "loop": {"episodes": 3, "steps_per_episode": 8}}, 5),
    "ppo_gridline_relu": ({"algorithm": "ppo", "env": {"type": "gridline", "num": 5, "params": {"length": 6}},
                           "learner": {"params": {"normalize_adv": False, "lr": 0.01}},
                           "policy_net": {"hidden": [8], "activation": "relu"},
                           "loop": {"episodes": 2, "steps_per_episode": 7}}, 11),
    "ppo_synth7": ({"algorithm": "ppo", "env": {"type": "synth17x6", "num": 8},
                    "policy_net": {"hidden": [16, 16, 16, 16, 16, 16]},
                    "loop": {"episodes": 2, "steps_per_episode": 8}}, 7),
    "ppo_synth_maxsteps": ({"algorithm": "ppo", "env": {"type": "synth17x6", "num": 6, "params": {"max_steps": 5}},
                            "learner": {"params": {"gamma": 0.99, "lam": 0.9, "clip_eps": 0.1, "train_iters": 3}},
                            "policy_net": {"hidden": [12, 12]}, "loop": {"episodes": 2, "steps_per_episode": 8}}, 3),
    "a3c_gridline": ({"algorithm": "a3c", "actor": {"num": 4}, "env": {"type": "gridline", "num": 4},
                      "policy_net": {"hidden": [8, 8]}, "loop": {"episodes": 2, "steps_per_episode": 8}}, 9),
    "mappo_spread3": ({"algorithm": "mappo", "agent": {"num": 3}, "env": {"type": "spread_lite", "num": 4,
                                                                          "params": {"accel": 1}},
                       "policy_net": {"hidden": [8, 8]}, "loop": {"episodes": 2, "steps_per_episode": 6}}, 13),
}

# name -> (algo config, seed, dp-d replicas k)
RUN_CASES = {
    "dpd_k1_synth": (TRACE_CASES["ppo_synth7"][0] | {"loop": {"episodes": 3, "steps_per_episode": 8}}, 7, 1),
    "dpd_k2_synth": ({"algorithm": "ppo", "actor": {"num": 2}, "env": {"type": "synth17x6", "num": 10},
                      "policy_net": {"hidden": [16, 16]}, "loop": {"episodes": 3, "steps_per_episode": 8}}, 21, 2),
    "dpd_k3_gridline": ({"algorithm": "ppo", "actor": {"num": 3}, "env": {"type": "gridline", "num": 10},
                         "policy_net": {"hidden": [8, 8]}, "loop": {"episodes": 3, "steps_per_episode": 8}}, 4, 3),
    "dpd_a3c_k4": ({"algorithm": "a3c", "actor": {"num": 4}, "env": {"type": "gridline", "num": 4},
                    "policy_net": {"hidden": [8, 8]}, "loop": {"episodes": 3, "steps_per_episode": 8}}, 2, 4),
    # BASELINE configs[4] (C5) shape: A3C, 24 actors = 24 gridline envs, T=32 (small net)
    "dpd_a3c_k24": ({"algorithm": "a3c", "actor": {"num": 24}, "env": {"type": "gridline", "num": 24},
                     "policy_net": {"hidden": [16, 16]}, "loop": {"episodes": 3, "steps_per_episode": 32}}, 5, 24),
    # uneven replicas (20 envs over 6: 4,4,3,3,3,3) with per-replica advantage normalisation
    "dpd_k6_synth_uneven": ({"algorithm": "ppo", "actor": {"num": 6}, "env": {"type": "synth17x6", "num": 20},
                             "policy_net": {"hidden": [16, 16]}, "loop": {"episodes": 3, "steps_per_episode": 8}},
                            11, 6),
}


# (algo, deploy) pairs for the control-plane parity: DP-D plans and the errors the reference raises.
_G = {"algorithm": "ppo", "env": {"type": "gridline", "num": 10}}
PLAN_CASES = [
    (_G, {"distribution_policy": "dp-d"}),
    (_G | {"actor": {"num": 3}}, {"workers": ["a", "b"], "slots_per_worker": {"cpu": 2, "accel": 2},
                                  "distribution_policy": "GPU_only"}),
    (_G | {"actor": {"num": 4}}, {"workers": ["local"], "slots_per_worker": {"cpu": 1, "accel": 4},
                                  "distribution_policy": "dp-d"}),
    (_G | {"actor": {"num": 5}}, {"workers": ["w0", "w1"], "slots_per_worker": {"cpu": 1, "accel": 2},
                                  "distribution_policy": "dp-d"}),
    ({"algorithm": "ppo", "env": {"type": "cartpole_lite", "num": 4}}, {"distribution_policy": "dp-d"}),
    ({"algorithm": "ppo", "env": {"type": "nope", "num": 4}}, {"distribution_policy": "dp-d"}),
    ({"algorithm": "a3c", "actor": {"num": 2}, "env": {"type": "gridline", "num": 4}}, {"distribution_policy": "dp-d"}),
    ({"algorithm": "a3c", "actor": {"num": 4}, "env": {"type": "gridline", "num": 4}},
     {"slots_per_worker": {"cpu": 1, "accel": 4}, "distribution_policy": "dp-d"}),
    (_G | {"learner": {"params": {"gamma": 1.5}}}, {"distribution_policy": "dp-d"}),
    (_G | {"policy_net": {"hidden": []}}, {"distribution_policy": "dp-d"}),
    (_G, {"distribution_policy": "dp-z"}),
    (_G, {"workers": [], "distribution_policy": "dp-d"}),
    (_G | {"actor": {"num": 11}}, {"distribution_policy": "dp-d"}),
    ({"algorithm": "ppo", "env": {"type": "synth17x6", "num": 4096}, "actor": {"num": 8},
      "policy_net": {"hidden": [64, 64, 64, 64, 64, 64]}}, {"slots_per_worker": {"cpu": 8, "accel": 8},
                                                            "distribution_policy": "dp-d"}),
]


def build_ref():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)


def main():
    only = set(sys.argv[1:])
    build_ref()
    with tempfile.TemporaryDirectory() as tmp:
        plans = []
        for i, (algo, deploy) in enumerate(PLAN_CASES if not only else []):
            ap, dp = os.path.join(tmp, f"pa{i}.json"), os.path.join(tmp, f"pd{i}.json")
            json.dump(algo, open(ap, "w"))
            json.dump(deploy, open(dp, "w"))
            out = subprocess.run([pyoracle.REF_TOOL, "plan", ap, dp], check=True, capture_output=True,
                                 text=True).stdout
            plans.append({"algo": algo, "deploy": deploy, **json.loads(out)})
        if not only:
            json.dump(plans, open(os.path.join(HERE, "plans.json"), "w"), indent=1)
        print("plans", len(plans))
        for name, (algo, seed) in TRACE_CASES.items():
            if only and name not in only:
                continue
            ap = os.path.join(tmp, name + ".json")
            json.dump(algo, open(ap, "w"))
            prefix = os.path.join(tmp, name)
            subprocess.run([pyoracle.REF_TOOL, "trace", ap, str(seed), prefix], check=True)
            tr = pyoracle.load_trace(prefix)
            np.savez_compressed(os.path.join(HERE, f"trace_{name}.npz"),
                                __algo__=np.array(json.dumps(algo)), __seed__=np.array(seed),
                                **{k.replace("/", "__"): v for k, v in tr.items()})
            print("trace", name, len(tr), "tensors")
        for name, (algo, seed, k) in RUN_CASES.items():
            if only and name not in only:
                continue
            algo = dict(algo)
            algo["actor"] = {"num": k}
            ap = os.path.join(tmp, name + ".json")
            dp = os.path.join(tmp, name + "_deploy.json")
            json.dump(algo, open(ap, "w"))
            slots = max(16, k)
            json.dump({"workers": ["local"], "slots_per_worker": {"cpu": slots, "accel": slots},
                       "distribution_policy": "dp-d"}, open(dp, "w"))
            out = subprocess.run([pyoracle.REF_TOOL, "run", ap, dp, str(seed), "--params"], check=True,
                                 capture_output=True, text=True).stdout
            r = json.loads(out)
            np.savez_compressed(os.path.join(HERE, f"run_{name}.npz"),
                                __algo__=np.array(json.dumps(algo)), __seed__=np.array(seed), k=np.array(k),
                                rewards=np.array([e["reward"] for e in r["episodes"]]),
                                final_params=np.array(r["final_params"]), steps=np.array(r["steps"]),
                                grad_messages=np.array(r["grad_messages"]),
                                bytes_total=np.array([e["bytes_total"] for e in r["episodes"]]))
            print("run", name, r["units"], "units", r["steps"], "steps")


# dataflow-graph JSON (flw_program_dump(FLW_DUMP_DFG) = dfg::dump_json) of standard programs, with
# every algo field explicit: the seam's graph input (tests/test_capi_cpu.py test_algo_from_graph)
def _full(algorithm, agents, env, envs, params, hidden, act, hyper, loop):
    return {"algorithm": algorithm, "agent": {"num": agents}, "actor": {"num": 1},
            "env": {"type": env, "num": envs, **({"params": params} if params else {})},
            "learner": {"params": hyper}, "policy_net": {"hidden": hidden, "activation": act}, "loop": loop}


DFG_CASES = {
    "ppo_synth_c2": _full("ppo", 1, "synth17x6", 4096, None, [64] * 6, "tanh",
                          {"gamma": 0.97, "lam": 0.95, "clip_eps": 0.2, "lr": 3e-3, "train_iters": 4,
                           "value_coef": 0.5, "entropy_coef": 0.01, "normalize_adv": True},
                          {"episodes": 10, "steps_per_episode": 32}),
    "ppo_gridline_relu": _full("ppo", 1, "gridline", 40, {"length": 12.0}, [32, 16], "relu",
                               {"gamma": 0.9, "lam": 0.8, "clip_eps": 0.3, "lr": 5e-3, "train_iters": 2,
                                "value_coef": 0.25, "entropy_coef": 0.0, "normalize_adv": False},
                               {"episodes": 3, "steps_per_episode": 16}),
    "mappo_spread3": _full("mappo", 3, "spread_lite", 16, None, [32, 32], "tanh",
                           {"gamma": 0.99, "lam": 0.9, "clip_eps": 0.1, "lr": 1e-3, "train_iters": 3,
                            "value_coef": 1.0, "entropy_coef": 0.02, "normalize_adv": True},
                           {"episodes": 2, "steps_per_episode": 8}),
}


def make_dfg():
    out = {}
    with tempfile.TemporaryDirectory() as tmp:
        for name, algo in DFG_CASES.items():
            ap = os.path.join(tmp, name + ".json")
            json.dump(algo, open(ap, "w"))
            g = subprocess.run([pyoracle.REF_TOOL, "dfg", ap], check=True, capture_output=True, text=True).stdout
            out[name] = {"algo": algo, "graph": json.loads(g)}
    json.dump(out, open(os.path.join(HERE, "dfg.json"), "w"))
    print("dfg", len(out))


if __name__ == "__main__":
    if sys.argv[1:] == ["dfg"]:
        build_ref()
        make_dfg()
    else:
        main()
