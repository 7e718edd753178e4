"""ctypes view of oracle/liboracle.so -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import this module, and
only as the checker. The algo-config mapping mirrors the reference parser
(/root/reference/proj/src/config.cpp:24-63) and its defaults (rl.hpp:11-19, programs.hpp:9-22).
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_TOOL = os.path.join(HERE, "_ref", "ref_tool")

ALGOS = {"ppo": 0, "a3c": 1, "mappo": 2}
ENVS = {"gridline": 0, "synth17x6": 1, "spread_lite": 2}


class OrcCfg(C.Structure):
    _fields_ = [
        ("algo", C.c_int32), ("env", C.c_int32), ("n_agents", C.c_int32), ("activation", C.c_int32),
        ("n_hidden", C.c_int32), ("hidden", C.c_int32 * 8), ("normalize_adv", C.c_int32),
        ("steps_per_episode", C.c_int64), ("train_iters", C.c_int64), ("max_steps", C.c_int64),
        ("env_length", C.c_double), ("gamma", C.c_double), ("lam", C.c_double), ("clip_eps", C.c_double),
        ("lr", C.c_double), ("value_coef", C.c_double), ("entropy_coef", C.c_double),
    ]


def ensure_built() -> str:
    if not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(ensure_built())
        P = C.POINTER
        d, i64, u64 = C.c_double, C.c_int64, C.c_uint64
        L.orc_unit_new.restype = C.c_void_p
        L.orc_unit_new.argtypes = [P(OrcCfg), u64, i64, i64, i64]
        L.orc_unit_free.argtypes = [C.c_void_p]
        for f in ("orc_param_count", "orc_learn_iters", "orc_steps"):
            getattr(L, f).restype = i64
            getattr(L, f).argtypes = [C.c_void_p]
        L.orc_reward_sum.restype = d
        L.orc_reward_sum.argtypes = [C.c_void_p]
        L.orc_get_params.argtypes = [C.c_void_p, P(d)]
        L.orc_set_params.argtypes = [C.c_void_p, P(d)]
        L.orc_reset.argtypes = [C.c_void_p, i64]
        L.orc_step.argtypes = [C.c_void_p, i64, i64]
        L.orc_learn_grads.argtypes = [C.c_void_p, i64, i64, P(d)]
        L.orc_apply_grads.argtypes = [C.c_void_p, P(d)]
        L.orc_learn.argtypes = [C.c_void_p, i64, i64]
        L.orc_size.restype = i64
        L.orc_size.argtypes = [C.c_void_p, C.c_char_p]
        L.orc_get.argtypes = [C.c_void_p, C.c_char_p, P(d)]
        L.orc_set.argtypes = [C.c_void_p, C.c_char_p, P(d), i64]
        L.orc_run.argtypes = [P(OrcCfg), u64, i64, C.c_int32, i64, P(d), P(d), P(i64)]
        L.orc_key.restype = u64
        L.orc_key.argtypes = [u64, u64, u64, u64, u64]
        L.orc_uniform.restype = d
        L.orc_uniform.argtypes = [u64]
        L.orc_gae_streams.argtypes = [P(d), P(d), P(d), P(d), i64, i64, d, d, P(d)]
        L.orc_returns_streams.argtypes = [P(d), P(d), P(d), i64, i64, d, P(d)]
        L.orc_normalize.argtypes = [P(d), i64]
        L.orc_adam.argtypes = [P(d), P(d), P(d), P(d), i64, i64, d, d, d, d]
        L.orc_ppo_loss.restype = d
        L.orc_ppo_loss.argtypes = [P(d)] * 6 + [i64, i64, d, d, d, P(d), P(d)]
        _lib = L
    return _lib


def dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


def parse_algo(algo: dict | str) -> dict:
    """Reference parse_algo_config (config.cpp:24-63) + AlgoConfig defaults."""
    j = json.loads(algo) if isinstance(algo, str) else algo
    env = j.get("env", {})
    lp = j.get("learner", {}).get("params", {})
    pn = j.get("policy_net", {})
    loop = j.get("loop", {})
    return {
        "algorithm": j.get("algorithm", "ppo"),
        "agents": int(j.get("agent", {}).get("num", 1)),
        "actors": int(j.get("actor", {}).get("num", 1)),
        "env": env.get("type", "gridline"),
        "envs": int(env.get("num", 1)),
        "env_params": {k: float(v) for k, v in env.get("params", {}).items()},
        "gamma": float(lp.get("gamma", 0.97)), "lam": float(lp.get("lam", 0.95)),
        "clip_eps": float(lp.get("clip_eps", 0.2)), "lr": float(lp.get("lr", 3e-3)),
        "train_iters": int(lp.get("train_iters", 4)), "value_coef": float(lp.get("value_coef", 0.5)),
        "entropy_coef": float(lp.get("entropy_coef", 0.01)),
        "normalize_adv": bool(lp.get("normalize_adv", True)),
        "hidden": [int(h) for h in pn.get("hidden", [16, 16])],
        "activation": pn.get("activation", "tanh"),
        "episodes": int(loop.get("episodes", 1)), "steps_per_episode": int(loop.get("steps_per_episode", 32)),
    }


def make_cfg(algo: dict | str) -> OrcCfg:
    a = parse_algo(algo)
    c = OrcCfg()
    c.algo = ALGOS[a["algorithm"]]
    c.env = ENVS[a["env"]]
    c.n_agents = a["agents"] if a["algorithm"] == "mappo" else int(a["env_params"].get("n_agents", 2))
    c.activation = 0 if a["activation"] == "tanh" else 1
    c.n_hidden = len(a["hidden"])
    for k, h in enumerate(a["hidden"]):
        c.hidden[k] = h
    c.normalize_adv = int(a["normalize_adv"])
    c.steps_per_episode = a["steps_per_episode"]
    c.train_iters = a["train_iters"]
    c.max_steps = int(a["env_params"].get("max_steps", 0))
    c.env_length = a["env_params"].get("length", 8.0)
    for f in ("gamma", "lam", "clip_eps", "lr", "value_coef", "entropy_coef"):
        setattr(c, f, a[f])
    return c


class Unit:
    """One DP-D unit (the reference Interp over the fused fragment, interp.hpp:34-115)."""

    def __init__(self, algo, seed: int, env_lo: int = 0, env_hi: int | None = None, env_total: int | None = None):
        a = parse_algo(algo)
        self.cfg = make_cfg(algo)
        env_total = a["envs"] if env_total is None else env_total
        env_hi = env_total if env_hi is None else env_hi
        self.L = lib()
        self.h = self.L.orc_unit_new(C.byref(self.cfg), seed, env_lo, env_hi, env_total)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.orc_unit_free(self.h)
            self.h = None

    @property
    def param_count(self) -> int:
        return self.L.orc_param_count(self.h)

    @property
    def learn_iters(self) -> int:
        return self.L.orc_learn_iters(self.h)

    def params(self) -> np.ndarray:
        out = np.zeros(self.param_count)
        self.L.orc_get_params(self.h, dptr(out))
        return out

    def set_params(self, p):
        p = np.ascontiguousarray(p, dtype=np.float64)
        self.L.orc_set_params(self.h, dptr(p))

    def reset(self, ep: int):
        self.L.orc_reset(self.h, ep)

    def step(self, ep: int, st: int):
        self.L.orc_step(self.h, ep, st)

    def learn_grads(self, ep: int, k: int) -> np.ndarray:
        g = np.zeros(self.param_count)
        self.L.orc_learn_grads(self.h, ep, k, dptr(g))
        return g

    def apply_grads(self, g):
        g = np.ascontiguousarray(g, dtype=np.float64)
        self.L.orc_apply_grads(self.h, dptr(g))

    def learn(self, ep: int, k: int):
        self.L.orc_learn(self.h, ep, k)

    @property
    def reward_sum(self) -> float:
        return self.L.orc_reward_sum(self.h)

    @property
    def steps(self) -> int:
        return self.L.orc_steps(self.h)

    def get(self, name: str) -> np.ndarray:
        n = self.L.orc_size(self.h, name.encode())
        if n < 0:
            raise KeyError(name)
        out = np.zeros(n)
        self.L.orc_get(self.h, name.encode(), dptr(out))
        return out

    def set(self, name: str, values):
        v = np.ascontiguousarray(values, dtype=np.float64).ravel()
        if self.L.orc_set(self.h, name.encode(), dptr(v), v.size) != 0:
            raise ValueError(f"cannot set {name} with {v.size} values")


def run(algo, seed: int, k: int = 1, episodes: int | None = None):
    """DP-D with k replicas (≡ DP-C k): (episode rewards, final params, steps)."""
    a = parse_algo(algo)
    eps = a["episodes"] if episodes is None else episodes
    cfg = make_cfg(algo)
    u = Unit(algo, seed)
    P = u.param_count
    del u
    rew = np.zeros(max(eps, 1))
    par = np.zeros(P)
    steps = C.c_int64(0)
    rc = lib().orc_run(C.byref(cfg), seed, a["envs"], k, eps, dptr(rew), dptr(par), C.byref(steps))
    if rc != 0:
        raise RuntimeError("orc_run failed")
    return rew[:eps], par, steps.value


def load_trace(prefix: str) -> dict:
    """Reads a ref_tool trace (<prefix>.json manifest + <prefix>.bin float64)."""
    man = json.load(open(prefix + ".json"))
    blob = np.fromfile(prefix + ".bin", dtype="<f8")
    return {m["name"]: blob[m["offset"]: m["offset"] + m["count"]].reshape(m["shape"]) for m in man}
