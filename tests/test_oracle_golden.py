"""Pins the C restatement (oracle/fraglow_oracle.c) to the reference itself: every tensor of
every golden trace (tests/golden/make_golden.py, produced by the unmodified reference) must be
reproduced BIT-EXACTLY, and the dp-d plan runs (k replicas, GradSync ordered mean) too."""
import glob
import json
import os

import numpy as np
import pytest

from oracle import pyoracle

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TRACES = sorted(glob.glob(os.path.join(GOLDEN, "trace_*.npz")))
RUNS = sorted(glob.glob(os.path.join(GOLDEN, "run_*.npz")))


def _load(path):
    z = np.load(path)
    d = {k.replace("__", "/"): z[k] for k in z.files if not k.startswith("__")}
    return json.loads(str(z["__algo__"])), int(z["__seed__"]), d


def _eq(name, got, want):
    got = np.asarray(got, dtype=np.float64).ravel()
    want = np.asarray(want, dtype=np.float64).ravel()
    assert got.shape == want.shape, f"{name}: shape {got.shape} vs {want.shape}"
    bad = np.flatnonzero(got != want)
    assert bad.size == 0, f"{name}: {bad.size} mismatches, first at {bad[0]}: {got[bad[0]]!r} vs {want[bad[0]]!r}"


@pytest.mark.parametrize("path", TRACES, ids=[os.path.basename(p)[6:-4] for p in TRACES])
def test_trace_bit_exact(path):
    algo, seed, tr = _load(path)
    a = pyoracle.parse_algo(algo)
    u = pyoracle.Unit(algo, seed)
    _eq("params0", u.params(), tr["params0"])
    ep = 0
    while f"ep{ep}/reset_obs" in tr:
        u.reset(ep)
        _eq(f"ep{ep}/reset_obs", u.get("reset_obs"), tr[f"ep{ep}/reset_obs"])
        for st in range(a["steps_per_episode"]):
            p = f"ep{ep}/st{st}/"
            _eq(p + "state_in", u.get("state_in"), tr[p + "state_in"])
            u.step(ep, st)
            for n in ("logits", "pa", "envstep"):
                _eq(p + n, u.get(n), tr[p + n])
        _eq(f"ep{ep}/reward_sum", u.reward_sum, tr[f"ep{ep}/reward_sum"])
        _eq(f"ep{ep}/steps", u.steps, tr[f"ep{ep}/steps"])
        for k in range(u.learn_iters):
            p = f"ep{ep}/it{k}/"
            u.learn(ep, k)
            if k == 0:
                _eq(f"ep{ep}/sample", u.get("sample"), tr[f"ep{ep}/sample"])
            names = ["values", "last_value", "ret", "logits_new", "loss", "grads"]
            if p + "adv" in tr:
                names.append("adv")
            for n in names:
                _eq(p + n, u.get(n), tr[p + n])
            _eq(p + "params", u.params(), tr[p + "params"])
        ep += 1
    assert ep >= 2


@pytest.mark.parametrize("path", RUNS, ids=[os.path.basename(p)[4:-4] for p in RUNS])
def test_dpd_plan_run_bit_exact(path):
    z = np.load(path)
    algo = json.loads(str(z["__algo__"]))
    rew, par, steps = pyoracle.run(algo, int(z["__seed__"]), int(z["k"]))
    _eq("rewards", rew, z["rewards"])
    _eq("final_params", par, z["final_params"])
    assert steps == int(z["steps"])
