"""GPU parity of the B200 engine (exact numerics) against the reference and the oracle.

Exact numerics reproduce the reference's per-op f32 rounding with FP64 accumulation in the same
order, so results are expected to be bit-identical; the only admitted deviation is libm vs CUDA
transcendentals (exp/log/tanh) landing on a different side of an f32 rounding boundary, which
we bound explicitly: at most MAX_ULP_FRACTION of elements may differ, each by <= 2 f32 ulps
relative (2.4e-7), and integer/index data (actions, dones, counters) must match exactly.
"""
import glob
import json
import os

import numpy as np
import pytest

from oracle import pyoracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
MAX_ULP_FRACTION = 1e-3
REL_TOL = 2.5e-7


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def close(name, got, want, exact=False):
    got = np.asarray(got, dtype=np.float64).ravel()
    want = np.asarray(want, dtype=np.float64).ravel()
    assert got.shape == want.shape, f"{name}: shape {got.shape} vs {want.shape}"
    diff = got != want
    if not diff.any():
        return 0
    assert not exact, f"{name}: {diff.sum()} mismatches in integer/index data"
    rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-30)
    assert rel[diff].max() <= REL_TOL or np.abs(got - want)[diff].max() < 1e-12, \
        f"{name}: max rel err {rel[diff].max():.3g} ({diff.sum()} of {diff.size} differ)"
    assert diff.mean() <= MAX_ULP_FRACTION, f"{name}: {diff.sum()} of {diff.size} elements differ"
    return int(diff.sum())


def _load_trace(path):
    z = np.load(path)
    d = {k.replace("__", "/"): z[k] for k in z.files if not k.startswith("__")}
    return json.loads(str(z["__algo__"])), int(z["__seed__"]), d


TRACES = [p for p in sorted(glob.glob(os.path.join(GOLDEN, "trace_*.npz"))) if "mappo" not in p]


@pytest.mark.parametrize("path", TRACES, ids=[os.path.basename(p)[6:-4] for p in TRACES])
def test_engine_matches_reference_trace(path):
    """Phase by phase against the UNMODIFIED reference's own trace (tests/golden)."""
    _need_gpu()
    from paper_2210_00882_b200 import DpdEngine

    algo, seed, tr = _load_trace(path)
    a = pyoracle.parse_algo(algo)
    eng = DpdEngine(algo, device=0, seed=seed, numerics="exact")
    close("params0", eng.params(), tr["params0"])
    ep = 0
    while f"ep{ep}/reset_obs" in tr:
        eng.reset(ep)
        close("reset_obs", eng.get("reset_obs"), tr[f"ep{ep}/reset_obs"])
        for st in range(a["steps_per_episode"]):
            p = f"ep{ep}/st{st}/"
            close(p + "state_in", eng.get("state_in"), tr[p + "state_in"])
            eng.step(ep, st)
            close(p + "logits", eng.get("logits"), tr[p + "logits"])
            pa, want = eng.get("pa").reshape(-1, 2), tr[p + "pa"].reshape(-1, 2)
            close(p + "action", pa[:, 0], want[:, 0], exact=True)
            close(p + "logp", pa[:, 1], want[:, 1])
            es, wes = eng.get("envstep").reshape(want.shape[0], -1), tr[p + "envstep"].reshape(want.shape[0], -1)
            close(p + "envstep.obs", es[:, :-1], wes[:, :-1])
            close(p + "envstep.done", es[:, -1], wes[:, -1], exact=True)
        assert eng.stats()["steps"] == int(tr[f"ep{ep}/steps"][0])
        for k in range(eng.stats()["learn_iters"]):
            p = f"ep{ep}/it{k}/"
            eng.learn(ep, k)
            if k == 0:
                close(f"ep{ep}/sample", eng.get("sample"), tr[f"ep{ep}/sample"])
            for n in ("values", "last_value", "ret", "logits_new", "loss", "grads"):
                close(p + n, eng.get(n), tr[p + n])
            if p + "adv" in tr:
                close(p + "adv", eng.get("adv"), tr[p + "adv"])
            close(p + "params", eng.params(), tr[p + "params"])
        ep += 1
    assert ep >= 2


CASES = {
    "ppo_synth_h64": {"algorithm": "ppo", "env": {"type": "synth17x6", "num": 64},
                      "policy_net": {"hidden": [64] * 6}, "loop": {"episodes": 3, "steps_per_episode": 16}},
    "ppo_gridline16": {"algorithm": "ppo", "env": {"type": "gridline", "num": 40, "params": {"length": 16}},
                       "learner": {"params": {"lr": 0.005}},
                       "policy_net": {"hidden": [32, 32]}, "loop": {"episodes": 4, "steps_per_episode": 32}},
    "a3c_synth": {"algorithm": "a3c", "actor": {"num": 8}, "env": {"type": "synth17x6", "num": 8},
                  "policy_net": {"hidden": [16, 16]}, "loop": {"episodes": 3, "steps_per_episode": 12}},
}


@pytest.mark.parametrize("name", list(CASES))
def test_episode_graph_matches_oracle(name):
    """Whole episodes as the captured CUDA graph vs the pinned C oracle (DP-D k=1)."""
    _need_gpu()
    from paper_2210_00882_b200 import DpdEngine

    algo = CASES[name]
    seed = 17
    rew, par, steps = pyoracle.run(algo, seed, 1)
    eng = DpdEngine(algo, device=0, seed=seed, numerics="exact")
    n_env = algo["env"]["num"]
    got = []
    for ep in range(algo["loop"]["episodes"]):
        r, ms = eng.run_episode(ep)
        assert ms > 0
        got.append(r / n_env)
    close("episode_rewards", got, rew)
    close("final_params", eng.params(), par)
    assert eng.stats()["steps"] == steps
    assert eng.stats()["graph_kernels"] > 0


def test_phase_api_equals_graph():
    """Phase-level driving and the episode graph are the same computation."""
    _need_gpu()
    from paper_2210_00882_b200 import DpdEngine

    algo = CASES["ppo_synth_h64"]
    a = DpdEngine(algo, seed=3)
    b = DpdEngine(algo, seed=3)
    for ep in range(2):
        ra, _ = a.run_episode(ep)
        b.reset(ep)
        for st in range(algo["loop"]["steps_per_episode"]):
            b.step(ep, st)
        for k in range(b.stats()["learn_iters"]):
            b.learn(ep, k)
        np.testing.assert_array_equal(a.params(), b.params())


@pytest.mark.parametrize("numerics", ["exact", "fast"])
def test_pipelined_episodes_equal_synchronous(numerics):
    """launch_episode / finish_episode (two episodes in flight) are the same computation as
    run_episode: identical rewards per episode and identical final params."""
    _need_gpu()
    from paper_2210_00882_b200 import DpdEngine

    algo = CASES["ppo_synth_h64"]
    a = DpdEngine(algo, seed=5, numerics=numerics)
    b = DpdEngine(algo, seed=5, numerics=numerics)
    ra = [a.run_episode(ep)[0] for ep in range(4)]
    b.launch_episode(0)
    rb = []
    for ep in range(4):
        if ep + 1 < 4:
            b.launch_episode(ep + 1)
        rb.append(b.finish_episode())
    assert ra == rb
    np.testing.assert_array_equal(a.params(), b.params())
    with pytest.raises(Exception):
        b.finish_episode()  # nothing in flight


@pytest.mark.parametrize("numerics", ["exact", "fast"])
def test_pipelined_episode_indices_and_reinit(numerics):
    """The pipelined gate keeps the device episode counter when launches are consecutive and
    copies the index otherwise (a jump, or after run_episode / reinit); the graph publishes the
    reward sums into a host-mapped ring slot per graph run. Any index sequence, mixed with
    run_episode and reinit, gives run_episode's rewards and params."""
    _need_gpu()
    from paper_2210_00882_b200 import DpdEngine

    algo = CASES["ppo_synth_h64"]
    seq = [0, 1, 5, 6, 2]
    a = DpdEngine(algo, seed=9, numerics=numerics)
    ra = [a.run_episode(ep)[0] for ep in seq]
    b = DpdEngine(algo, seed=3, numerics=numerics)
    b.launch_episode(4)  # a different run first: reinit must forget its counter and params
    b.finish_episode()
    b.reinit(9)
    rb = [b.run_episode(seq[0])[0]]  # synchronous first (a graph run: the ring slot advances)
    b.launch_episode(seq[1])
    for i in range(1, len(seq)):
        if i + 1 < len(seq):
            b.launch_episode(seq[i + 1])
        rb.append(b.finish_episode())
    assert ra == rb
    np.testing.assert_array_equal(a.params(), b.params())


def test_run_local_summary_schema():
    _need_gpu()
    from paper_2210_00882_b200 import Program

    algo = dict(CASES["ppo_gridline16"])
    prog = Program(algo, {"workers": ["local"], "slots_per_worker": {"cpu": 4, "accel": 1},
                          "distribution_policy": "dp-d", "numerics": "exact"})
    csv, s = prog.run_local(seed=17, episodes=3, reward_threshold=0.5)
    lines = csv.strip().split("\n")
    assert lines[0] == "episode,wall_ms,reward,bytes_total" and len(lines) == 4
    for key in ("episodes", "steps", "grad_messages", "final_reward", "total_wall_ms", "bytes_total",
                "bytes_per_channel", "param_count", "param_checksum", "param_l2", "reward_threshold",
                "time_to_threshold_ms", "device_exchange"):
        assert key in s
    assert s["device_exchange"] == {"kind": "none", "bytes_per_episode": 0, "bytes_total": 0}  # one unit
    rew, par, _ = pyoracle.run(algo, 17, 1, episodes=3)
    close("final_reward", s["final_reward"], rew[-1])
    assert s["param_count"] == par.size
    assert abs(s["param_checksum"] - par.sum()) <= 1e-6 * max(1.0, np.abs(par).sum())
    # a second run on the same program reuses the engine and re-initialises it
    _, s2 = prog.run_local(seed=17, episodes=3, reward_threshold=0.5)
    assert s2["param_checksum"] == s["param_checksum"]


def test_learning_gridline_reaches_goal():
    """Behavioural check from the reference acceptance suite (acceptance_main.cpp:389-414):
    PPO on gridline reaches mean reward 0.9 within the 40-episode budget."""
    _need_gpu()
    from paper_2210_00882_b200 import Program

    algo = {
        "algorithm": "ppo", "actor": {"num": 1}, "env": {"type": "gridline", "num": 8, "params": {"length": 16}},
        "learner": {"params": {"gamma": 0.99, "lam": 0.95, "clip_eps": 0.2, "lr": 0.005, "train_iters": 4,
                               "value_coef": 0.5, "entropy_coef": 0.01, "normalize_adv": True}},
        "policy_net": {"hidden": [16, 16], "activation": "tanh"}, "loop": {"episodes": 40, "steps_per_episode": 32}}
    prog = Program(algo, {"distribution_policy": "dp-d", "slots_per_worker": {"cpu": 1, "accel": 1},
                          "numerics": "exact"})
    csv, s = prog.run_local(seed=1, reward_threshold=0.9)
    assert s["time_to_threshold_ms"] >= 0, csv


def test_degenerate_advantages_skip_normalisation():
    """normalize_advantages' `std < 1e-8` branch (rl.cpp:104): T = 1 step, no env reaches the
    goal (rewards 0), the critic outputs the constant 0.5 (zero weights, last bias 0.5), so every
    advantage is (gamma - 1) * 0.5 and their std is 0 -> left unnormalised (normalising would
    give 0). The exact engine matches the oracle bit-for-bit (grads, loss, adv); the fast engine
    keeps the unnormalised advantages too."""
    _need_gpu()
    from paper_2210_00882_b200 import DpdEngine

    algo = {"algorithm": "ppo", "env": {"type": "gridline", "num": 32, "params": {"length": 16}},
            "learner": {"params": {"gamma": 0.9}}, "policy_net": {"hidden": [16, 16]},
            "loop": {"episodes": 1, "steps_per_episode": 1}}
    ex = DpdEngine(algo, seed=4, numerics="exact")
    u = pyoracle.Unit(algo, 4)
    p = u.params()
    dims_c = [1, 16, 16, 1]
    pc = sum(i * o + o for i, o in zip(dims_c[:-1], dims_c[1:]))
    p[-pc:] = 0.0
    p[-1] = 0.5  # critic output bias
    ex.set_params(p)
    u.set_params(p)
    fa = DpdEngine(algo, seed=4, numerics="fast")
    fa.set_params(p)
    for e in (ex, fa):
        e.reset(0)
        e.step(0, 0)
    u.reset(0)
    u.step(0, 0)
    g_o = u.learn_grads(0, 0)
    ex.learn_grads(0, 0)
    fa.learn_grads(0, 0)
    want_adv = (0.9 - 1.0) * 0.5
    np.testing.assert_allclose(u.get("adv"), want_adv, rtol=1e-6)  # (f32-rounded terms)
    np.testing.assert_array_equal(ex.get("adv"), u.get("adv"))
    np.testing.assert_array_equal(ex.get("grads"), g_o)
    np.testing.assert_array_equal(ex.get("loss"), u.get("loss"))
    np.testing.assert_allclose(fa.get("adv"), want_adv, rtol=1e-6)


@pytest.mark.parametrize("case,numerics", [("ppo_gridline_relu", "exact"), ("ppo_gridline_relu", "fast"),
                                           ("ppo_synth_c2", "fast")])
def test_engine_from_graph_json_equals_algo_json(case, numerics):
    """flw_dpd_create given the reference's dataflow-graph JSON (the bundle a worker receives,
    SURVEY §8b) runs the same program as given the algo JSON: identical rewards and params."""
    _need_gpu()
    from paper_2210_00882_b200 import DpdEngine

    c = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "dfg.json")))[case]
    a = DpdEngine(c["algo"], seed=3, numerics=numerics)
    b = DpdEngine(c["graph"], seed=3, numerics=numerics)
    ra = [a.run_episode(ep)[0] for ep in range(2)]
    rb = [b.run_episode(ep)[0] for ep in range(2)]
    assert ra == rb
    np.testing.assert_array_equal(a.params(), b.params())
