"""MAPPO on spread_lite (exact numerics) against the unmodified reference's trace
(tests/golden/trace_mappo_spread3.npz): agent-major policy rows, joint-observation critic with
agent one-hot, per-agent rewards, GAE over n*E streams (programs.cpp:349-454)."""
import json
import os

import numpy as np
import pytest

from oracle import pyoracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _close(name, got, want, exact=False):
    got, want = np.asarray(got, float).ravel(), np.asarray(want, float).ravel()
    assert got.shape == want.shape, name
    diff = got != want
    if not diff.any():
        return
    assert not exact, f"{name}: {diff.sum()} integer mismatches"
    rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-30)
    assert rel[diff].max() <= 2.5e-7 and diff.mean() <= 1e-3, f"{name}: {diff.sum()} differ, max rel {rel.max():.3g}"


def test_mappo_matches_reference_trace():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2210_00882_b200 import DpdEngine

    z = np.load(os.path.join(GOLDEN, "trace_mappo_spread3.npz"))
    tr = {k.replace("__", "/"): z[k] for k in z.files if not k.startswith("__")}
    algo, seed = json.loads(str(z["__algo__"])), int(z["__seed__"])
    a = pyoracle.parse_algo(algo)
    eng = DpdEngine(algo, seed=seed, numerics="exact")
    _close("params0", eng.params(), tr["params0"])
    for ep in range(2):
        eng.reset(ep)
        _close("reset_obs", eng.get("reset_obs"), tr[f"ep{ep}/reset_obs"])
        for st in range(a["steps_per_episode"]):
            p = f"ep{ep}/st{st}/"
            _close(p + "state_in", eng.get("state_in"), tr[p + "state_in"])
            eng.step(ep, st)
            _close(p + "logits", eng.get("logits"), tr[p + "logits"])
            pa, want = eng.get("pa").reshape(-1, 2), tr[p + "pa"].reshape(-1, 2)
            _close(p + "action", pa[:, 0], want[:, 0], exact=True)
            _close(p + "logp", pa[:, 1], want[:, 1])
            _close(p + "envstep", eng.get("envstep"), tr[p + "envstep"])
        for k in range(eng.stats()["learn_iters"]):
            p = f"ep{ep}/it{k}/"
            eng.learn(ep, k)
            if k == 0:
                _close(f"ep{ep}/sample", eng.get("sample"), tr[f"ep{ep}/sample"])
            for n in ("values", "last_value", "adv", "ret", "logits_new", "loss", "grads"):
                _close(p + n, eng.get(n), tr[p + n])
            _close(p + "params", eng.params(), tr[p + "params"])


@pytest.mark.parametrize("n_agents", [2, 4, 6, 9])  # n > 4: the block-per-env step kernel
def test_mappo_episodes_match_oracle(n_agents):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2210_00882_b200 import DpdEngine

    algo = {"algorithm": "mappo", "agent": {"num": n_agents},
            "env": {"type": "spread_lite", "num": 16, "params": {"accel": 1, "max_steps": 10}},
            "policy_net": {"hidden": [16, 16]}, "loop": {"episodes": 3, "steps_per_episode": 12}}
    rew, par, _ = pyoracle.run(algo, 3, 1)
    eng = DpdEngine(algo, seed=3, numerics="exact")
    got = [eng.run_episode(ep)[0] / 16 for ep in range(3)]
    _close("rewards", got, rew)
    _close("params", eng.params(), par)


@pytest.mark.parametrize("n_agents", [3, 4])
def test_fast_mappo_tracks_exact(n_agents):
    """Fast numerics for MAPPO (n <= 4, critic input 2n^2+3n <= 64): the fused tensor-core
    rollout (test_fast_mappo_rollout_matches_exact) + the tensor-core learn kernels over
    [joint | one-hot] rows keep the episode rewards and trained parameters close to the exact
    run."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2210_00882_b200 import DpdEngine

    algo = {"algorithm": "mappo", "agent": {"num": n_agents},
            "env": {"type": "spread_lite", "num": 256, "params": {"accel": 1}},
            "policy_net": {"hidden": [64, 64]}, "loop": {"episodes": 4, "steps_per_episode": 16}}
    ex = DpdEngine(algo, seed=5, numerics="exact")
    fa = DpdEngine(algo, seed=5, numerics="fast")
    r_ex = [ex.run_episode(ep)[0] for ep in range(4)]
    r_fa = [fa.run_episode(ep)[0] for ep in range(4)]
    # first episode: same parameters, rollouts differ only by near-tie action draws
    assert r_fa[0] == pytest.approx(r_ex[0], rel=2e-2)
    np.testing.assert_allclose(r_fa, r_ex, rtol=5e-2)
    p_ex, p_fa = np.asarray(ex.params()), np.asarray(fa.params())
    rel = np.linalg.norm(p_fa - p_ex) / np.linalg.norm(p_ex)
    assert rel < 2e-2, rel


@pytest.mark.parametrize("n_agents", [6, 10])
def test_fast_mappo_compact_critic_tracks_exact(n_agents):
    """n > 4: the critic input [joint | one-hot] (2n^2+3n) is wider than the fused kernel, so
    its layer 0 runs compact - a tcgen05 joint GEMM once per env (kernels_tgemm.cu) plus W[J+a] -
    and its gradients come from the fused kernel's input-gradient stage (dW_J = joint^T . sum_a
    dZ0 as a split-K tcgen05 GEMM, one-hot rows, bias). Same checks as the direct path."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2210_00882_b200 import DpdEngine

    algo = {"algorithm": "mappo", "agent": {"num": n_agents},
            "env": {"type": "spread_lite", "num": 128, "params": {"accel": 1}},
            "policy_net": {"hidden": [64, 64]}, "loop": {"episodes": 4, "steps_per_episode": 16}}
    ex = DpdEngine(algo, seed=5, numerics="exact")
    fa = DpdEngine(algo, seed=5, numerics="fast")
    r_ex = [ex.run_episode(ep)[0] for ep in range(4)]
    r_fa = [fa.run_episode(ep)[0] for ep in range(4)]
    assert r_fa[0] == pytest.approx(r_ex[0], rel=2e-2)
    np.testing.assert_allclose(r_fa, r_ex, rtol=5e-2)
    p_ex, p_fa = np.asarray(ex.params()), np.asarray(fa.params())
    rel = np.linalg.norm(p_fa - p_ex) / np.linalg.norm(p_ex)
    assert rel < 2e-2, rel


@pytest.mark.parametrize("n_agents", [3, 10, 24, 40])
def test_fast_mappo_rollout_matches_exact(n_agents):
    """The fused fast MAPPO rollout (n <= 16; n = 24, 40: the policy forward as f32-accurate
    split-f16 tcgen05 GEMMs) (3-term F16 tensor-core MLP over the agent rows, f32 softmax,
    the reference's draws, exact spread_lite dynamics in double) against the exact per-step
    rollout from the same reset: step 0's actions agree except near-tie draws and their logp to
    1e-5; over the episode the draws agree for >= 98% of the agent rows (a flip changes that
    env's later trajectory)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2210_00882_b200 import DpdEngine

    T = 16
    algo = {"algorithm": "mappo", "agent": {"num": n_agents},
            "env": {"type": "spread_lite", "num": 96, "params": {"accel": 1}},
            "policy_net": {"hidden": [64] * 6}, "loop": {"episodes": 1, "steps_per_episode": T}}
    ex = DpdEngine(algo, seed=11, numerics="exact")
    fa = DpdEngine(algo, seed=11, numerics="fast")
    ex.reset(0)
    fa.reset(0)
    np.testing.assert_array_equal(fa.get("state_in"), ex.get("state_in"))
    same_all = total = 0
    for st in range(T):
        ex.step(0, st)
        fa.step(0, st)
        pe, pf = ex.get("pa").reshape(-1, 2), fa.get("pa").reshape(-1, 2)
        same = pe[:, 0] == pf[:, 0]
        if st == 0:
            assert same.mean() >= 0.99, same.mean()
            np.testing.assert_allclose(pf[same, 1], pe[same, 1], rtol=1e-5, atol=1e-6)
        same_all += int(same.sum())
        total += same.size
    assert same_all >= 0.98 * total, (same_all, total)


@pytest.mark.parametrize("n_agents", [32, 64])
def test_fast_mappo_wide_tracks_exact(n_agents):
    """n = 32, 64 (C3's upper end; joint observation 2112 / 8320 wide, per-agent observation
    66 / 130 > the fused kernel's 64): split-GEMM rollout, layer-wise policy learn, compact
    critic on tcgen05 GEMMs, against the exact (reference-arithmetic) engine.
      1. episode 0's rollout (same initial params): sampled actions identical but for near-ties;
      2. the first train iteration on that (identical) trajectory: gradient cosine / rel-L2;
      3. three free-running episodes: rewards within 5%, params within 5% (Adam's sign-like
         steps amplify tiny gradient differences along the trajectory)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2210_00882_b200 import DpdEngine

    algo = {"algorithm": "mappo", "agent": {"num": n_agents},
            "env": {"type": "spread_lite", "num": 32, "params": {"accel": 1}},
            "policy_net": {"hidden": [64] * 6}, "loop": {"episodes": 3, "steps_per_episode": 16}}
    ex = DpdEngine(algo, seed=5, numerics="exact")
    fa = DpdEngine(algo, seed=5, numerics="fast")
    ex.reset(0)
    fa.reset(0)
    same = total = 0
    for st in range(16):
        ex.step(0, st)
        fa.step(0, st)
        pe, pf = ex.get("pa").reshape(-1, 2), fa.get("pa").reshape(-1, 2)
        same += int((pe[:, 0] == pf[:, 0]).sum())
        total += pe.shape[0]
    assert same >= 0.999 * total, (same, total)
    ex.learn_grads(0, 0)
    fa.learn_grads(0, 0)
    g_e, g_f = ex.get("grads"), fa.get("grads")
    cos = float(g_e @ g_f / (np.linalg.norm(g_e) * np.linalg.norm(g_f)))
    rel = float(np.linalg.norm(g_f - g_e) / np.linalg.norm(g_e))
    print(f"n={n_agents}: actions same {same}/{total}, grads cos {cos:.6f} rel {rel:.2e}")
    if same == total:
        assert cos >= 0.9999 and rel <= 2e-2, (cos, rel)
    ex = DpdEngine(algo, seed=5, numerics="exact")
    fa = DpdEngine(algo, seed=5, numerics="fast")
    r_ex = [ex.run_episode(ep)[0] for ep in range(3)]
    r_fa = [fa.run_episode(ep)[0] for ep in range(3)]
    assert r_fa[0] == pytest.approx(r_ex[0], rel=2e-2)
    np.testing.assert_allclose(r_fa, r_ex, rtol=5e-2)
    p_ex, p_fa = np.asarray(ex.params()), np.asarray(fa.params())
    prel = np.linalg.norm(p_fa - p_ex) / np.linalg.norm(p_ex)
    print(f"n={n_agents}: rewards {r_ex} vs {r_fa}, params rel {prel:.3g}")
    assert prel < 5e-2, prel
