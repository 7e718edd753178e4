"""Fast numerics for MLPs wider than the fused kernel's 64 columns: the layer-wise tcgen05 GEMM
learn path (kernels_tgemm.cu + kernels_wide.cu), SURVEY §8 "use H=64 and also report H=256".

Checked against the exact CUDA path (bit-exact with the reference interpreter) on identical
params and trajectory: one teacher-forced train iteration (PPO loss rl.cpp:137-172, backward
interp.cpp:392-499), at H=256 on the C2 shape (4096 synth17x6 envs, 7 layers, T=32) and at
H=128 / A3C on smaller shapes; plus determinism of whole episodes.

Bounds (bf16 operands and activations, f32 accumulation; ~3x the errors measured on the B200,
profiles/r02_wide_errors.txt):
"""
import numpy as np
import pytest

import bench

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

VALUES_REL_RMS = 3e-2
GRAD_REL_L2 = 3e-2
GRAD_COS = 0.9995
LOSS_REL = 1e-4


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _rel_rms(got, want):
    return float(np.sqrt(np.mean((got - want) ** 2)) / max(np.sqrt(np.mean(want ** 2)), 1e-30))


def _algo(envs, hidden, algorithm="ppo"):
    a = bench.algo_config(envs)
    a["policy_net"]["hidden"] = [hidden] * 6
    a["algorithm"] = algorithm
    if algorithm == "a3c":  # a3c pairs one env per actor (the reference's config rule)
        a["actor"]["num"] = envs
    return a


@pytest.mark.parametrize("envs,hidden,algorithm", [(4096, 256, "ppo"), (512, 128, "ppo"), (256, 256, "a3c")],
                         ids=["c2_h256", "h128", "a3c_h256"])
def test_wide_learn_teacher_forced(envs, hidden, algorithm):
    _need_gpu()
    from paper_2210_00882_b200 import DpdEngine

    algo = _algo(envs, hidden, algorithm)
    ex = DpdEngine(algo, seed=17, numerics="exact")
    fa = DpdEngine(algo, seed=17, numerics="fast")
    np.testing.assert_array_equal(ex.params(), fa.params())
    ex.reset(0)
    for st in range(32):
        ex.step(0, st)
    fa.set("sample", ex.get("sample"))
    ex.learn_grads(0, 0)
    fa.learn_grads(0, 0)
    v = _rel_rms(fa.get("values"), ex.get("values"))
    g_e, g_f = ex.get("grads"), fa.get("grads")
    cos = float(g_e @ g_f / (np.linalg.norm(g_e) * np.linalg.norm(g_f)))
    rel = float(np.linalg.norm(g_f - g_e) / np.linalg.norm(g_e))
    l_e, l_f = ex.get("loss")[0], fa.get("loss")[0]
    lrel = abs(l_f - l_e) / max(abs(l_e), 1e-3)
    print(f"wide {envs}x{hidden} {algorithm}: values {v:.2e} grads cos {cos:.6f} rel {rel:.2e} loss rel {lrel:.2e}")
    assert v <= VALUES_REL_RMS
    assert cos >= GRAD_COS and rel <= GRAD_REL_L2
    assert lrel <= LOSS_REL


def test_wide_episodes_deterministic_and_learn():
    """Whole fast episodes at H=256 (exact rollout + layer-wise learn in one CUDA graph): two
    engines stay bit-identical, equal a phase-by-phase run, and the params move."""
    _need_gpu()
    from paper_2210_00882_b200 import DpdEngine

    algo = _algo(512, 256)
    a = DpdEngine(algo, seed=3, numerics="fast")
    b = DpdEngine(algo, seed=3, numerics="fast")
    c = DpdEngine(algo, seed=3, numerics="fast")
    p0 = a.params()
    for ep in range(2):
        ra, _ = a.run_episode(ep)
        rb, _ = b.run_episode(ep)
        c.reset(ep)
        for st in range(32):
            c.step(ep, st)
        for k in range(4):
            c.learn(ep, k)
        assert ra == rb
    np.testing.assert_array_equal(a.params(), b.params())
    np.testing.assert_array_equal(a.params(), c.params())
    assert np.abs(a.params() - p0).max() > 1e-4


def test_wide_rollout_teacher_forced():
    """The wide policy's rollout (f32-accurate split-f16 GEMMs, K = hi | lo | hi) against the
    exact one at H=256 on the C2 shape, the exact engine's state fed in before every step:
    logp within 1e-5 relative where the sampled action agrees, flips <= 1e-3, env outputs equal."""
    _need_gpu()
    from paper_2210_00882_b200 import DpdEngine

    algo = _algo(4096, 256)
    ex = DpdEngine(algo, seed=5, numerics="exact")
    fa = DpdEngine(algo, seed=5, numerics="fast")
    ex.reset(0)
    fa.reset(0)
    flips = total = 0
    worst = 0.0
    for st in range(32):
        fa.set("state_in", ex.get("state_in"))
        fa.set("env_full", ex.get("env_full"))
        ex.step(0, st)
        fa.step(0, st)
        pe, pf = ex.get("pa").reshape(-1, 2), fa.get("pa").reshape(-1, 2)
        same = pe[:, 0] == pf[:, 0]
        flips += int((~same).sum())
        total += same.size
        rel = np.abs(pf[same, 1] - pe[same, 1]) / np.maximum(np.abs(pe[same, 1]), 1e-6)
        worst = max(worst, float(rel.max()))
        ee, ef = ex.get("envstep").reshape(pe.shape[0], -1), fa.get("envstep").reshape(pe.shape[0], -1)
        np.testing.assert_array_equal(ef[same], ee[same])
    print(f"wide rollout H=256: flips {flips}/{total}, worst logp rel {worst:.2e}")
    assert worst <= 1e-5
    assert flips <= 1e-3 * total
