"""The fused peer-memory gradient exchange (kernels_p2p.cu: k_reduce_push + k_sum_adam) on ONE
GPU: two unit processes on cuda:0 map each other's exchange region through CUDA IPC exactly as
one-process-per-GPU runs do (same-device IPC across processes; the GPU time-slices the two
contexts, so a rank spinning on its peer's flags cannot starve the peer).

Reference semantics: GradSync (local_run.cpp:379-414) -- every unit applies the mean of the k
units' gradients, summed in unit order, then Adam (mlp.cpp:146-161); replica env ranges are
split_envs (plan.cpp:46-55). Bounded waits / PeerFailure: local_run.cpp:543-546.

Checked: (1) both ranks end with identical params, (2) those equal a host-side emulation of
the exchange -- each unit's own fast gradient (flw_dpd_learn_grads), the f32 sum in rank order,
x 1/k, then flw_dpd_apply_grads -- bit for bit, (3) a rank whose peer never arrives fails with
Timeout after its deadline instead of hanging (the abort word releases the flag waits).
"""
import multiprocessing as mp
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ALGO = {"algorithm": "ppo", "actor": {"num": 2}, "env": {"type": "synth17x6", "num": 1024},
        "policy_net": {"hidden": [64] * 6}, "loop": {"episodes": 2, "steps_per_episode": 32}}
K = 2
SEED = 21


def _range(rank, total=1024, k=K):
    base, rem = divmod(total, k)  # split_envs (plan.cpp:46-55)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def _unit(rank, q_up, q_down, q_res, q_bye, episodes, timeout_ms):
    import sys

    sys.path.insert(0, ROOT)
    from paper_2210_00882_b200 import DpdEngine

    try:
        lo, hi = _range(rank)
        eng = DpdEngine(ALGO, device=0, seed=SEED, env_lo=lo, env_hi=hi, env_total=1024, numerics="fast")
        eng.set_timeout(timeout_ms)
        q_up.put((rank, eng.p2p_export(K)))
        handles = q_down.get(timeout=120)
        eng.p2p_import(handles, rank)
        rewards = [eng.run_episode(ep)[0] for ep in range(episodes)]
        q_res.put((rank, "ok", rewards, eng.params()))
    except Exception as exc:  # noqa: BLE001
        q_res.put((rank, "error", repr(exc), None))
    # keep this rank's exchange region mapped until every rank is done with it
    q_bye.get(timeout=600)


def _group(episodes, timeout_ms=60000):
    ctx = mp.get_context("spawn")
    q_up, q_res = ctx.Queue(), ctx.Queue()
    q_down = [ctx.Queue() for _ in range(K)]
    q_bye = [ctx.Queue() for _ in range(K)]
    procs = [ctx.Process(target=_unit, args=(r, q_up, q_down[r], q_res, q_bye[r], episodes[r], timeout_ms))
             for r in range(K)]
    for p in procs:
        p.start()
    hs = dict(q_up.get(timeout=300) for _ in range(K))
    for r in range(K):
        q_down[r].put([hs[i] for i in range(K)])
    res = {}
    for _ in range(K):
        r, status, a, b = q_res.get(timeout=300)
        res[r] = (status, a, b)
    for q in q_bye:
        q.put("bye")
    for p in procs:
        p.join(timeout=60)
    return res


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_p2p_exchange_two_units_one_gpu_matches_host_mean():
    _need_gpu()
    from paper_2210_00882_b200 import DpdEngine

    res = _group([2, 2])
    for r in range(K):
        assert res[r][0] == "ok", res[r]
    p0, p1 = res[0][2], res[1][2]
    np.testing.assert_array_equal(p0, p1)

    # host-side GradSync emulation, same process, no group: per-unit fast gradients, the f32 sum
    # in rank order (k_sum_adam's order), x 1/k in double, Adam through flw_dpd_apply_grads
    units = []
    for r in range(K):
        lo, hi = _range(r)
        units.append(DpdEngine(ALGO, device=0, seed=SEED, env_lo=lo, env_hi=hi, env_total=1024, numerics="fast"))
    for ep in range(2):
        for r, u in enumerate(units):
            u.reset(ep)
            for st in range(32):
                u.step(ep, st)
        for it in range(4):
            gs = np.zeros(units[0].param_count, dtype=np.float32)
            for u in units:
                u.learn_grads(ep, it)
                gs = gs + u.get("grads").astype(np.float32)
            gmean = gs.astype(np.float64) * (1.0 / K)
            for u in units:
                u.apply_grads(gmean)
    for r in range(K):
        np.testing.assert_array_equal(units[r].params(), units[0].params())
    diff = np.abs(units[0].params() - p0).max()
    print(f"p2p vs host mean: max |dparam| {diff:.3g}")
    np.testing.assert_array_equal(units[0].params(), p0)


def test_p2p_exchange_times_out_when_a_peer_never_arrives():
    """Rank 1 maps the group and never runs an episode: rank 0's flag waits are released by the
    abort word once its 3 s deadline passes, and the call raises Timeout (no hang)."""
    _need_gpu()
    res = _group([1, 0], timeout_ms=3000)
    assert res[1][0] == "ok"
    assert res[0][0] == "error" and "Timeout" in res[0][1], res[0]
