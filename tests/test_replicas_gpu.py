"""R reference units folded into one engine per GPU ("R per GPU with segmented
statistics"; BASELINE configs[4] = C5, 24 A3C actors on 1 and 8 GPUs). Exact numerics must
reproduce the unmodified reference's k-replica DP-D runs bit for bit: every folded replica keeps
its own advantage statistics, loss mean (over its T*E_r rows), gradient and reward sum, and the
gradients are averaged in unit order (local_run.cpp:408-411)."""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _run(name, reps_per_gpu, numerics="exact"):
    from paper_2210_00882_b200 import Program

    z = np.load(os.path.join(GOLDEN, f"run_{name}.npz"))
    algo = json.loads(str(z["__algo__"]))
    k = int(z["k"])
    prog = Program(algo, {"workers": ["local"], "slots_per_worker": {"cpu": max(16, k), "accel": max(16, k)},
                          "distribution_policy": "dp-d", "numerics": numerics, "replicas_per_gpu": reps_per_gpu})
    csv, s = prog.run_local(seed=int(z["__seed__"]))
    return z, csv, s


def _check_exact(z, csv, s):
    rewards = [float(l.split(",")[2]) for l in csv.strip().split("\n")[1:]]
    np.testing.assert_allclose(rewards, z["rewards"], rtol=1e-5)
    assert s["steps"] == int(z["steps"])
    assert s["bytes_total"] == int(np.sum(z["bytes_total"]))
    par = z["final_params"]
    assert s["param_count"] == par.size
    assert s["param_checksum"] == pytest.approx(par.sum(), rel=1e-12, abs=1e-12)
    assert s["param_l2"] == pytest.approx(np.sqrt((par ** 2).sum()), rel=1e-12)


@pytest.mark.parametrize("name", ["dpd_k2_synth", "dpd_k3_gridline", "dpd_a3c_k4", "dpd_a3c_k24",
                                  "dpd_k6_synth_uneven"])
def test_all_units_folded_on_one_gpu_bit_exact(name):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    k = int(np.load(os.path.join(GOLDEN, f"run_{name}.npz"))["k"])
    _check_exact(*_run(name, k))


@pytest.mark.parametrize("name,gpus", [("dpd_k6_synth_uneven", 2), ("dpd_a3c_k24", 2), ("dpd_a3c_k24", 4),
                                       ("dpd_a3c_k4", 2)])
def test_units_folded_over_gpus_bit_exact(name, gpus):
    """R = k / #GPUs units per GPU, AllGather of each rank's R gradients + unit-ordered mean."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < gpus:
        pytest.skip(f"needs {gpus} GPUs")
    k = int(np.load(os.path.join(GOLDEN, f"run_{name}.npz"))["k"])
    _check_exact(*_run(name, k // gpus))


def test_fast_folded_matches_exact_folded():
    """Fast numerics with folded replicas: per-replica weights/statistics inside the tensor-core
    learn kernel; the trained parameters stay close to the exact run."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    z, _, s_exact = _run("dpd_k6_synth_uneven", 6, "exact")
    _, csv, s_fast = _run("dpd_k6_synth_uneven", 6, "fast")
    assert s_fast["steps"] == s_exact["steps"]
    assert s_fast["param_l2"] == pytest.approx(s_exact["param_l2"], rel=2e-3)
    r_fast = [float(l.split(",")[2]) for l in csv.strip().split("\n")[1:]]
    np.testing.assert_allclose(r_fast, z["rewards"], rtol=2e-2)


def test_engine_replicas_rewards_unit_order():
    """flw_dpd_create_replicas: per-replica reward sums equal R single-replica engines' sums on
    the first (pre-learning) episode."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2210_00882_b200 import DpdEngine

    algo = {"algorithm": "ppo", "env": {"type": "gridline", "num": 10}, "policy_net": {"hidden": [8]},
            "loop": {"episodes": 1, "steps_per_episode": 8}}
    eng = DpdEngine(algo, seed=3, env_lo=0, env_hi=10, env_total=10, numerics="exact", replicas=3)
    eng.run_episode(0)
    got = eng.replica_rewards()
    bounds = [(0, 4), (4, 7), (7, 10)]  # split_envs(10, 3)
    for r, (lo, hi) in enumerate(bounds):
        one = DpdEngine(algo, seed=3, env_lo=lo, env_hi=hi, env_total=10, numerics="exact")
        assert one.run_episode(0)[0] == got[r]
