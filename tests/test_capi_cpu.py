"""CPU-side checks of the C-ABI boundary (no GPU needed): the library loads, exports every
symbol include/fraglow_b200.h declares, and its control plane (config parsing/validation, the
DP-D placement, plan dump, error codes and messages) matches the reference's own C API on the
same documents (tests/golden/plans.json, produced by the unmodified reference)."""
import json
import os

import pytest

from paper_2210_00882_b200 import FlwError, Program
from paper_2210_00882_b200 import _native as N

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
PLANS = json.load(open(os.path.join(GOLDEN, "plans.json")))


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    syms = N.header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


@pytest.mark.parametrize("case", PLANS, ids=[f"plan{i}" for i in range(len(PLANS))])
def test_program_matches_reference_c_api(case):
    if case["rc"] == 0:
        p = Program(case["algo"], case["deploy"])
        assert json.loads(p.dump()) == case["plan"]
        viol, n = p.validate_plan()
        assert n == len(case["violations"]) and viol == case["violations"]
    else:
        with pytest.raises(FlwError) as ei:
            Program(case["algo"], case["deploy"])
        assert ei.value.code == case["rc"]
        assert ei.value.message == case["error"]


def test_non_dpd_policies_are_refused_loudly():
    for pol in ("dp-a", "single_learner_fine", "dp-c", "dp-e", "central"):
        with pytest.raises(FlwError) as ei:
            Program({"algorithm": "ppo", "env": {"type": "gridline", "num": 4}}, {"distribution_policy": pol})
        assert ei.value.code == N.FLW_ERR_CONFIG and ei.value.message.startswith("PolicyInapplicable")
    with pytest.raises(FlwError):  # default deploy (capi.cpp:211-212) is dp-a
        Program({"algorithm": "ppo", "env": {"type": "gridline", "num": 4}}, None)


def test_only_plan_dump_is_served():
    p = Program({"algorithm": "ppo", "env": {"type": "gridline", "num": 4}}, {"distribution_policy": "dp-d"})
    for what in (N.FLW_DUMP_DFG, N.FLW_DUMP_FDG, N.FLW_DUMP_DOT):
        with pytest.raises(FlwError) as ei:
            p.dump(what)
        assert ei.value.code == N.FLW_ERR_CONFIG


def test_numerics_selection_is_validated():
    with pytest.raises(FlwError):
        Program({"algorithm": "ppo", "env": {"type": "gridline", "num": 4}},
                {"distribution_policy": "dp-d", "numerics": "approximate"})


def test_last_error_is_thread_local():
    import threading

    errs = {}

    def bad(tag, algo):
        try:
            Program(algo, {"distribution_policy": "dp-d"})
        except FlwError as e:
            errs[tag] = e.message

    t1 = threading.Thread(target=bad, args=("a", {"algorithm": "xx"}))
    t2 = threading.Thread(target=bad, args=("b", {"algorithm": "ppo", "env": {"type": "nope"}}))
    t1.start(), t2.start(), t1.join(), t2.join()
    assert errs["a"].startswith("ConfigError") and errs["b"].startswith("UnknownEnv")


def test_engine_fails_loudly_without_a_gpu():
    """The product path has no CPU fallback: creating an engine or running a program on a host
    without a visible CUDA device returns a runtime error through the ABI."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_2210_00882_b200 import DpdEngine

    algo = {"algorithm": "ppo", "env": {"type": "gridline", "num": 4}}
    with pytest.raises(FlwError) as ei:
        DpdEngine(algo, numerics="exact")
    assert ei.value.code == N.FLW_ERR_RUNTIME
    with pytest.raises(FlwError) as ei:
        DpdEngine(algo, numerics="fast", replicas=2)
    assert ei.value.code == N.FLW_ERR_RUNTIME
    p = Program(algo, {"distribution_policy": "dp-d"})
    with pytest.raises(FlwError) as ei:
        p.run_local(seed=1)
    assert ei.value.code == N.FLW_ERR_RUNTIME and "no CUDA device" in ei.value.message


def test_deploy_extension_keys_are_accepted_and_validated():
    algo = {"algorithm": "ppo", "env": {"type": "gridline", "num": 8}, "actor": {"num": 4}}
    p = Program(algo, {"distribution_policy": "dp-d", "slots_per_worker": {"cpu": 4, "accel": 4},
                       "numerics": "fast", "replicas_per_gpu": 2, "exchange": "nccl"})
    # the plan itself is the reference's (the extension keys only steer the engine)
    assert len(json.loads(p.dump())["instances"]) == 4


def test_algo_from_graph_recovers_the_algo_config():
    """The seam's graph input: the reference's own dataflow-graph JSON of a PPO / MAPPO
    standard program (tests/golden/dfg.json, dumped by oracle/_ref via flw_program_dump(DFG))
    translates back to exactly the algo config it was built from."""
    from paper_2210_00882_b200.api import algo_from_graph

    cases = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "dfg.json")))
    assert len(cases) == 3
    for name, c in cases.items():
        got, want = algo_from_graph(c["graph"]), c["algo"]
        assert got["algorithm"] == want["algorithm"], name
        assert got["agent"]["num"] == want["agent"]["num"], name
        assert got["env"]["type"] == want["env"]["type"] and got["env"]["num"] == want["env"]["num"], name
        assert got["env"].get("params", {}) == {k: float(v) for k, v in want["env"].get("params", {}).items()}, name
        assert got["policy_net"] == want["policy_net"], name
        assert got["learner"]["params"] == want["learner"]["params"], name
        assert got["loop"] == want["loop"], name


def test_algo_from_graph_refuses_what_it_cannot_read():
    from paper_2210_00882_b200.api import algo_from_graph

    with pytest.raises(FlwError, match="nodes"):
        algo_from_graph({"edges": []})
    with pytest.raises(FlwError, match="standard program"):
        algo_from_graph({"nodes": [{"id": 0, "kind": "Input", "attrs": {}}]})
    with pytest.raises(FlwError, match="A3C"):
        algo_from_graph({"nodes": [{"id": 0, "kind": "A3cLoss", "attrs": {}}]})
