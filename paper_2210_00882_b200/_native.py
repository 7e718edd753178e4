"""ctypes binding of the in-tree product library libfraglow_b200.so (include/fraglow_b200.h).

There is no fallback: if the library is missing or fails to load, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "libfraglow_b200.so")
HEADER = os.path.join(os.path.dirname(PKG_DIR), "include", "fraglow_b200.h")

FLW_OK, FLW_ERR_CONFIG, FLW_ERR_RUNTIME, FLW_ERR_BIND, FLW_ERR_CHECK = 0, 2, 3, 4, 5
FLW_DUMP_DFG, FLW_DUMP_FDG, FLW_DUMP_PLAN, FLW_DUMP_DOT = 0, 1, 2, 3
FLW_NUMERICS_EXACT, FLW_NUMERICS_FAST = 0, 1


class RunOptions(C.Structure):  # flw_run_options (fraglow.h:32-39)
    _fields_ = [("seed", C.c_uint64), ("episodes", C.c_int64), ("latency_us", C.c_int64),
                ("timeout_ms", C.c_int64), ("reward_threshold", C.c_double), ("unpartitioned", C.c_int)]


class FlwError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"[{code}] {message}")
        self.code = code
        self.message = message


def build(jobs: int = 8) -> str:
    subprocess.run(["make", "-s", "-C", PKG_DIR, f"-j{jobs}"], check=True)
    return LIB_PATH


_lib = None


def lib():
    """Loads the product library (raises if it is absent: no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise FileNotFoundError(f"{LIB_PATH} is not built; run __graft_entry__.build() or make -C {PKG_DIR}")
    L = C.CDLL(LIB_PATH)
    P, vp, i64, u64, d, ci = C.POINTER, C.c_void_p, C.c_int64, C.c_uint64, C.c_double, C.c_int
    cs, pcs = C.c_char_p, P(C.c_char_p)
    sig = {
        "flw_program_create": (ci, [cs, cs, P(vp)]),
        "flw_program_destroy": (None, [vp]),
        "flw_program_dump": (ci, [vp, ci, P(vp)]),
        "flw_algo_from_graph": (ci, [C.c_char_p, P(vp)]),
        "flw_validate_plan": (ci, [vp, P(vp), P(ci)]),
        "flw_run_local": (ci, [vp, P(RunOptions), P(vp), P(vp)]),
        "flw_string_free": (None, [vp]),
        "flw_last_error": (cs, []),
        "flw_dpd_create": (ci, [cs, ci, u64, i64, i64, i64, ci, P(vp)]),
        "flw_dpd_create_replicas": (ci, [cs, ci, u64, i64, i64, i64, ci, ci, P(vp)]),
        "flw_dpd_replica_rewards": (ci, [vp, P(C.c_double), i64]),
        "flw_dpd_p2p_export": (ci, [vp, ci, C.c_char_p, i64]),
        "flw_dpd_p2p_import": (ci, [vp, C.c_char_p, i64, ci, ci]),
        "flw_dpd_p2p_disable": (ci, [vp]),
        "flw_dpd_set_timeout": (ci, [vp, i64]),
        "flw_dpd_abort": (ci, [vp]),
        "flw_dpd_destroy": (ci, [vp]),
        "flw_dpd_comm_unique_id": (ci, [C.c_char_p, i64]),
        "flw_dpd_comm_init": (ci, [vp, C.c_char_p, i64, ci, ci]),
        "flw_dpd_run_episode": (ci, [vp, i64, P(d), P(C.c_float)]),
        "flw_dpd_run_episodes": (ci, [vp, i64, i64, P(C.c_float)]),
        "flw_dpd_launch_episode": (ci, [vp, i64]),
        "flw_dpd_finish_episode": (ci, [vp, P(d)]),
        "flw_dpd_reinit": (ci, [vp, u64]),
        "flw_dpd_param_count": (ci, [vp, P(i64)]),
        "flw_dpd_get_params": (ci, [vp, P(d), i64]),
        "flw_dpd_set_params": (ci, [vp, P(d), i64]),
        "flw_dpd_stats": (ci, [vp, P(i64), P(i64), P(i64), P(i64)]),
        "flw_dpd_reset": (ci, [vp, i64]),
        "flw_dpd_step": (ci, [vp, i64, i64]),
        "flw_dpd_learn": (ci, [vp, i64, i64]),
        "flw_dpd_learn_grads": (ci, [vp, i64, i64]),
        "flw_dpd_apply_grads": (ci, [vp, P(d), i64]),
        "flw_dpd_tensor_size": (ci, [vp, cs, P(i64)]),
        "flw_dpd_read": (ci, [vp, cs, P(d), i64]),
        "flw_dpd_write": (ci, [vp, cs, P(d), i64]),
        "flw_selftest_umma": (ci, [ci, ci, ci, ci, ci, ci, P(C.c_float), P(C.c_float), P(C.c_float)]),
        "flw_selftest_tgemm": (ci, [i64, i64, i64, ci, ci, ci, ci, ci, P(C.c_float), P(C.c_float), P(C.c_float)]),
        "flw_bench_tgemm": (ci, [i64, i64, i64, ci, ci, ci, ci, P(d)]),
        "flw_microbench": (ci, [cs, i64, ci, P(d), P(d)]),
        "flw_dpd_enable_probes": (ci, [vp, ci]),
        "flw_dpd_probe_times": (ci, [vp, P(vp)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(rc: int):
    if rc != FLW_OK:
        raise FlwError(rc, lib().flw_last_error().decode(errors="replace"))


def take_string(p: C.c_void_p) -> str:
    if not p.value:
        return ""
    s = C.cast(p, C.c_char_p).value.decode()
    lib().flw_string_free(p)
    return s


def header_symbols(path: str = HEADER) -> list[str]:
    """Function names declared in include/fraglow_b200.h."""
    import re

    text = open(path).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(flw_[a-z_0-9]+)\s*\(", text)))
