"""Python mirror of the reference's C API for the DP-D path (fraglow.h) and of the per-unit
engine seam. Every call goes through libfraglow_b200.so; nothing computes in Python.

    prog = Program(algo_json, deploy_json)          # flw_program_create (dp-d plans only)
    csv, summary = prog.run_local(seed=7)           # flw_run_local -> (CSV text, summary dict)

    eng = DpdEngine(algo_json, device=0, seed=7)    # one unit (replica) on one GPU
    reward_sum, ms = eng.run_episode(0)             # one fused episode (CUDA graph replay)
"""
from __future__ import annotations

import ctypes as C
import json

import numpy as np

from . import _native as N


def _json(x) -> bytes:
    return (x if isinstance(x, str) else json.dumps(x)).encode()


class Program:
    """flw_program: parsed configs + DP-D placement; runs on local GPUs."""

    def __init__(self, algo, deploy=None):
        self._h = C.c_void_p()
        N.check(N.lib().flw_program_create(_json(algo), _json(deploy) if deploy is not None else None,
                                           C.byref(self._h)))

    def close(self):
        if self._h:
            N.lib().flw_program_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def dump(self, what: int = N.FLW_DUMP_PLAN) -> str:
        out = C.c_void_p()
        N.check(N.lib().flw_program_dump(self._h, what, C.byref(out)))
        return N.take_string(out)

    def validate_plan(self) -> tuple[list, int]:
        out, n = C.c_void_p(), C.c_int(0)
        N.check(N.lib().flw_validate_plan(self._h, C.byref(out), C.byref(n)))
        return json.loads(N.take_string(out)), n.value

    def run_local(self, seed: int = 0, episodes: int = 0, reward_threshold: float = -1.0,
                  unpartitioned: bool = False, timeout_ms: int = 0) -> tuple[str, dict]:
        opts = N.RunOptions(seed, episodes, 0, timeout_ms, reward_threshold, int(unpartitioned))
        csv, summ = C.c_void_p(), C.c_void_p()
        N.check(N.lib().flw_run_local(self._h, C.byref(opts), C.byref(csv), C.byref(summ)))
        return N.take_string(csv), json.loads(N.take_string(summ))


def algo_from_graph(graph) -> dict:
    """flw_algo_from_graph: the algo config of a PPO / MAPPO dataflow-graph JSON (dfg::dump_json)."""
    out = C.c_void_p()
    N.check(N.lib().flw_algo_from_graph(_json(graph), C.byref(out)))
    return json.loads(N.take_string(out))


def microbench(which: str, n: int, iters: int = 10) -> tuple[float, float]:
    """flw_microbench: (ms per launch, algorithmic bytes per launch) of an element-wise kernel."""
    ms, nbytes = C.c_double(), C.c_double()
    N.check(N.lib().flw_microbench(which.encode(), n, iters, C.byref(ms), C.byref(nbytes)))
    return ms.value, nbytes.value


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class DpdEngine:
    """flw_dpd: one DP-D unit owning envs [env_lo, env_hi) of env_total on `device`."""

    def __init__(self, algo, device: int = 0, seed: int = 0, env_lo: int = 0, env_hi: int | None = None,
                 env_total: int | None = None, numerics: str = "exact", replicas: int = 1):
        a = json.loads(algo) if isinstance(algo, str) else algo
        if "nodes" in a:  # the dataflow-graph JSON (the seam's graph input): its env count
            total = int(algo_from_graph(a)["env"]["num"]) if env_total is None else env_total
        else:
            total = int(a.get("env", {}).get("num", 1)) if env_total is None else env_total
        hi = total if env_hi is None else env_hi
        num = {"exact": N.FLW_NUMERICS_EXACT, "fast": N.FLW_NUMERICS_FAST}[numerics]
        self._h = C.c_void_p()
        self.replicas = replicas
        if replicas == 1:
            N.check(N.lib().flw_dpd_create(_json(a), device, seed, env_lo, hi, total, num, C.byref(self._h)))
        else:
            N.check(N.lib().flw_dpd_create_replicas(_json(a), device, seed, env_lo, hi, total, num, replicas,
                                                    C.byref(self._h)))

    def replica_rewards(self):
        """Per-replica reward sums of the last episode (unit order)."""
        out = (C.c_double * self.replicas)()
        N.check(N.lib().flw_dpd_replica_rewards(self._h, out, self.replicas))
        return list(out)

    def close(self):
        if self._h:
            N.lib().flw_dpd_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- gradient group
    @staticmethod
    def comm_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        N.check(N.lib().flw_dpd_comm_unique_id(buf, 128))
        return buf.raw

    def p2p_export(self, nranks: int) -> bytes:
        """CUDA IPC handle of this unit's peer-memory exchange region (fast numerics)."""
        buf = C.create_string_buffer(80)  # FLW_P2P_HANDLE_BYTES: IPC handle + GPU UUID
        N.check(N.lib().flw_dpd_p2p_export(self._h, nranks, buf, 80))
        return buf.raw

    def p2p_import(self, handles: list, rank: int):
        """Map every rank's exchange region (handles in rank order): gradients then move over
        NVLink peer memory inside one fused reduce/all-reduce/Adam kernel instead of NCCL."""
        blob = b"".join(handles)
        N.check(N.lib().flw_dpd_p2p_import(self._h, blob, len(blob), rank, len(handles)))

    def set_timeout(self, timeout_ms: int):
        """Bound on a grouped unit's waits for its peers (0: 30 s); past it the call raises Timeout."""
        N.check(N.lib().flw_dpd_set_timeout(self._h, timeout_ms))

    def abort(self):
        """Abort this unit's gradient group (its waits fail with PeerFailure)."""
        N.check(N.lib().flw_dpd_abort(self._h))

    def p2p_disable(self):
        N.check(N.lib().flw_dpd_p2p_disable(self._h))

    def comm_init(self, uid: bytes, rank: int, nranks: int):
        N.check(N.lib().flw_dpd_comm_init(self._h, uid, len(uid), rank, nranks))

    # -- whole episodes
    def run_episode(self, episode: int) -> tuple[float, float]:
        r, ms = C.c_double(), C.c_float()
        N.check(N.lib().flw_dpd_run_episode(self._h, episode, C.byref(r), C.byref(ms)))
        return r.value, ms.value

    def launch_episode(self, episode: int):
        """Enqueue one episode (at most two in flight); finish_episode() returns the oldest's reward."""
        N.check(N.lib().flw_dpd_launch_episode(self._h, episode))

    def finish_episode(self) -> float:
        r = C.c_double()
        N.check(N.lib().flw_dpd_finish_episode(self._h, C.byref(r)))
        return r.value

    def run_episodes(self, first: int, count: int) -> float:
        ms = C.c_float()
        N.check(N.lib().flw_dpd_run_episodes(self._h, first, count, C.byref(ms)))
        return ms.value

    def reinit(self, seed: int):
        N.check(N.lib().flw_dpd_reinit(self._h, seed))

    def enable_probes(self, on: bool = True):
        """CUDA-event probes around the main kernels inside the episode graph."""
        N.check(N.lib().flw_dpd_enable_probes(self._h, int(on)))

    def probe_times(self) -> dict:
        """Per-kernel device ms of the most recent episode replay."""
        out = C.c_void_p()
        N.check(N.lib().flw_dpd_probe_times(self._h, C.byref(out)))
        return json.loads(N.take_string(out))

    # -- params / stats
    @property
    def param_count(self) -> int:
        n = C.c_int64()
        N.check(N.lib().flw_dpd_param_count(self._h, C.byref(n)))
        return n.value

    def params(self) -> np.ndarray:
        out = np.zeros(self.param_count)
        N.check(N.lib().flw_dpd_get_params(self._h, _dp(out), out.size))
        return out

    def set_params(self, p):
        p = np.ascontiguousarray(p, dtype=np.float64)
        N.check(N.lib().flw_dpd_set_params(self._h, _dp(p), p.size))

    def stats(self) -> dict:
        s, e, i, g = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        N.check(N.lib().flw_dpd_stats(self._h, C.byref(s), C.byref(e), C.byref(i), C.byref(g)))
        return {"steps": s.value, "env_count": e.value, "learn_iters": i.value, "graph_kernels": g.value}

    # -- phases
    def reset(self, episode: int):
        N.check(N.lib().flw_dpd_reset(self._h, episode))

    def step(self, episode: int, step: int):
        N.check(N.lib().flw_dpd_step(self._h, episode, step))

    def learn(self, episode: int, it: int):
        N.check(N.lib().flw_dpd_learn(self._h, episode, it))

    def learn_grads(self, episode: int, it: int):
        N.check(N.lib().flw_dpd_learn_grads(self._h, episode, it))

    def apply_grads(self, grads=None):
        if grads is None:
            N.check(N.lib().flw_dpd_apply_grads(self._h, None, 0))
        else:
            g = np.ascontiguousarray(grads, dtype=np.float64)
            N.check(N.lib().flw_dpd_apply_grads(self._h, _dp(g), g.size))

    # -- named tensors
    def size(self, name: str) -> int:
        n = C.c_int64()
        N.check(N.lib().flw_dpd_tensor_size(self._h, name.encode(), C.byref(n)))
        return n.value

    def get(self, name: str) -> np.ndarray:
        out = np.zeros(self.size(name))
        N.check(N.lib().flw_dpd_read(self._h, name.encode(), _dp(out), out.size))
        return out

    def set(self, name: str, values):
        v = np.ascontiguousarray(values, dtype=np.float64).ravel()
        N.check(N.lib().flw_dpd_write(self._h, name.encode(), _dp(v), v.size))
