#!/usr/bin/env python3
"""Benchmark of the fused DP-D PPO loop (BASELINE.json metric: env-steps/s and episode time).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--numerics fast|exact]

Workload (BASELINE.json configs[1], "C2"): PPO, builder env synth17x6 (obs 17, 6 actions),
4096 envs per GPU, 7-layer MLP (hidden [64]*6) policy and critic, T=32 steps, 4 train iters.
One bench "step" = one whole episode (reset, 32 env steps, 4 PPO iterations) of every unit.
N>1 (torchrun): one unit per GPU, 4096 envs each (weak scaling; 16384 total at N=4 = configs[3]),
gradients averaged every train iteration over NVLink (the DP-C == replicated DP-D exchange).

--impl reference times the reference's own CPU implementation (oracle/_ref/ref_tool: the
unmodified reference compiled from its sources) on this host's cores on the same workload
(4096 envs per GPU of the run), DP-D with one replica thread per core, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ENVS_PER_GPU = 4096
T_STEPS = 32
HIDDEN = [64] * 6
METRIC = "env-steps/sec (fused DP-D PPO loop, episode incl. learn)"


def algo_config(envs: int, actors: int = 1, episodes: int = 1) -> dict:
    return {
        "algorithm": "ppo",
        "agent": {"num": 1},
        "actor": {"num": actors},
        "env": {"type": "synth17x6", "num": envs},
        "learner": {"num": 1, "params": {"gamma": 0.97, "lam": 0.95, "clip_eps": 0.2, "lr": 3e-3,
                                         "train_iters": 4, "value_coef": 0.5, "entropy_coef": 0.01,
                                         "normalize_adv": True}},
        "policy_net": {"hidden": HIDDEN, "activation": "tanh"},
        "loop": {"episodes": episodes, "steps_per_episode": T_STEPS},
    }


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def wait_ready(self, timeout_s: float = 5.0):
        """nvidia-smi's start-up (driver init) must not land in the timed region: it can stall
        this process's CUDA launches for milliseconds, and at N > 1 the other ranks then wait
        for it inside the gradient exchange."""
        t0 = time.perf_counter()
        while self.proc and not self.samples and time.perf_counter() - t0 < timeout_s:
            time.sleep(0.02)

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit())
        mx = max(float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[5 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.samples)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo", rank=rank, world_size=world)
    return world, rank, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def ref_tool_path() -> str:
    return os.path.join(ROOT, "oracle", "_ref", "ref_tool")


def run_reference(envs: int, replicas: int, episodes: int, seed: int = 7) -> dict:
    """One ref_tool run (the unmodified reference, DP-D with `replicas` unit threads)."""
    algo = algo_config(envs, actors=replicas, episodes=episodes)
    with tempfile.TemporaryDirectory() as tmp:
        ap, dp = os.path.join(tmp, "a.json"), os.path.join(tmp, "d.json")
        json.dump(algo, open(ap, "w"))
        json.dump({"workers": ["local"], "slots_per_worker": {"cpu": replicas, "accel": replicas},
                   "distribution_policy": "dp-d"}, open(dp, "w"))
        out = subprocess.run([ref_tool_path(), "run", ap, dp, str(seed)], check=True, capture_output=True,
                             text=True).stdout
    return json.loads(out)


def reference_sample(cores: int, target_s: float) -> tuple[int, int]:
    """Bounded sample: envs so that one episode is ~target_s on `cores` threads (C2 cost measured
    on the GPU box host: ~0.023 s of one core per env per episode), one replica per core."""
    envs = int(max(cores, min(ENVS_PER_GPU, round(target_s * cores / 0.023))))
    envs -= envs % cores
    return max(envs, cores), cores


def mlp_macs(dims) -> tuple[int, int]:
    """(sum in*out over layers, same without the first layer) for one MLP."""
    macs = [dims[i] * dims[i + 1] for i in range(len(dims) - 1)]
    return sum(macs), sum(macs[1:])


def load_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"], "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback"}


def ncu_traffic(tag: str):
    """dram read+write bytes per launch of kernel `tag` from the committed ncu summary, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        return json.load(open(p)).get(tag)
    return None


def roofline_for(tag: str, ms: float, envs: int, peaks: dict) -> dict:
    """Dominant-kernel roofline. Learn kernels are tensor-core GEMM chains: algorithmic FLOPs =
    2 * rows * (forward + dW + dH) MACs of that net (real, unpadded dims)."""
    pol = [17] + HIDDEN + [6]
    cri = [17] + HIDDEN + [1]
    rows = envs * T_STEPS
    if tag == "learn":  # policy || critic learn kernels, concurrent on a 60/40 SM split
        pf, pdh = mlp_macs(pol)
        cf, cdh = mlp_macs(cri)
        # policy: forward + dW + dH; critic: dW + dH (its forward is the values pass, reused)
        flops = 2.0 * rows * ((pf + pf + pdh) + (cf + cdh))
        ach = flops / (ms * 1e-3) / 1e12
        return {"kernel": "learn (k_learn policy || k_learn critic, concurrent)", "bound": "tensor", "achieved": ach,
                "peak": peaks["bf16_tflops"], "unit": "TFLOP/s", "frac": ach / peaks["bf16_tflops"],
                "traffic": ncu_traffic("learn"), "peak_source": peaks["source"],
                "work_per_launch": f"{flops:.4g} FLOP ({rows} rows, both nets)", "launch_ms": ms}
    if tag in ("learn_policy", "learn_critic", "critic_fwd"):
        dims = pol if tag == "learn_policy" else cri
        fwd, dh = mlp_macs(dims)
        flops = 2.0 * rows * (fwd if tag == "critic_fwd" else fwd + fwd + dh)
        ach = flops / (ms * 1e-3) / 1e12
        return {"kernel": tag, "bound": "tensor", "achieved": ach, "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
                "frac": ach / peaks["bf16_tflops"], "traffic": ncu_traffic(tag), "peak_source": peaks["source"],
                "work_per_launch": f"{flops:.4g} FLOP ({rows} rows x 2 x MACs)", "launch_ms": ms}
    if tag == "rollout":
        # per env-step: (8S+9) B trajectory/env bytes + policy MLP FLOPs on CUDA cores
        nbytes = envs * T_STEPS * (8 * 17 + 9)
        ach = nbytes / (ms * 1e-3) / 1e9
        return {"kernel": tag, "bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": ach / peaks["hbm_gbs"], "traffic": ncu_traffic(tag), "peak_source": peaks["source"],
                "work_per_launch": f"{nbytes} B ((8S+9) B x {envs * T_STEPS} env-steps)", "launch_ms": ms}
    return {"kernel": tag, "bound": "hbm", "achieved": None, "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": None,
            "traffic": None}


def hbm_microbenchmarks(peaks: dict) -> dict:
    """The HBM-bound kernels the episodes launch, at scaled sizes (at C2 they move
    < 20 MB and are launch/L2 bound), with the survey's algorithmic bytes per unit:
      rollout_env   k_rollout (PolicyApply + env step of the per-step rollouts), 2^21 envs, 173 B/env-step
      gae_scan32    k_gae_scan32 (the episodes' GAE, T = 32), 2^26 rows, 17 B/row
      gae_streams   k_fast_gae<8,4> (the GAE kernel for T != 32), 2^26 rows, 17 B/row
      reduce_adam   k_reduce_adam (the fused per-iteration update, 1 GPU), 2^26 params, 8 partial slots:
                    44 B/param (Adam, f64 moments) + 4 B/param per slot
      exchange_adam k_exchange_adam (the k-GPU peer-memory update, k = 1), same
    In the C2 fast episode the env step is fused into k_rollout_episode (MMA-latency bound: see
    kernel_shares / rollout_only)."""
    from paper_2210_00882_b200.api import microbench

    out = {}
    for name, kern, n in (("rollout_env", "rollout_env", 1 << 21), ("gae_scan32", "gae_scan32", 1 << 26),
                          ("gae_streams", "gae", 1 << 26), ("reduce_adam", "reduce_adam", 1 << 26),
                          ("exchange_adam", "exchange_adam", 1 << 26)):
        ms, nbytes = microbench(kern, n, 10)
        gbs = nbytes / (ms * 1e-3) / 1e9
        out[name] = {"n": n, "ms": ms, "bytes": nbytes, "achieved_gbs": gbs, "frac": gbs / peaks["hbm_gbs"]}
    return out


def cpu_baseline(target_s: float = 12.0) -> dict:
    cores = os.cpu_count() or 1
    if not os.path.exists(ref_tool_path()):
        return {"value": None, "unit": "env-steps/s", "cores": cores, "kind": "reference",
                "sample": "unavailable: oracle/_ref/ref_tool not built"}
    envs, k = reference_sample(cores, target_s)
    r = run_reference(envs, k, episodes=1)
    ms = sum(e["wall_ms"] for e in r["episodes"])
    # the same path on ONE core (one dp-d unit), bounded sample
    e1 = int(max(8, min(ENVS_PER_GPU, round(0.4 * target_s / 0.023))))
    r1 = run_reference(e1, 1, episodes=1)
    ms1 = sum(e["wall_ms"] for e in r1["episodes"])
    return {"value": envs * T_STEPS * len(r["episodes"]) / (ms / 1e3), "unit": "env-steps/s", "cores": cores,
            "kind": "reference", "cpu_model": cpu_model(),
            "sample": f"1 episode of C2 at {envs} envs (dp-d, {k} replica threads), {ms / 1e3:.1f} s",
            "single_core": {"value": e1 * T_STEPS / (ms1 / 1e3), "unit": "env-steps/s", "cores": 1,
                            "sample": f"1 episode of C2 at {e1} envs (dp-d, 1 unit), {ms1 / 1e3:.1f} s"}}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def bench_reference(args, world, rank):
    """The reference's own CPU implementation of the path (oracle/_ref/ref_tool = the unmodified
    reference compiled from its sources) on this host's cores, on OUR arm's config: C2 at 4096
    envs (ENVS_PER_GPU x world when N > 1, timed on rank 0's host only), DP-D with one replica
    thread per core. One ref_tool process runs W + K episodes; the reference's own per-episode
    wall_ms (local_run.cpp:540-551) of the last K are the steps."""
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    envs = ENVS_PER_GPU * world
    k = min(cores, envs)
    # N > 1: the whole job's envs on one host; the episode count shrinks by the same factor
    # (>= 1 warm-up + 1 timed) so the CPU arm stays within minutes
    warm, steps = args.warmup, args.steps
    if world > 1:
        warm = 1
        steps = max(1, round(args.steps / world))
    r = run_reference(envs, k, episodes=warm + steps)
    times = [e["wall_ms"] for e in r["episodes"]][warm:]
    ms = sum(times) / len(times)
    value = envs * T_STEPS / (ms / 1e3)
    line = {"metric": METRIC, "value": value, "unit": "env-steps/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32-storage/f64-accumulate", "data": "synthetic (synth17x6 env, seeded)",
            "impl": "reference",
            "config": {"workload": f"C2: PPO synth17x6, {envs} envs, 7-layer MLP (hidden 6x{HIDDEN[0]}), T=32, "
                                   f"train_iters=4, dp-d with {k} CPU replica threads",
                       "envs_total": envs, "envs_per_gpu": ENVS_PER_GPU, "replicas": k, "numerics": "reference",
                       "cpu_model": cpu_model()},
            "cpu_baseline": {"value": value, "unit": "env-steps/s", "cores": k, "kind": "reference",
                             "cpu_model": cpu_model(),
                             "sample": f"{steps} timed episodes (after {warm} warm-up) of the full "
                                       f"workload, {envs} envs, {k} replica threads"},
            "e2e": {"value": value, "unit": "env-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def bench_ours(args, world, rank, local):
    import torch

    from paper_2210_00882_b200 import DpdEngine, Program

    torch.cuda.set_device(local)
    total = ENVS_PER_GPU * world
    algo = algo_config(total, actors=world, episodes=args.warmup + 2 * args.steps + 8)
    lo, hi = rank * ENVS_PER_GPU, (rank + 1) * ENVS_PER_GPU
    eng = DpdEngine(algo, device=local, seed=args.seed, env_lo=lo, env_hi=hi, env_total=total,
                    numerics=args.numerics)
    if world > 1:
        import torch.distributed as dist

        obj = [DpdEngine.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        eng.comm_init(obj[0], rank, world)
        if args.numerics == "fast" and args.exchange == "p2p":
            # gradient exchange over NVLink peer memory (CUDA IPC), fused with reduce + Adam;
            # the group falls back to NCCL together if any rank cannot map its peers
            ok = True
            try:
                hs = [None] * world
                dist.all_gather_object(hs, eng.p2p_export(world))
                eng.p2p_import(hs, rank)
            except Exception as exc:  # noqa: BLE001
                print(f"rank {rank}: peer-memory exchange unavailable ({exc}); using NCCL", file=sys.stderr)
                ok = False
            oks = [None] * world
            dist.all_gather_object(oks, ok)
            if not all(oks):
                eng.p2p_disable()
                args.exchange = "nccl"
    # warm-up (also captures the episode graph; no instrumentation in the timed graph)
    eng.enable_probes(False)
    eng.run_episodes(0, args.warmup)
    with ClockSampler(local) as clk:
        clk.wait_ready()
        barrier(world)
        torch.cuda.synchronize()
        dev_ms = eng.run_episodes(args.warmup, args.steps)
        torch.cuda.synchronize()
    barrier(world)
    dev_ms = max_over_ranks(dev_ms, world)
    value = total * T_STEPS * args.steps / (dev_ms / 1e3)
    stats = eng.stats()

    # e2e through the reference's public API (flw_run_local, fraglow.h:55) on one GPU: a dp-d
    # program runs K episodes with the host episode gate - per episode the episode index goes
    # host->device and the reward sum device->host; per run the initial params go in and the
    # final params come out. N > 1 (one process per GPU): the per-unit seam flw_dpd_run_episode
    # with the same per-episode round trips (flw_run_local drives in-process GPUs only).
    barrier(world)
    P = eng.param_count
    if world == 1:
        prog = Program(algo_config(total, episodes=args.steps),
                       {"workers": ["local"], "slots_per_worker": {"cpu": 1, "accel": 1},
                        "distribution_policy": "dp-d", "numerics": args.numerics})
        prog.run_local(seed=args.seed, episodes=2)  # engine build + graph capture (untimed)
        t0 = time.perf_counter()
        _, summ = prog.run_local(seed=args.seed, episodes=args.steps)
        e2e_s = time.perf_counter() - t0
        assert summ["episodes"] == args.steps
        e2e = {"value": total * T_STEPS * args.steps / e2e_s, "unit": "env-steps/s", "api": "flw_run_local",
               "h2d_bytes_per_step": 8 + 4 * P / args.steps, "d2h_bytes_per_step": 8 + 4 * P / args.steps}
        prog.close()
    else:
        # (pipelined: episode i + 1 enqueued before the host waits for episode i's reward)
        t0 = time.perf_counter()
        base = args.warmup + args.steps
        eng.launch_episode(base)
        for i in range(args.steps):
            if i + 1 < args.steps:
                eng.launch_episode(base + i + 1)
            eng.finish_episode()
        e2e_s = max_over_ranks(time.perf_counter() - t0, world)
        e2e = {"value": total * T_STEPS * args.steps / e2e_s, "unit": "env-steps/s", "api": "flw_dpd_launch_episode/flw_dpd_finish_episode",
               "h2d_bytes_per_step": 8, "d2h_bytes_per_step": 8}

    # per-kernel shares (roofline, kernel_shares): a separately captured graph with CUDA-event
    # probes around the main kernels (external event-record nodes), outside the timed regions
    eng.enable_probes(True)
    eng.run_episodes(args.warmup + 2 * args.steps, 1)  # captures the probed graph (per-rank delay)
    torch.cuda.synchronize()
    barrier(world)  # ranks aligned again: the exchange probes must not absorb the capture skew
    eng.run_episodes(args.warmup + 2 * args.steps + 1, 2)
    torch.cuda.synchronize()
    probes = eng.probe_times()  # per-kernel ms of the last probed episode
    eng.enable_probes(False)
    barrier(world)

    if rank != 0:
        return
    peaks = load_peaks()
    episode_ms = dev_ms / args.steps
    shares = {k: {"ms_per_episode": sum(v), "launches": len(v), "share": sum(v) / episode_ms} for k, v in probes.items()}
    dom = max(shares, key=lambda k: shares[k]["ms_per_episode"]) if shares else None
    if dom == "learn_policy" and "learn_critic" not in probes:
        dom = "learn"  # the critic learn kernel runs inside the policy kernel's window
        probes_dom = probes["learn_policy"]
    else:
        probes_dom = probes.get(dom, [])
    roofline = roofline_for(dom, sum(probes_dom) / len(probes_dom), ENVS_PER_GPU, peaks) if dom else None
    line = {"metric": METRIC, "value": value, "unit": "env-steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if args.envs_total else "weak", "vs_baseline": None,
            "dtype": "f32-storage/f64-accumulate" if args.numerics == "exact" else "bf16-mma/f32-accumulate",
            "data": "synthetic (synth17x6 env, seeded)",
            "config": {"workload": (f"C4: PPO synth17x6, {total} envs over {world} learners" if args.envs_total else
                                    "C2: PPO synth17x6, 4096 envs/GPU") +
                                   f", 7-layer MLP (hidden 6x{HIDDEN[0]}), T=32, train_iters=4, dp-d fused loop",
                       "envs_total": total, "envs_per_gpu":
                       ENVS_PER_GPU, "numerics": args.numerics, "parallelism": f"dp{world}",
                       "exchange": (args.exchange if args.numerics == "fast" else "nccl") if world > 1 else None,
                       "l2": "per-episode working set (activations, ~0.9 GB) exceeds the 126 MB L2"},
            "episode_ms": episode_ms, "gpu_launches": stats["graph_kernels"] * args.steps,
            "clocks": clk.summary(), "e2e": e2e, "roofline": roofline, "kernel_shares": shares}
    if "rollout" in probes:  # "also report rollout-only"
        r_ms = sum(probes["rollout"])
        line["rollout_only"] = {"value": total * T_STEPS / (r_ms * 1e-3), "unit": "env-steps/s",
                                "ms_per_episode": r_ms, "note": "Reset + 32 fused policy/env steps, per GPU x N"}
    if not args.no_microbench:
        line["hbm_kernels"] = hbm_microbenchmarks(peaks)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline()
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--numerics", choices=["exact", "fast"], default="fast")
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exchange", choices=["p2p", "nccl"], default="p2p",
                    help="N>1 fast numerics: gradient exchange over NVLink peer memory (one fused kernel) or NCCL")
    ap.add_argument("--hidden", type=int, default=64,
                    help="hidden width H of the 7-layer MLP (SURVEY §8: H=64, also report H=256; fast numerics "
                         "supports H <= 64)")
    ap.add_argument("--envs-total", type=int, default=0,
                    help="strong scaling: this many envs split over the N GPUs (C4: 16384); default 4096 per GPU")
    ap.add_argument("--no-microbench", action="store_true",
                    help="skip the scaled HBM kernel sweeps (profiling runs: the launch list then holds episodes only)")
    args = ap.parse_args()
    global HIDDEN, ENVS_PER_GPU
    HIDDEN = [args.hidden] * 6
    world, rank, local = dist_setup()
    if args.envs_total:  # strong scaling (BASELINE configs[3]: 16384 envs over N learners)
        if args.envs_total % world:
            raise SystemExit("--envs-total must be a multiple of the GPU count")
        ENVS_PER_GPU = args.envs_total // world
    if args.impl == "reference":
        bench_reference(args, world, rank)
    else:
        bench_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
