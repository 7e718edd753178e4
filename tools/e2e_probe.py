"""e2e breakdown of flw_run_local at C2 (diagnostic): total wall time vs per-episode wall_ms."""
import sys, time
sys.path.insert(0, ".")
import bench
from paper_2210_00882_b200.api import Program

for eps in (20, 20, 100):
    prog = Program(bench.algo_config(4096, episodes=eps),
                   {"workers": ["local"], "slots_per_worker": {"cpu": 1, "accel": 1},
                    "distribution_policy": "dp-d", "numerics": "fast"})
    prog.run_local(seed=0, episodes=2)
    for rep in range(2):
        t0 = time.perf_counter()
        csv, summ = prog.run_local(seed=0, episodes=eps)
        dt = time.perf_counter() - t0
        rows = [l.split(",") for l in csv.strip().splitlines()]
        hdr = rows[0]
        wi = hdr.index("wall_ms") if "wall_ms" in hdr else None
        w = [float(r[wi]) for r in rows[1:]] if wi is not None else []
        print(f"eps {eps} total {dt*1e3:.3f} ms  per-ep {dt*1e3/eps:.4f}  wall_ms first {w[:3]} median {sorted(w)[len(w)//2]:.4f} sum {sum(w):.3f}", flush=True)
    prog.close()
