"""One fast-numerics episode on the C2 workload (used with a -DFLW_LEARN_TRACE build to print the
k_learn stage timeline of CTA 0)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_00882_b200 import DpdEngine
import bench

algo = bench.algo_config(4096)
eng = DpdEngine(algo, device=0, seed=1, env_lo=0, env_hi=4096, env_total=4096, numerics="fast")
eng.run_episodes(0, 1)
