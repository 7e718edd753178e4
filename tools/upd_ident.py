"""Dumps params + reward after 3 fast C2 episodes (for bit-identity A/B across update variants)."""
import sys, hashlib
sys.path.insert(0, ".")
import bench
from paper_2210_00882_b200.api import DpdEngine
e = DpdEngine(bench.algo_config(4096), 0, seed=7, numerics="fast")
r = [e.run_episode(i) for i in range(3)]
p = e.params()
print(sys.argv[1] if len(sys.argv) > 1 else "", hashlib.sha1(p.tobytes()).hexdigest()[:16], r[-1])
