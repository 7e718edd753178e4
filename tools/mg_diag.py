"""Diagnose single-process multi-GPU run_local (k units on k GPUs)."""
import json, os, sys
if os.environ.get("DIAG_TORCH"):
    import torch  # noqa: F401  (loads the torch-bundled libnccl first)
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_00882_b200 import Program

z = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "run_dpd_k2_synth.npz"))
algo = json.loads(str(z["__algo__"]))
num = sys.argv[1] if len(sys.argv) > 1 else "exact"
prog = Program(algo, {"workers": ["local"], "slots_per_worker": {"cpu": 16, "accel": 16},
                      "distribution_policy": "dp-d", "numerics": num})
csv, s = prog.run_local(seed=int(z["__seed__"]))
print(csv.splitlines()[-1], flush=True)
