"""Times the generic tcgen05 GEMM (flw_bench_tgemm) on the shapes of the layer-wise path and the
split-GEMM rollout; prints ms, TFLOP/s and the operand/output traffic rate."""
import ctypes as C
import sys

sys.path.insert(0, ".")
from paper_2210_00882_b200 import _native as N

CASES = [  # (name, M, N, K, dt, mode, bn)
    ("fwd H256 bf16 bias+tanh", 135168, 256, 256, 0, 1, 256),
    ("fwd H256 bf16 f32 store", 135168, 256, 256, 0, 0, 256),
    ("fwd H64 bf16 bias+tanh (MAPPO n=64 rows)", 4194304, 64, 64, 0, 1, 64),
    ("rollout split f16 K=576 (n=64 layer 0)", 131072, 64, 576, 1, 4, 64),
    ("rollout split f16 K=192", 131072, 64, 192, 1, 4, 64),
    ("rollout split f16 K=192 f32 store", 131072, 64, 192, 1, 0, 64),
    ("square 8192 bf16 f32 store", 8192, 8192, 8192, 0, 0, 256),
]
for name, M, Nn, K, dt, mode, bn in CASES:
    ms = C.c_double()
    rc = N.lib().flw_bench_tgemm(M, Nn, K, dt, mode, bn, 10, C.byref(ms))
    esz = 2
    outb = {0: 4, 1: 2, 4: 6}[mode]
    traffic = M * K * esz + M * Nn * outb
    print(f"{name:45s} rc={rc} {ms.value*1e3:9.1f} us  {2*M*Nn*K/ms.value/1e9:8.1f} TFLOP/s  {traffic/ms.value/1e6:7.0f} GB/s")
