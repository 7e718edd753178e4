"""Pins the tcgen05 operand/descriptor convention (csrc/umma.cuh) against numpy: every major
combination the fused learn kernels use, M=128 and M=64 (incl. the interleaved second M=64
accumulator at TMEM lane 16), K up to 128, N 16..64. Operands are bf16, accumulation f32."""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _bf16(x):
    return torch.tensor(x, dtype=torch.float32).to(torch.bfloat16).to(torch.float32).numpy().astype(np.float64)


CASES = [
    # M, N, K, a_mn, b_mn, lane_off
    (128, 64, 64, 0, 0, 0),
    (128, 64, 64, 0, 1, 0),
    (128, 16, 64, 0, 0, 0),
    (128, 64, 16, 0, 1, 0),
    (128, 64, 32, 1, 0, 0),
    (64, 64, 128, 1, 1, 0),
    (64, 64, 128, 1, 1, 16),
    (64, 16, 128, 1, 1, 0),
    (128, 32, 48, 0, 0, 0),
]


@pytest.mark.parametrize("case", CASES, ids=[f"M{c[0]}N{c[1]}K{c[2]}a{c[3]}b{c[4]}l{c[5]}" for c in CASES])
def test_umma_matches_numpy(case):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2210_00882_b200 import _native as N

    M, Nn, K, a_mn, b_mn, lane_off = case
    rng = np.random.default_rng(hash(case) % 2**32)
    A = rng.uniform(-1, 1, size=(K, M) if a_mn else (M, K)).astype(np.float32)
    B = rng.uniform(-1, 1, size=(K, Nn) if b_mn else (Nn, K)).astype(np.float32)
    D = np.zeros((M, Nn), dtype=np.float32)
    fp = C.POINTER(C.c_float)
    N.check(N.lib().flw_selftest_umma(M, Nn, K, a_mn, b_mn, lane_off, A.ctypes.data_as(fp), B.ctypes.data_as(fp),
                                      D.ctypes.data_as(fp)))
    Aop = _bf16(A).T if a_mn else _bf16(A)
    Bop = _bf16(B) if b_mn else _bf16(B).T
    want = Aop @ Bop
    np.testing.assert_allclose(D, want, rtol=1e-5, atol=1e-4)
