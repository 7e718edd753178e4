"""The generic TMA + tcgen05 GEMM of the layer-wise learn path (kernels_tgemm.cu) against a
float64 numpy product of the same (bf16-rounded / f32) operands, over every operand-major
combination, the three N tiles, ragged shapes (TMA zero fill) and split-K.

The layer-wise path computes the reference's matmul / matmul_grad_lhs / matmul_grad_rhs
(ops.cpp:75-106, 213-240) as these GEMMs: Z = H W (A K-major, B MN-major), dH = dZ W^T (A K-major,
B K-major), dW = H^T dZ (A MN-major, B MN-major).
"""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _bf16(x):
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)  # round to nearest even
    return r.view(np.float32).astype(np.float64)


def _run(M, N, K, a_mn, b_mn, tf32, splits, bn, seed=0):
    from paper_2210_00882_b200 import _native as Nt

    rng = np.random.default_rng(seed)
    A = rng.uniform(-1, 1, (K, M) if a_mn else (M, K)).astype(np.float32)
    B = rng.uniform(-1, 1, (K, N) if b_mn else (N, K)).astype(np.float32)
    D = np.zeros((M, N), dtype=np.float32)
    fp = C.POINTER(C.c_float)
    rc = Nt.lib().flw_selftest_tgemm(M, N, K, a_mn, b_mn, tf32, splits, bn, A.ctypes.data_as(fp),
                                     B.ctypes.data_as(fp), D.ctypes.data_as(fp))
    assert rc == 0
    Am = A.T if a_mn else A
    Bm = B if b_mn else B.T
    if tf32 == 1:
        want = Am.astype(np.float64) @ Bm.astype(np.float64)
        tol = 2e-3  # tf32 operands (10-bit mantissa)
    elif tf32 == 2:
        want = Am.astype(np.float16).astype(np.float64) @ Bm.astype(np.float16).astype(np.float64)
        tol = 1e-5  # exact f16 products, f32 accumulation
    else:
        want = _bf16(Am) @ _bf16(Bm)
        tol = 1e-5  # exact bf16 products, f32 accumulation
    err = np.abs(D - want).max() / max(np.abs(want).max(), 1e-30)
    return err, tol


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("a_mn", [0, 1])
@pytest.mark.parametrize("b_mn", [0, 1])
@pytest.mark.parametrize("tf32", [0, 1, 2])  # bf16, tf32, f16
def test_tgemm_majors(a_mn, b_mn, tf32):
    _need_gpu()
    if tf32 == 1 and (a_mn or b_mn):
        pytest.skip("tf32 operands are K-major only (32-bit MN-major needs the BASE32B swizzle)")
    for (M, N, K, bn, splits) in [(128, 64, 64, 64, 1), (256, 128, 192, 128, 1), (300, 200, 130, 256, 1),
                                  (130, 70, 1000, 64, 3)]:
        err, tol = _run(M, N, K, a_mn, b_mn, tf32, splits, bn)
        assert err <= tol, (M, N, K, bn, splits, err)


def test_tgemm_weight_grad_shape():
    """dW = H^T dZ at the layer-wise path's H=256 shape: K = 16384 rows split 16 ways."""
    _need_gpu()
    err, tol = _run(256, 256, 16384, 1, 1, 0, 16, 256)
    assert err <= tol, err


@pytest.mark.parametrize("a_mn,b_mn,bn", [(0, 1, 256), (0, 0, 128), (0, 1, 64)])
def test_tgemm_b_resident(a_mn, b_mn, bn):
    """More 128-row tiles than SMs, one N tile, no split-K: B loads once per CTA into shared
    memory and the ring streams A only (the layer-wise forward / dH GEMMs)."""
    _need_gpu()
    err, tol = _run(128 * 160 + 5, bn if bn < 256 else 200, 256, a_mn, b_mn, 0, 1, bn, seed=3)
    assert err <= tol, err
