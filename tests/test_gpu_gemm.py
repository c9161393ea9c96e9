"""Kernel unit tests of the GEMM engines through chg_debug_gemm (include/chg.h) against a float64
product of the same fp32 operands: the row GEMM out = A·W and the weight-gradient GEMM
out = Aᵀ·D, on the fp32 CUDA cores (engine 0), tcgen05 3xTF32 (engine 1, split operands, the
strict mode) and tcgen05 TF32 (engine 2).  Shapes span several 128-row tiles with a ragged
tail, the K / N of every GatedMLP call site (64..256), and the 3xTF32 column-group and K splits.

Bars (relative Frobenius error vs the fp64 product): fp32 and 3xTF32 1e-5 (fp32 rounding of
K-term sums), TF32 2e-3 (10-bit mantissa operands)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2412_20796_b200 import chg  # noqa: E402

BARS = {0: 1e-5, 1: 1e-5, 2: 2e-3, 3: 5e-3}


@pytest.fixture(scope="module")
def ctx():
    c = chg.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("engine", [0, 1, 2, 3])
@pytest.mark.parametrize("M,K,N", [(1000, 64, 128), (130, 192, 128), (4097, 256, 256), (1, 64, 64), (777, 128, 192),
                                   (777, 256, 64), (1000, 512, 64), (9000, 256, 64)])
def test_row_gemm(ctx, engine, M, K, N):
    rng = np.random.default_rng(M + K + N)
    A = rng.normal(size=(M, K)).astype(np.float32)
    W = (rng.normal(size=(K, N)) / np.sqrt(K)).astype(np.float32)
    out = ctx.debug_gemm(0, engine, A, W)
    ref = A.astype(np.float64) @ W.astype(np.float64)
    rel = np.linalg.norm(out - ref) / np.linalg.norm(ref)
    assert rel <= BARS[engine], rel
    if engine == 1:   # 3xTF32 must be much better than plain TF32 rounding (2^-11 ~ 5e-4)
        assert rel <= 1e-6 * np.sqrt(K), rel


@pytest.mark.parametrize("engine", [0, 1, 2, 3])
@pytest.mark.parametrize("M,K,N", [(1000, 64, 64), (5003, 192, 128), (20000, 256, 256), (33, 128, 128)])
def test_weight_gradient_gemm(ctx, engine, M, K, N):
    rng = np.random.default_rng(7 * M + K + N)
    A = rng.normal(size=(M, K)).astype(np.float32)
    D = rng.normal(size=(M, N)).astype(np.float32)
    out = ctx.debug_gemm(1, engine, A, D)
    ref = A.astype(np.float64).T @ D.astype(np.float64)
    rel = np.linalg.norm(out - ref) / np.linalg.norm(ref)
    assert rel <= BARS[engine], rel
