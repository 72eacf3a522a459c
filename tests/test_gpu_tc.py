"""tcgen05 building blocks: swizzled K-major operand layouts, UMMA descriptors, k-advance inside
a swizzle row, B-operand row offsets, TMEM loads -- exact fp16 -> fp32 GEMMs."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("row_bytes,K,N,off", [
    (32, 16, 16, 0), (32, 32, 64, 8), (32, 64, 112, 16), (64, 32, 32, 0), (64, 32, 128, 0),
    (64, 64, 208, 16), (64, 32, 256, 0), (128, 64, 256, 0), (128, 128, 96, 24)])
def test_tc_gemm_exact(row_bytes, K, N, off):
    import torch
    from paper_2403_08131_b200 import gpbo
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rng = np.random.default_rng(K * 1000 + N + off)
    A = (rng.integers(-128, 129, (128, K)) / 64.0).astype(np.float16)
    B = (rng.integers(-128, 129, (N, K)) / 64.0).astype(np.float16)
    D = gpbo.tc_selftest(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), row_bytes, off)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    np.testing.assert_array_equal(D.cpu().numpy().astype(np.float64), ref)
