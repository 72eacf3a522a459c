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


@pytest.mark.parametrize("row_bytes,K,N,off", [(64, 32, 208, 0), (64, 32, 96, 16), (32, 16, 64, 0)])
def test_tc_gemm_a_from_tmem_exact(row_bytes, K, N, off):
    """A operand staged in TMEM (thread = row, k = 2c / 2c+1 in column c) and read by the MMA
    from TMEM ("TS" form) -- the layout the scoring kernel's K* operand uses."""
    import ctypes
    import torch
    from paper_2403_08131_b200 import gpbo
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rng = np.random.default_rng(K * 7 + N + off)
    A = (rng.integers(-128, 129, (128, K)) / 64.0).astype(np.float16)
    B = (rng.integers(-128, 129, (N, K)) / 64.0).astype(np.float16)
    At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    D = torch.empty(128, N, dtype=torch.float32, device="cuda")
    cyc = (ctypes.c_longlong * 2)()
    st = gpbo.load().gpbo_tc_bench(At.data_ptr(), Bt.data_ptr(), D.data_ptr(), N, K, row_bytes,
                                   off, -1, cyc)
    assert st == 0
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    np.testing.assert_array_equal(D.cpu().numpy().astype(np.float64), ref)
