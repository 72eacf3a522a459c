"""GPU: gp_posterior's dense float64 path (refine.cu posterior64_kernel: K* from float64 GEMM-form
distances and V^T = L^-1 K*^T on the FP64 tensor cores) against the oracle, element by element.

Edges of that kernel: the 8-warp / 16-warp variants (n8 <= 256 / > 256), ragged 32-candidate
tiles, a single candidate, candidates ON the training points of a noise-free fit (the GEMM-form
distance's cancellation error is the largest there -- reading R1 / DESIGN.md §6.5: T1's variance
term is relative to sf2), the RBF kernel, and a NaN row.  Tolerances: tests/helpers.py (T1)."""
import numpy as np
import pytest

from oracle import gp
from tests import helpers as H
from workloads import gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2403_08131_b200 import gpbo
    ctx = gpbo.Context(device=0)
    yield gpbo, ctx
    ctx.close()


def _posterior_vs_oracle(G, w, label, Xs=None):
    gpbo, ctx = G
    m = ctx.fit(*H.pack(w), kernel=w.kernel)
    om = H.oracle_fits(w)[0]
    Xs = w.Xstar[0] if Xs is None else Xs
    mu, var, ei = ctx.posterior(m, 0, np.ascontiguousarray(Xs, np.float32))
    assert ctx.last_impl == 5, (label, ctx.last_impl)
    res = gp.score(om, Xs)
    worst = H.check_T1(om, res, mu, var, ei, label)
    m.free()
    return om, res, (mu, var, ei), worst


# n = 256: the last 8-warp shape (n8 = 256); 257: the first 16-warp one; ragged M
@pytest.mark.parametrize("n,d,M", [(65, 3, 33), (120, 7, 95), (256, 20, 1025), (257, 20, 777),
                                   (333, 64, 161), (512, 9, 300)])
def test_posterior_shapes(G, n, d, M):
    w = gen.random_case(31, n, d, M)
    _posterior_vs_oracle(G, w, f"n{n}_d{d}_M{M}")


@pytest.mark.parametrize("kernel", [gp.MATERN52, gp.RBF])
def test_posterior_at_training_points_noise_free(G, kernel):
    """sn2 = 0: at the training points the posterior mean interpolates y and the variance is
    ~ the jitter (closed form of the GP posterior; the oracle pins it, tests/test_oracle_gp.py).
    The GPU's GEMM-form distances are not exactly 0 there; T1 must still hold element-wise."""
    w = gen.random_case(32, 150, 6, 1, kernel=kernel, sn2=0.0)
    s = w.searches[0]
    Xs = np.concatenate([s.X, w.Xstar[0]])
    om, res, (mu, var, ei), _ = _posterior_vs_oracle(G, w, f"interp_k{kernel}", Xs)
    n = s.X.shape[0]
    # interpolation up to the jitter actually used: |mu_i - y_i| = (sn2 + j) |alpha_i| std and
    # var_i <= sn2 + j (standardised), with float32 output rounding
    a = np.abs(om.alpha) * om.jitter * om.std
    assert np.all(np.abs(mu[:n].astype(np.float64) - s.y) <= 10 * a + 1e-5 * (np.abs(s.y) + om.std))
    assert np.max(var[:n]) <= (om.jitter + 1e-4 * om.sf2) * om.std ** 2


def test_posterior_single_candidate_and_nan_row(G):
    gpbo, ctx = G
    w = gen.random_case(33, 180, 12, 64)
    m = ctx.fit(*H.pack(w), kernel=w.kernel)
    om = H.oracle_fits(w)[0]
    one = np.ascontiguousarray(w.Xstar[0][:1])
    mu, var, ei = ctx.posterior(m, 0, one)
    assert ctx.last_impl == 5
    H.check_T1(om, gp.score(om, one), mu, var, ei, "M1")
    Xs = w.Xstar[0].copy()
    Xs[17, 3] = np.nan
    mu, var, ei = ctx.posterior(m, 0, np.ascontiguousarray(Xs))
    assert np.isnan(mu[17]) and np.isnan(var[17]) and np.isnan(ei[17])
    keep = np.arange(64) != 17
    H.check_T1(om, gp.score(om, w.Xstar[0][keep]), mu[keep], var[keep], ei[keep], "nan-row")
    m.free()


def test_posterior_is_deterministic(G):
    """Fixed-order reductions: two calls give bit-identical outputs."""
    gpbo, ctx = G
    w = gen.random_case(34, 300, 20, 2048)
    m = ctx.fit(*H.pack(w), kernel=w.kernel)
    a = ctx.posterior(m, 0, w.Xstar[0])
    b = ctx.posterior(m, 0, w.Xstar[0])
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    m.free()


@pytest.mark.parametrize("cfg", [2, 4])
def test_posterior_full_shape_sampled(G, cfg):
    """gp_posterior at the bench's shapes (config 2: 2^20 candidates, the posterior pass of
    bench.py; config 4: 2^18 of the n = 500, d = 60 search -- the 16-warp variant): T1 on 4,096
    sampled rows the oracle computes one by one, and every row finite."""
    gpbo, ctx = G
    w = gen.make(cfg, M=(1 << 20) if cfg == 2 else (1 << 18))
    m = ctx.fit(*H.pack(w), kernel=w.kernel)
    om = H.oracle_fits(w)[0]
    X = w.Xstar[0]
    mu, var, ei = ctx.posterior(m, 0, X)
    assert ctx.last_impl == 5
    assert np.all(np.isfinite(mu)) and np.all(np.isfinite(var)) and np.all(np.isfinite(ei))
    smp = np.sort(np.random.default_rng(cfg).choice(X.shape[0], 4096, replace=False))
    res = gp.score(om, X[smp])
    # T1's EI term is relative to the maximum EI; over a sample use the sample's maximum
    H.check_T1(om, res, mu[smp], var[smp], ei[smp], f"cfg{cfg}-sampled")
    m.free()
