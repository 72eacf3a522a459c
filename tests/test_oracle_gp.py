"""Pins of the float64 oracle (oracle/gp.py) against things other than itself.

Each test names the pin it implements (P1..P15) and what fixes the expected value: a library
routine that computes the same mathematical object by a different algorithm, a closed form,
an invariant, brute force, or a value printed in PAPER.md / SPEC.md.
"""
import math

import mpmath
import numpy as np
import pytest
import scipy.linalg
from sklearn.gaussian_process import GaussianProcessRegressor
from sklearn.gaussian_process.kernels import RBF as SkRBF
from sklearn.gaussian_process.kernels import ConstantKernel, Matern

from oracle import gp
from workloads import gen


def _case(seed=0, n=30, d=3, m=200, clustered=False, sn2=1e-4, kernel=gp.MATERN52):
    w = gen.random_case(seed, n, d, m, kernel=kernel, sn2=sn2, clustered=clustered)
    return w.searches[0], w.Xstar[0]


# ---------------------------------------------------------------- P1: library equivalence
@pytest.mark.parametrize("kernel", [gp.MATERN52, gp.RBF])
@pytest.mark.parametrize("seed", [0, 1])
def test_p1_matches_sklearn_gpr(kernel, seed):
    """P1: sklearn GaussianProcessRegressor (LAPACK Cholesky, its own kernel code, normalize_y
    with ddof=0) at the same fixed hyper-parameters.  alpha = sn2 + jitter_0 (reading R9)."""
    s, Xs = _case(seed, n=40, d=4, m=300, kernel=kernel)
    m = gp.fit(s.X, s.y, s.lengthscale, s.sf2, s.sn2, kernel)
    assert m.jitter_k == 0
    ls = s.lengthscale.astype(np.float64)
    base = Matern(length_scale=ls, nu=2.5, length_scale_bounds="fixed") if kernel == gp.MATERN52 \
        else SkRBF(length_scale=ls, length_scale_bounds="fixed")
    k = ConstantKernel(s.sf2, constant_value_bounds="fixed") * base
    reg = GaussianProcessRegressor(kernel=k, alpha=m.sn2 + m.jitter, optimizer=None,
                                   normalize_y=True)
    reg.fit(s.X.astype(np.float64), s.y)
    mu_sk, sd_sk = reg.predict(Xs.astype(np.float64), return_std=True)
    mu, var = gp.posterior(m, Xs)
    mu_raw, var_raw = gp.raw_posterior(m, mu, var)
    np.testing.assert_allclose(mu_raw, mu_sk, rtol=0, atol=1e-9 * max(1.0, np.abs(mu_sk).max()))
    np.testing.assert_allclose(var_raw, sd_sk ** 2, rtol=0, atol=1e-9 * m.std ** 2)


def test_p1_cholesky_and_substitution_match_lapack():
    """P1: the hand-written Cholesky and substitutions against LAPACK (numpy / scipy)."""
    s, Xs = _case(3, n=60, d=5)
    K = gp.kernel_from_sq_dist(gp.sq_dist(s.X, s.X, s.lengthscale), 1.0, gp.MATERN52)
    K += 1e-4 * np.eye(60)
    L = gp.cholesky_lower(K)
    np.testing.assert_allclose(L, np.linalg.cholesky(K), rtol=0, atol=1e-12)
    B = np.random.default_rng(0).standard_normal((60, 7))
    np.testing.assert_allclose(gp.forward_sub(L, B),
                               scipy.linalg.solve_triangular(L, B, lower=True), atol=1e-9)
    np.testing.assert_allclose(gp.back_sub_transposed(L, B),
                               scipy.linalg.solve_triangular(L, B, lower=True, trans="T"),
                               atol=1e-9)


def test_dense_solve_equivalence():
    """SPEC acceptance #7: equal to a naive dense-solve GP within 1e-8."""
    s, Xs = _case(5, n=50, d=2, m=100)
    m = gp.fit(s.X, s.y, s.lengthscale, s.sf2, s.sn2)
    X = s.X.astype(np.float64)
    ls = s.lengthscale.astype(np.float64)
    K = np.empty((50, 50))
    for i in range(50):  # kernel by explicit per-pair loop (Matern-5/2 definition)
        for j in range(50):
            r = math.sqrt(np.sum(((X[i] - X[j]) / ls) ** 2))
            K[i, j] = (1 + math.sqrt(5) * r + 5 * r * r / 3) * math.exp(-math.sqrt(5) * r)
    K += (m.sn2 + m.jitter) * np.eye(50)
    for c in range(0, 100, 9):
        x = Xs[c].astype(np.float64)
        r = np.sqrt(np.sum(((X - x) / ls) ** 2, axis=1))
        ks = (1 + math.sqrt(5) * r + 5 * r * r / 3) * np.exp(-math.sqrt(5) * r)
        mu_ref = ks @ np.linalg.solve(K, m.ytilde)
        var_ref = 1.0 - ks @ np.linalg.solve(K, ks)
        mu, var = gp.posterior(m, Xs[c:c + 1])
        assert abs(mu[0] - mu_ref) < 1e-8
        assert abs(var[0] - max(var_ref, 0.0)) < 1e-8


# ---------------------------------------------------------------- P2, P3: interpolation, prior
def test_p2_interpolation():
    """P2: SPEC's example -- 20 samples of y = (x - 0.3)^2 on [0, 1] with the
    noise at the jitter floor -> mean within 1e-4 of y~ and variance <= 1e-4 at the inputs.
    Also the exact identity mu~(x_i) - y~_i = -(sn2 + j) alpha_i (K (K + eI)^-1 = I - e(K + eI)^-1)."""
    X = (np.arange(20, dtype=np.float64) / 19.0).astype(np.float32)[:, None]
    y = (X[:, 0].astype(np.float64) - 0.3) ** 2
    m = gp.fit(X, y, np.array([0.3], np.float32), 1.0, 1e-8)
    mu, var = gp.posterior(m, X)
    assert np.max(np.abs(mu - m.ytilde)) < 1e-4
    assert np.max(var) < 1e-4
    s, _ = _case(7, n=25, d=2, sn2=1e-6)
    m = gp.fit(s.X, s.y, s.lengthscale, s.sf2, s.sn2)
    mu, _ = gp.posterior(m, s.X)
    np.testing.assert_allclose(mu - m.ytilde, -(m.sn2 + m.jitter) * m.alpha, rtol=1e-6,
                               atol=1e-12)


def test_p3_prior_reversion():
    """P3: far from every observation s2~ -> sf2 and mu~ -> 0."""
    s, _ = _case(8, n=20, d=3)
    m = gp.fit(s.X, s.y, s.lengthscale * 0 + 0.05, s.sf2, s.sn2)
    far = np.full((4, 3), 50.0, dtype=np.float32)
    mu, var = gp.posterior(m, far)
    assert np.max(np.abs(mu)) < 1e-12
    assert np.max(np.abs(var - m.sf2)) < 1e-12


# ---------------------------------------------------------------- P4: n = 2 closed form
def test_p4_two_point_closed_form():
    """P4: n = 2 by the explicit 2x2 inverse [[a,-b],[-b,a]] / (a^2 - b^2)."""
    X = np.array([[0.2], [0.7]], dtype=np.float32)
    y = np.array([1.0, 3.0])
    ls = np.array([0.3], dtype=np.float32)
    m = gp.fit(X, y, ls, 1.0, 1e-3, gp.RBF)
    ls64 = float(ls[0])
    yt = np.array([-1.0, 1.0])  # (y - 2) / 1, ddof = 0
    a = 1.0 + float(np.float32(1e-3)) + 1e-8
    b = math.exp(-0.5 * ((float(X[0, 0]) - float(X[1, 0])) / ls64) ** 2)
    det = a * a - b * b
    for xs in (0.0, 0.45, 0.9):
        xs = float(np.float32(xs))
        k1 = math.exp(-0.5 * ((xs - float(X[0, 0])) / ls64) ** 2)
        k2 = math.exp(-0.5 * ((xs - float(X[1, 0])) / ls64) ** 2)
        w1 = (a * yt[0] - b * yt[1]) / det
        w2 = (-b * yt[0] + a * yt[1]) / det
        mu_ref = k1 * w1 + k2 * w2
        q = (a * k1 * k1 - 2 * b * k1 * k2 + a * k2 * k2) / det
        mu, var = gp.posterior(m, np.array([[xs]], dtype=np.float32))
        assert abs(mu[0] - mu_ref) < 1e-13
        assert abs(var[0] - (1.0 - q)) < 1e-13


# ---------------------------------------------------------------- P5, P6: EI
@pytest.mark.parametrize("z", [1.0, 0.0, -1.0, 2.0, -3.0, -6.0, -10.0, 3.5, -0.25])
def test_p5_tau_closed_form(z):
    """P5: tau(z) = phi(z) + z Phi(z) against 40-digit mpmath (tau(1) ~ 1.0833)."""
    mpmath.mp.dps = 40
    ref = mpmath.npdf(z) + z * mpmath.ncdf(z)
    got = float(gp.tau(np.array([z]))[0])
    assert abs(got - float(ref)) <= 1e-12 * float(ref)


def test_p5_spec_example():
    """mu = best - sigma (z = 1) -> EI = sigma (Phi(1) + phi(1)) ~ 1.0833 sigma."""
    ei = gp.expected_improvement(np.array([2.0 - 0.5]), np.array([0.25]), 2.0)
    assert abs(ei[0] / 0.5 - 1.0833154705876864) < 1e-12


def test_p6_ei_invariants():
    """P6: EI >= max(best - mu, 0) >= 0; increasing in sigma; decreasing in mu;
    sigma -> 0 limit; EI = 0 at sigma = 0 and mu >= best."""
    rng = np.random.default_rng(1)
    mu = rng.uniform(-3, 3, 10000)
    s = rng.uniform(0, 2, 10000)
    best = 0.3
    ei = gp.expected_improvement(mu, s * s, best)
    assert np.all(ei >= np.maximum(best - mu, 0) - 1e-15)
    ei_s = gp.expected_improvement(mu, (s * 1.1) ** 2, best)
    assert np.all(ei_s >= ei - 1e-15)
    ei_m = gp.expected_improvement(mu + 0.01, s * s, best)
    assert np.all(ei_m <= ei + 1e-15)
    tiny = gp.expected_improvement(mu, np.full_like(mu, 1e-24), best)
    np.testing.assert_allclose(tiny, np.maximum(best - mu, 0), atol=1e-11)
    z0 = gp.expected_improvement(np.array([0.3, 1.0]), np.zeros(2), best)
    assert np.all(z0 == 0.0)


# ---------------------------------------------------------------- P7: brute-force argmax
def test_p7_bruteforce_argmax_and_ties():
    """P7: argmax on a tiny grid by enumeration; a constructed exact tie resolves to the lowest
    index (S:L407 'ties -> first').  Data symmetric about 0.5 make mirror candidates tie."""
    X = np.array([[0.25], [0.75]], dtype=np.float32)  # symmetric about 0.5
    y = np.array([2.0, 2.0])
    ls = np.array([0.2], dtype=np.float32)
    m = gp.fit(X, y, ls, 1.0, 1e-4, gp.MATERN52)
    # rows 1 and 3 are the same point (exact tie); rows 1 and 4 mirror about 0.5 (near tie)
    grid = np.array([[0.5], [0.0], [0.5], [0.0], [1.0]], dtype=np.float32)
    r = gp.score(m, grid)
    mu, var = gp.posterior(m, grid)
    ei = gp.expected_improvement(mu, var, m.best)
    assert ei[1] == ei[3] and abs(ei[1] - ei[4]) < 1e-12
    best = max(range(5), key=lambda i: (ei[i], -i))  # enumeration with explicit tie rule
    assert r.idx == best
    assert r.idx in (1, 4) and r.idx != 3
    # random tiny grids: argmax equals enumeration
    for seed in range(5):
        s, Xs = _case(20 + seed, n=5, d=2, m=64)
        m = gp.fit(s.X, s.y, s.lengthscale, s.sf2, s.sn2)
        r = gp.score(m, Xs)
        e = [float(gp.score(m, Xs[i:i + 1]).ei) for i in range(64)]
        assert r.idx == max(range(64), key=lambda i: (e[i], -i))


# ---------------------------------------------------------------- P8: symmetry
def test_p8_symmetry():
    """P8: data symmetric about 0.5 -> mu(0.5 - d) = mu(0.5 + d) within 1e-8."""
    xs = np.array([0.1, 0.3, 0.45, 0.55, 0.7, 0.9], dtype=np.float32)
    X = xs[:, None]
    y = np.array([1.0, 2.0, 0.5, 0.5, 2.0, 1.0])
    m = gp.fit(X, y, np.array([0.25], dtype=np.float32), 1.0, 1e-4)
    for dlt in (0.05, 0.2, 0.37):
        a = np.array([[0.5 - dlt]], dtype=np.float32)
        b = np.array([[0.5 + dlt]], dtype=np.float32)
        (ma, va), (mb, vb) = gp.posterior(m, a), gp.posterior(m, b)
        # float32 inputs are only approximately mirrored; the tolerance covers that rounding
        assert abs(ma[0] - mb[0]) < 1e-6 and abs(va[0] - vb[0]) < 1e-6


# ---------------------------------------------------------------- P9: kernel values
def test_p9_kernel_values_at_r1():
    """P9: Matern-5/2(r=1) = (1 + sqrt5 + 5/3) e^-sqrt5 = 0.5239941088318203,
    RBF(r=1) = e^-1/2 = 0.6065306597126334 (also sklearn's kernels, printed above)."""
    assert abs(gp.kernel_from_sq_dist(1.0, 1.0, gp.MATERN52) - 0.5239941088318203) < 1e-15
    assert abs(gp.kernel_from_sq_dist(1.0, 1.0, gp.RBF) - 0.6065306597126334) < 1e-15
    for kind, sk in ((gp.MATERN52, Matern(length_scale=0.7, nu=2.5)), (gp.RBF, SkRBF(0.7))):
        A = np.random.default_rng(2).random((5, 1))
        B = np.random.default_rng(3).random((6, 1))
        got = gp.kernel_from_sq_dist(gp.sq_dist(A, B, np.array([0.7])), 1.0, kind)
        np.testing.assert_allclose(got, sk(A, B), atol=1e-15)


# ---------------------------------------------------------------- P10: degenerate y
def test_p10_degenerate_targets():
    """P10: constant y -> flagged, mu~ = 0, EI = phi(0) s~, argmax EI = argmax s2~."""
    s, Xs = _case(9, n=12, d=2, m=50)
    y = np.full(12, 4.2)
    m = gp.fit(s.X, y, s.lengthscale, s.sf2, s.sn2)
    assert m.status == gp.STATUS_WDEGENERATE and m.std == 1.0
    r = gp.score(m, Xs)
    assert np.max(np.abs(r.mu)) == 0.0
    np.testing.assert_allclose(r.ei_all, np.sqrt(r.var) / math.sqrt(2 * math.pi), rtol=1e-14)
    assert r.idx == int(np.argmax(r.var))


# ---------------------------------------------------------------- jitter escalation (R9)
def test_jitter_escalation_duplicates():
    """R9: duplicated rows with sn2 = 0 need jitter; the k chosen equals the first k at which
    LAPACK's Cholesky succeeds on the same matrix."""
    X = np.repeat(np.random.default_rng(4).random((6, 2)).astype(np.float32), 3, axis=0)
    y = np.random.default_rng(5).standard_normal(18)
    ls = np.array([0.3, 0.4], dtype=np.float32)
    m = gp.fit(X, y, ls, 1.0, 0.0, gp.RBF)
    K0 = gp.kernel_from_sq_dist(gp.sq_dist(X, X, ls), 1.0, gp.RBF)
    first = None
    for k in range(7):
        try:
            np.linalg.cholesky(K0 + 1e-8 * 10 ** k * np.eye(18))
            first = k
            break
        except np.linalg.LinAlgError:
            pass
    assert m.jitter_k == first
    assert m.status in (gp.STATUS_OK,)


def test_jitter_exhaustion_reports_enotpd():
    """R9: a matrix that no jitter of the ladder repairs -> ENOTPD."""
    X = np.zeros((3, 1), dtype=np.float32)
    m = gp.fit(X, np.array([0.0, 1.0, 2.0]), np.array([1.0], dtype=np.float32), 1.0, -1.0)
    assert m.status == gp.STATUS_ENOTPD and m.L is None


# ---------------------------------------------------------------- P14, P15
def test_p14_zero_padding_d_is_exact():
    """P14: zero columns appended to X and X* leave every output bit-identical."""
    s, Xs = _case(10, n=20, d=3, m=64)
    m = gp.fit(s.X, s.y, s.lengthscale, s.sf2, s.sn2)
    pad = lambda A: np.concatenate([A, np.zeros((A.shape[0], 2), np.float32)], 1)
    ls = np.concatenate([s.lengthscale, np.ones(2, np.float32)])
    m2 = gp.fit(pad(s.X), s.y, ls, s.sf2, s.sn2)
    a, b = gp.score(m, Xs), gp.score(m2, pad(Xs))
    assert np.array_equal(a.ei_all, b.ei_all) and a.idx == b.idx


def test_p15_permutations():
    """P15: permuting training rows changes mu, var only within rounding; permuting candidates
    permutes EI."""
    s, Xs = _case(11, n=30, d=4, m=80)
    m = gp.fit(s.X, s.y, s.lengthscale, s.sf2, s.sn2)
    p = np.random.default_rng(6).permutation(30)
    mp = gp.fit(s.X[p], s.y[p], s.lengthscale, s.sf2, s.sn2)
    (mu, var), (mu2, var2) = gp.posterior(m, Xs), gp.posterior(mp, Xs)
    np.testing.assert_allclose(mu2, mu, atol=1e-9)
    np.testing.assert_allclose(var2, var, atol=1e-9)
    q = np.random.default_rng(7).permutation(80)
    a, b = gp.score(m, Xs), gp.score(m, Xs[q])
    np.testing.assert_allclose(b.ei_all, a.ei_all[q], rtol=0, atol=0)
