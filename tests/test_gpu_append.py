"""GPU: §8(f)2 O(n^2) append update (gp_fit_append) against a full refactorisation.

Pins: the appended model equals the oracle's full fit of the n + 1 observations (L, L^-1, alpha,
LML, mean / std / best, the jitter k) to the same float64 tolerances as a fresh gp_fit
(tests/test_gpu_parity.py::test_fit_matches_oracle); a chain of appends (the config-5 replay's
use) stays within them; scoring the appended model gives the fresh model's suggestion."""
import numpy as np
import pytest

from oracle import gp
from oracle import ml2
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


def _check_against_oracle(m, s, X, y, ls, sf2, sn2, kernel, label):
    om = gp.fit(X, y, ls, sf2, sn2, kernel)
    assert m.jitter_k[s] == om.jitter_k, label
    L, Li, a = m.export(s)
    st = m.stats(s)
    assert abs(st["mean"] - om.mean) <= 1e-12 * max(1, abs(om.mean)), label
    assert abs(st["std"] - om.std) <= 1e-12 * om.std, label
    assert abs(st["best"] - om.best) <= 1e-12 * max(1, abs(om.best)), label
    np.testing.assert_allclose(L, om.L, rtol=0, atol=1e-12 * np.abs(om.L).max(), err_msg=label)
    Li_ref = np.linalg.inv(om.L)
    np.testing.assert_allclose(Li, Li_ref, rtol=0, atol=1e-9 * np.abs(Li_ref).max(), err_msg=label)
    np.testing.assert_allclose(a, om.alpha, rtol=0, atol=1e-7 * np.abs(om.alpha).max(), err_msg=label)
    ref = ml2.lml(om)
    assert abs(m.lml()[s] - ref) <= 1e-9 * abs(ref), (label, m.lml()[s], ref)


@pytest.mark.parametrize("n,d,kernel", [(1, 2, gp.MATERN52), (20, 2, gp.MATERN52),
                                        (199, 20, gp.MATERN52), (216, 6, gp.RBF),
                                        (300, 35, gp.MATERN52), (499, 60, gp.RBF)])
def test_append_equals_full_refit(G, n, d, kernel):
    gpbo, ctx = G
    w = gen.random_case(n + 3 * d, n + 1, d, 4, kernel=kernel)
    s = w.searches[0]
    m0 = ctx.fit([n], [d], np.ascontiguousarray(s.X[:n].ravel()), s.y[:n].copy(), s.lengthscale,
                 np.ones(1, np.float32), np.full(1, s.sn2, np.float32), kernel=kernel)
    m1 = ctx.fit_append(m0, np.ascontiguousarray(s.X[n]), s.y[n:n + 1].copy())
    assert ctx.last_append_refit == 0 and list(m1.n) == [n + 1]
    _check_against_oracle(m1, 0, s.X, s.y, s.lengthscale, 1.0, s.sn2, kernel, f"append n={n}")
    m0.free()
    m1.free()


def test_append_chain_batch_and_scoring(G):
    """Three searches grown by 40 appends each (from n = 5): still equal to the full refit, and
    the suggestion on 2^15 candidates equals the fresh model's and the oracle's (R11)."""
    gpbo, ctx = G
    w = gen.random_case(77, [45, 45, 45], [3, 8, 20], [1 << 15] * 3, S=3)
    n0 = 5
    n, d, X, y, ls, sf2, sn2 = H.pack(w)
    cut = lambda k: (np.concatenate([s.X[:k].ravel() for s in w.searches]).astype(np.float32),
                     np.concatenate([s.y[:k] for s in w.searches]))
    X0, y0 = cut(n0)
    m = ctx.fit([n0] * 3, d, X0, y0, ls, sf2, sn2, kernel=w.kernel)
    for k in range(n0, 45):
        xn = np.concatenate([s.X[k] for s in w.searches]).astype(np.float32)
        yn = np.array([s.y[k] for s in w.searches])
        m2 = ctx.fit_append(m, xn, yn)
        m.free()
        m = m2
    assert list(m.n) == [45] * 3
    for s, q in enumerate(w.searches):
        _check_against_oracle(m, s, q.X, q.y, q.lengthscale, q.sf2, q.sn2, w.kernel, f"chain[{s}]")
    fresh = ctx.fit(n, d, X, y, ls, sf2, sn2, kernel=w.kernel)
    Xs, off = H.pack_candidates(w)
    i1, e1 = ctx.score_argmax(m, Xs, off)
    i2, e2 = ctx.score_argmax(fresh, Xs, off)
    assert np.array_equal(i1, i2)
    for s, om in enumerate(H.oracle_fits(w)):
        H.check_argmax(gp.score(om, w.Xstar[s]), int(i1[s]), f"chain-argmax[{s}]")
    m.free()
    fresh.free()


def test_append_device_inputs_and_errors(G):
    import torch
    gpbo, ctx = G
    w = gen.random_case(78, 31, 4, 4)
    s = w.searches[0]
    m0 = ctx.fit([30], [4], np.ascontiguousarray(s.X[:30].ravel()), s.y[:30].copy(),
                 s.lengthscale, np.ones(1, np.float32), np.full(1, s.sn2, np.float32))
    xd = torch.from_numpy(np.ascontiguousarray(s.X[30])).cuda()
    yd = torch.from_numpy(s.y[30:31].copy()).cuda()
    m1 = ctx.fit_append(m0, xd, yd)
    _check_against_oracle(m1, 0, s.X, s.y, s.lengthscale, 1.0, s.sn2, w.kernel, "device")
    with pytest.raises(gpbo.GpboError) as e:
        ctx.fit_append(m0, np.full(4, np.nan, np.float32), np.zeros(1))
    assert e.value.status == gpbo.EINVAL
    m0.free()
    m1.free()
