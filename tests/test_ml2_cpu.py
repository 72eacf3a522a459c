"""§8(f)1 ML-II on the CPU: pins of the oracle (oracle/ml2.py) and of the library's host-side
Nelder-Mead (through the host-only hook gpbo_nm_selftest; no GPU needed).

* LML vs sklearn's GaussianProcessRegressor.log_marginal_likelihood (LAPACK Cholesky, its own
  kernel code; normalize_y = True uses the same ddof-0 standardisation) to 1e-10 relative.
* splitmix64 vs its published reference outputs (seed 0: e220a8397b1dcdaf, 6e789e6aa1b965f4).
* The oracle's Nelder-Mead vs scipy.optimize.minimize(method="Nelder-Mead") given the same
  initial simplex, bounds (clipping) and iteration count: the same algorithm, independently
  implemented -> the same iterates.
* The library's Nelder-Mead state machine vs the oracle's on the same objectives: identical
  best point and evaluation count.
* SPEC.md L369 invariant on the oracle's ML-II: LML of the result >= LML of every start.
"""
import math

import numpy as np
import pytest
import scipy.optimize
from sklearn.gaussian_process import GaussianProcessRegressor
from sklearn.gaussian_process.kernels import RBF as SkRBF
from sklearn.gaussian_process.kernels import ConstantKernel, Matern

from oracle import gp
from oracle import ml2
from workloads import gen


@pytest.mark.parametrize("kernel", [gp.MATERN52, gp.RBF])
@pytest.mark.parametrize("seed,n,d", [(0, 30, 3), (1, 80, 6), (2, 12, 1)])
def test_lml_matches_sklearn(kernel, seed, n, d):
    w = gen.random_case(seed, n, d, 4, kernel=kernel, sn2=1e-3)
    s = w.searches[0]
    m = gp.fit(s.X, s.y, s.lengthscale, s.sf2, s.sn2, kernel)
    assert m.jitter_k == 0
    ls = s.lengthscale.astype(np.float64)
    base = (Matern(length_scale=ls, length_scale_bounds="fixed", nu=2.5) if kernel == gp.MATERN52
            else SkRBF(length_scale=ls, length_scale_bounds="fixed"))
    k = ConstantKernel(float(s.sf2), constant_value_bounds="fixed") * base
    # the fit adds the jitter ladder's j_0 = 1e-8 sf2 on top of sn2 (reading R9)
    g = GaussianProcessRegressor(kernel=k, alpha=float(np.float32(s.sn2)) + 1e-8 * float(s.sf2),
                                 optimizer=None, normalize_y=True)
    g.fit(s.X.astype(np.float64), s.y)
    ref = g.log_marginal_likelihood_value_
    assert abs(ml2.lml(m) - ref) <= 1e-10 * abs(ref), (ml2.lml(m), ref)


def test_splitmix64_reference_outputs():
    g = 0x9E3779B97F4A7C15
    assert ml2.splitmix64(g) == 0xE220A8397B1DCDAF
    assert ml2.splitmix64((2 * g) & ml2.MASK64) == 0x6E789E6AA1B965F4
    assert ml2.splitmix64((3 * g) & ml2.MASK64) == 0x06C45D188009454F


def _rosen(x):
    return float(np.sum(100.0 * (x[1:] - x[:-1] ** 2) ** 2 + (1 - x[:-1]) ** 2))


def _quartic(x):
    return float(np.sum((x - 0.3) ** 4 + 0.1 * np.sin(3 * x)) + 0.5 * x[0] * x[-1])


@pytest.mark.parametrize("fun,dim", [(_rosen, 4), (_quartic, 6), (_rosen, 2)])
def test_oracle_nelder_mead_matches_scipy(fun, dim):
    lo, hi = np.full(dim, -2.0), np.full(dim, 1.5)
    x0 = np.linspace(-1.2, 1.1, dim)
    iters = 150
    xb, fb, f0, nev = ml2.nelder_mead(fun, x0, lo, hi, step=0.5, iters=iters)
    sim = [x0.copy()]
    for i in range(dim):
        v = x0.copy()
        v[i] = v[i] + 0.5 if v[i] + 0.5 <= hi[i] else v[i] - 0.5
        sim.append(v)
    r = scipy.optimize.minimize(fun, x0, method="Nelder-Mead", bounds=list(zip(lo, hi)),
                                # scipy counts the initial simplex as iteration 1
                                options=dict(initial_simplex=np.array(sim), maxiter=iters + 1,
                                             maxfev=10 ** 6, xatol=-1.0, fatol=-1.0,
                                             adaptive=False))
    assert r.nit == iters + 1
    assert np.array_equal(xb, r.x) and fb == r.fun, (xb, r.x, fb, r.fun)
    assert nev == r.nfev


@pytest.mark.parametrize("fun,dim", [(_rosen, 4), (_quartic, 6), (_rosen, 2)])
def test_library_nelder_mead_matches_oracle(fun, dim):
    from paper_2403_08131_b200 import gpbo
    lo, hi = np.full(dim, -2.0), np.full(dim, 1.5)
    x0 = np.linspace(-1.2, 1.1, dim)
    xb, fb, f0, nev = ml2.nelder_mead(fun, x0, lo, hi, step=0.5, iters=150)
    gx, gf, gf0, gnev = gpbo.nm_selftest(fun, x0, lo, hi, step=0.5, iters=150)
    assert np.array_equal(xb, gx) and fb == gf and f0 == gf0 and nev == gnev


def test_oracle_ml2_invariant_and_bounds():
    w = gen.random_case(3, 25, 2, 4, sn2=1e-2)
    s = w.searches[0]
    r = ml2.fit_ml2(s.X, s.y, s.lengthscale, s.sf2, s.sn2, starts=4, iters=40, seed=11)
    assert np.all(r["lml"] >= r["lml_starts"])
    assert np.all((r["ls"] >= np.float32(1e-3)) & (r["ls"] <= np.float32(10.0)))
    assert 1e-3 <= float(r["sf2"]) <= 1e3 and 1e-6 <= float(r["sn2"]) <= 1.0
    # the optimum improves on the given theta
    m0 = gp.fit(s.X, s.y, s.lengthscale, s.sf2, s.sn2)
    assert r["lml"] > ml2.lml(m0)
    # and its LML is reproduced by a plain refit at the returned theta
    m = gp.fit(s.X, s.y, r["ls"], float(r["sf2"]), float(r["sn2"]))
    assert math.isclose(ml2.lml(m), r["lml"], rel_tol=0, abs_tol=1e-12 * abs(r["lml"]))
