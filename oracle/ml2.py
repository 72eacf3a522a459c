"""Oracle of §8(f)1 ML-II hyper-parameter fitting -- TEST INFRASTRUCTURE ONLY (same rules as
oracle/gp.py: only tests/, smoke() and bench.py's CPU legs may import it; no code is shared with
the CUDA path).

* Log marginal likelihood of the standardised targets (Rasmussen & Williams eq. 2.30), from the
  oracle's own fit (hand-written Cholesky with the jitter ladder of reading R9):
      log p(y~ | X, theta) = -1/2 y~^T alpha - sum_i log L_ii - n/2 log 2 pi
* Multi-start Nelder-Mead in log space ("Nelder-Mead in log-space from 8 seeded
  starts, 200 iterations each; bounds lengthscale in [1e-3, 10], signal in [1e-3, 1e3], noise in
  [1e-6, 1]"), maximising the LML; PAPER.md L249 names this GP training as the O(N^3) cost.
  The Nelder-Mead step is the textbook one (Nelder & Mead 1965): reflection 1, expansion 2,
  contraction 1/2, shrink 1/2, vertices ordered by f with a stable sort, points clipped to the
  box, exactly `iters` iterations.  Start 0 is the given theta; starts 1.. are uniform in the log
  box from the counter-based generator documented in include/gpbo.h (splitmix64).
"""
from __future__ import annotations

import math

import numpy as np

from oracle import gp

MASK64 = (1 << 64) - 1
LOG_2PI = math.log(2.0 * math.pi)


def lml(model: gp.GpModel) -> float:
    """Log marginal likelihood of a fitted oracle model (-inf if the factorisation failed)."""
    if model.L is None:
        return -math.inf
    n = model.X.shape[0]
    return float(-0.5 * model.ytilde @ model.alpha - np.sum(np.log(np.diag(model.L)))
                 - 0.5 * n * LOG_2PI)


def splitmix64(z):
    z &= MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def uniform(seed, s, k, i, dim, starts):
    c = 1 + i + dim * (k + starts * s)
    return (splitmix64((seed + 0x9E3779B97F4A7C15 * c) & MASK64) >> 11) * 2.0 ** -53


def nelder_mead(f, x0, lo, hi, step=0.5, iters=200):
    """Minimise f over the box [lo, hi] from x0 (textbook Nelder-Mead, see the module header).
    Returns (best x, best f, f(x0), number of evaluations)."""
    x0 = np.minimum(np.maximum(np.asarray(x0, np.float64), lo), hi)
    N = x0.size
    sim = [x0.copy()]
    for i in range(N):
        v = x0.copy()
        v[i] = v[i] + step if v[i] + step <= hi[i] else v[i] - step
        sim.append(np.minimum(np.maximum(v, lo), hi))
    fs = [f(v) for v in sim]
    nev = N + 1
    f0 = fs[0]
    order = sorted(range(N + 1), key=lambda j: fs[j])
    clip = lambda v: np.minimum(np.maximum(v, lo), hi)
    for _ in range(iters):
        w = order[N]
        xbar = np.zeros(N)
        for j in order[:N]:
            xbar += sim[j]
        xbar /= N
        xr = clip(2.0 * xbar - sim[w])                  # (1 + rho) xbar - rho x_w
        fr = f(xr)
        nev += 1
        fb, fsw, fw = fs[order[0]], fs[order[N - 1]], fs[w]
        new = None
        if fb <= fr < fsw:
            new = (xr, fr)
        elif fr < fb:
            xe = clip(3.0 * xbar - 2.0 * sim[w])        # (1 + rho chi) xbar - rho chi x_w
            fe = f(xe)
            nev += 1
            new = (xe, fe) if fe < fr else (xr, fr)
        else:
            if fr < fw:
                xc = clip(1.5 * xbar - 0.5 * sim[w])    # (1 + psi rho) xbar - psi rho x_w
                fc = f(xc)
                nev += 1
                if fc <= fr:
                    new = (xc, fc)
            else:
                xc = 0.5 * xbar + 0.5 * sim[w]          # (1 - psi) xbar + psi x_w
                fc = f(xc)
                nev += 1
                if fc < fw:
                    new = (xc, fc)
            if new is None:  # shrink towards the best vertex
                b = order[0]
                for j in order[1:]:
                    sim[j] = sim[b] + 0.5 * (sim[j] - sim[b])
                for j in order[1:]:
                    fs[j] = f(sim[j])
                    nev += 1
        if new is not None:
            sim[w], fs[w] = new
        order = sorted(order, key=lambda j: fs[j])
    b = order[0]
    return sim[b], fs[b], f0, nev


def fit_ml2(X, y, lengthscale, sf2, sn2, kind=gp.MATERN52, starts=8, iters=200, seed=0,
            step=0.5, bounds=((1e-3, 10.0), (1e-3, 1e3), (1e-6, 1.0)), search=0):
    """ML-II for one search (index `search` of the batch, for the start generator).  Returns
    dict(ls, sf2, sn2 (float32), lml, lml_starts)."""
    X = np.asarray(X, np.float32)
    d = X.shape[1]
    dim = d + 2
    (l0, l1), (f0, f1), (s0, s1) = bounds
    lo = np.array([math.log(l0)] * d + [math.log(f0), math.log(s0)])
    hi = np.array([math.log(l1)] * d + [math.log(f1), math.log(s1)])

    def theta(x):
        ls = np.exp(x[:d]).astype(np.float32)
        return ls, np.float32(math.exp(x[d])), np.float32(math.exp(x[d + 1]))

    def negl(x):
        ls, a, b = theta(x)
        v = lml(gp.fit(X, y, ls, float(a), float(b), kind))
        return -v if math.isfinite(v) else math.inf

    best = None
    lst = []
    for k in range(starts):
        if k == 0:
            x0 = np.log(np.concatenate([np.asarray(lengthscale, np.float32).astype(np.float64),
                                        [float(np.float32(sf2)), float(np.float32(sn2))]]))
        else:
            x0 = np.array([lo[i] + uniform(seed, search, k, i, dim, starts) * (hi[i] - lo[i])
                           for i in range(dim)])
        xb, fb, fs0, _ = nelder_mead(negl, x0, lo, hi, step, iters)
        lst.append(-fs0)
        if best is None or fb < best[1]:
            best = (xb, fb)
    ls, a, b = theta(best[0])
    return dict(ls=ls, sf2=a, sn2=b, lml=-best[1], lml_starts=np.array(lst))
