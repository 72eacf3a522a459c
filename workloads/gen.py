"""Seeded synthetic inputs for the five BASELINE.json configurations.

This module holds none of the GP / EI arithmetic.  It only draws numbers: training inputs X,
candidates X*, noise, hyper-parameters theta, and evaluates the paper's synthetic objectives
(workloads/synthetic.py) to produce y.  Both the oracle (tests, bench cpu_baseline) and the CUDA
path consume exactly what it returns.

Streams: ``numpy.random.Generator(numpy.random.Philox(key=(cfg << 32) | (purpose << 16) | search))``
with purpose 0 = X, 1 = X*, 2 = eps (objective noise), 3 = theta.

Encoded inputs live in [0, 1]^d as float32 (reading R8); raw = lo + (hi - lo) * u with the paper's
box [-50, 50].  theta recipe (reading R6): l_j = 0.4 sqrt(d) 2^U(-1,1), sf2 = 1,
sn2 = 1e-4 in standardised units.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import synthetic as syn

RBF = 0
MATERN52 = 1

LO, HI = -50.0, 50.0

# (S, n, d, M per search) of SURVEY.md §8 table
CONFIG_SHAPES = {
    1: (1, 20, 2, 4096),
    2: (1, 200, 20, 1 << 20),
    3: (64, 100, 5, 1 << 18),
    4: (1, 500, 60, 1 << 22),
    5: (1, 5, 35, 1 << 18),
}

CONFIG_NAMES = {
    1: "cfg1: 1 search, 2-D synthetic slice, n=20, M=4096 grid",
    2: "cfg2: 1 search, 20-D synthetic Case 3, n=200, M=1,048,576",
    3: "cfg3: 64 sub-searches x 5-D, n=100, M=262,144 each",
    4: "cfg4: 1 search, 60-D block-interdependent, n=500, M=4,194,304",
    5: "cfg5: RT-TDDFT-shaped replay, d_enc=35",
}


def rng(cfg, purpose, search=0):
    return np.random.Generator(np.random.Philox(key=(cfg << 32) | (purpose << 16) | search))


def to_raw(u):
    return LO + (HI - LO) * np.asarray(u, dtype=np.float64)


@dataclass
class Search:
    X: np.ndarray            # n x d float32 in [0, 1]
    y: np.ndarray            # n float64 raw objective
    lengthscale: np.ndarray  # d float32
    sf2: float
    sn2: float


@dataclass
class Workload:
    cfg: int
    kernel: int
    searches: list
    Xstar: list = field(default_factory=list)  # per search: M x d float32
    m_global_base: list = field(default_factory=list)  # per search: global index of row 0
    M_global: list = field(default_factory=list)

    @property
    def S(self):
        return len(self.searches)


def theta(cfg, search, d):
    g = rng(cfg, 3, search)
    ls = (0.4 * np.sqrt(d) * 2.0 ** g.uniform(-1.0, 1.0, size=d)).astype(np.float32)
    return ls, np.float32(1.0), np.float32(1e-4)


def _bo_like(g, n, d, f):
    """'BO-like' layout: 40% uniform, the rest within +-0.05 of the incumbent."""
    n0 = max(2, int(round(0.4 * n)))
    X = g.random((n, d), dtype=np.float32)
    y0 = f(X[:n0])
    inc = X[int(np.argmin(y0))]
    X[n0:] = np.clip(inc + g.uniform(-0.05, 0.05, size=(n - n0, d)), 0.0, 1.0).astype(np.float32)
    return X


def _objective(cfg, search, X, noise=True):
    """y for the training rows of ``search`` in ``cfg``; eps from stream purpose 2."""
    n = X.shape[0]
    raw = to_raw(X)
    if cfg == 1:
        return syn.f2_slice(raw)
    ge = rng(cfg, 2, search)
    if cfg == 2:
        eps = 0.1 * ge.standard_normal((n, syn.N_EPS)) if noise else None
        return syn.f20(raw, 3, eps)
    if cfg == 3:
        group = search % 4
        case = (search // 4) % 5 + 1
        eps = 0.1 * ge.standard_normal((n, syn.N_EPS)) if noise else None
        return syn.sub5(raw, group, case, eps)
    if cfg == 4:
        eps = 0.1 * ge.standard_normal((n, 3 * syn.N_EPS)) if noise else None
        return syn.f60(raw, eps)
    raise ValueError(cfg)


def lattice64():
    """Config 1 candidates: the 64 x 64 lattice u = i/63, idx = 64 i0 + i1."""
    u = (np.arange(64, dtype=np.float64) / 63.0).astype(np.float32)
    X0, X1 = np.meshgrid(u, u, indexing="ij")
    return np.stack([X0.ravel(), X1.ravel()], axis=1)


def make(cfg, n=None, d=None, M=None, S=None, layout="uniform", kernel=MATERN52,
         with_candidates=True, rank=0, world=1, search_ids=None):
    """Generate config ``cfg`` (optionally shrunk for parity tests).

    Candidates are sharded contiguously: rank r of ``world`` gets global rows
    [r*ceil(M/world), min(M, (r+1)*ceil(M/world))) of every search.  The rows
    are drawn from the search's X* stream in global order, so every sharding sees the same
    candidates.  ``search_ids`` selects a subset of the searches (search-sharded runs: rank r
    takes searches r, r + world, ...); each search is drawn from its own streams, identical to
    its draw in the full workload.
    """
    S0, n0, d0, M0 = CONFIG_SHAPES[cfg]
    S = S0 if S is None else S
    n = n0 if n is None else n
    d = d0 if d is None else d
    M = M0 if M is None else M
    searches, Xs, bases, Mg = [], [], [], []
    for s in (range(S) if search_ids is None else search_ids):
        g = rng(cfg, 0, s)
        if cfg == 3 and s % 4 == 3:
            X = g.random((n, d), dtype=np.float32)
            bad = np.abs(to_raw(X)) < 1e-6
            while bad.any():  # G4 singularity guard: resample (SURVEY.md §8(d) cfg 3)
                X[bad] = g.random(int(bad.sum()), dtype=np.float32)
                bad = np.abs(to_raw(X)) < 1e-6
        elif layout == "bo" and cfg in (2, 4):
            X = _bo_like(g, n, d, lambda Z: _objective(cfg, s, Z, noise=False))
        else:
            X = g.random((n, d), dtype=np.float32)
        y = _objective(cfg, s, X)
        ls, sf2, sn2 = theta(cfg, s, d)
        searches.append(Search(X, y, ls, float(sf2), float(sn2)))
        if with_candidates:
            per = -(-M // world)
            a, b = min(M, rank * per), min(M, (rank + 1) * per)
            if cfg == 1 and M == 4096 and d == 2:
                Xstar = lattice64()[a:b]
            else:
                gx = rng(cfg, 1, s)
                if a > 0:
                    gx.random((a, d), dtype=np.float32)  # skip to the shard start
                Xstar = gx.random((b - a, d), dtype=np.float32)
            Xs.append(np.ascontiguousarray(Xstar))
            bases.append(a)
            Mg.append(M)
    return Workload(cfg, kernel, searches, Xs, bases, Mg)


def random_case(seed, n, d, M, S=1, kernel=MATERN52, ls_scale=0.4, sn2=1e-4, clustered=False):
    """Generic seeded case for parity edge shapes (uniform X, smooth-ish y)."""
    searches, Xs = [], []
    for s in range(S):
        g = np.random.Generator(np.random.Philox(key=(0xABCD << 32) | (seed << 16) | s))
        ns = n[s] if isinstance(n, (list, tuple)) else n
        ds = d[s] if isinstance(d, (list, tuple)) else d
        Ms = M[s] if isinstance(M, (list, tuple)) else M
        X = g.random((ns, ds), dtype=np.float32)
        if clustered and ns > 4:
            k = int(0.6 * ns)
            X[ns - k:] = np.clip(X[0] + g.uniform(-0.05, 0.05, size=(k, ds)), 0, 1).astype(np.float32)
        w = g.standard_normal(ds)
        y = np.sin(3.0 * (X.astype(np.float64) @ w)) + 0.1 * g.standard_normal(ns)
        ls = (ls_scale * np.sqrt(ds) * 2.0 ** g.uniform(-1, 1, size=ds)).astype(np.float32)
        searches.append(Search(X, y, ls, 1.0, float(np.float32(sn2))))
        Xs.append(g.random((Ms, ds), dtype=np.float32))
    return Workload(0, kernel, searches, Xs, [0] * S, [x.shape[0] for x in Xs])
