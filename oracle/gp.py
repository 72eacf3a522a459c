"""Float64 CPU oracle of the GP-surrogate + Expected-Improvement hot path (H1-H4, H6-H9, H11).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module.  The product path
(``paper_2403_08131_b200/``) never imports it, shares no code with it and has no CPU fallback.

What it computes (PAPER.md = ``P:L``, SPEC.md = ``S:L``, SURVEY.md section 8 = ``§8``):

* P:L72 (§III.A, "Bayesian Optimization"): a surrogate model is trained on the observed
  configurations, and "an acquisition function guides the selection of the next configuration".
  The paper does not name the surrogate kernel or the acquisition; the readings R1-R13 of
  SURVEY.md §8(c) (listed in DESIGN.md) fix them: a Gaussian process with an ARD RBF or
  Matern-5/2 kernel, Expected Improvement for minimisation.
* P:L249 / P:L256 (§IV.D): "the training complexity of Gaussian Processes ... O(N^3)" -- the
  Cholesky factorisation below.

Everything is the textbook definition written out in float64, in the order the definition states
it, with no blocking or reordering:

    y~ = (y - mean(y)) / std(y)                          standardise (reading R7)
    K  = k(X, X) + (sn2 + j_k) I                         Gram matrix  (reading R9 for j_k)
    L  = chol(K)                                         hand-written column Cholesky
    alpha = L^-T L^-1 y~                                 forward + back substitution
    mu~(x*)  = k*^T alpha                                posterior mean
    s2~(x*)  = max(sf2 - |L^-1 k*|^2, 0)                 latent posterior variance (R5)
    EI(x*)   = s~ * (phi(z) + z Phi(z)),  z = (best - mu~) / s~
             = max(best - mu~, 0)       if s~ == 0                 (reading R4)
    argmax EI, ties -> lowest global index               (reading R10)

Inputs are taken exactly as the GPU path receives them (X, X* and the hyper-parameters stored as
float32, y as float64) and promoted exactly to float64, so input rounding is identical on both
sides.  Squared distances are formed by direct differences, sum_d ((x*_d - x_d)/l_d)^2, never by
the GEMM expansion.  LAPACK is not used on this path; it only appears in the oracle's own pins
(tests/test_oracle_*.py).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
from scipy.special import erfc

RBF = 0
MATERN52 = 1

# Jitter ladder j_k = 1e-8 * 10^k * sf2, k = 0..6 ("start 1e-8, escalate x10 up to 1e-2";
# reading R9: relative to sf2, always added on top of sn2).
JITTER_BASE = 1e-8
JITTER_STEPS = 7

STATUS_OK = 0
STATUS_ENOTPD = 2
STATUS_WDEGENERATE = 3


DEGENERATE_REL = 1e-12


def standardize(y):
    """H1: y~ = (y - mean) / std with ddof = 0; a zero std -> 1 and the search is flagged
    degenerate ("zero mean, unit variance"; S:L344 degenerate-data contract; R7).

    "Zero" is std <= 1e-12 max|y|, and then y~ := 0 (reading R7a): with constant y the computed std is
    rounding noise whose value depends on the summation order, so an exact test would not be
    reproducible across implementations."""
    y = np.asarray(y, dtype=np.float64)
    mean = float(np.mean(y))
    std = float(np.sqrt(np.mean((y - mean) ** 2)))
    degenerate = not (std > DEGENERATE_REL * float(np.max(np.abs(y))))
    if degenerate:  # constant-mean model: y~ is identically zero
        return np.zeros_like(y), mean, 1.0, True
    return (y - mean) / std, mean, std, degenerate


def sq_dist(A, B, lengthscale):
    """r^2[i, j] = sum_d ((A[i,d] - B[j,d]) / l_d)^2 by direct differences (ARD, reading R2)."""
    A = np.asarray(A, dtype=np.float64) / np.asarray(lengthscale, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64) / np.asarray(lengthscale, dtype=np.float64)
    r2 = np.zeros((A.shape[0], B.shape[0]))
    for d in range(A.shape[1]):
        diff = A[:, d][:, None] - B[:, d][None, :]
        r2 += diff * diff
    return r2


def kernel_from_sq_dist(r2, sf2, kind):
    """k(r) for the two kernels of reading R1/R2 (north star (a)).

    RBF:        sf2 * exp(-r^2 / 2)
    Matern-5/2: sf2 * (1 + sqrt(5) r + 5 r^2 / 3) * exp(-sqrt(5) r)
    """
    r2 = np.asarray(r2, dtype=np.float64)
    if kind == RBF:
        return sf2 * np.exp(-0.5 * r2)
    if kind == MATERN52:
        r = np.sqrt(r2)
        return sf2 * (1.0 + math.sqrt(5.0) * r + (5.0 / 3.0) * r2) * np.exp(-math.sqrt(5.0) * r)
    raise ValueError(f"unknown kernel {kind}")


def cholesky_lower(A):
    """Hand-written column (Cholesky-Crout) factorisation A = L L^T.

    Returns L, or None when a pivot is <= 0 or not finite (the failure test of reading R9).
    """
    A = np.asarray(A, dtype=np.float64)
    n = A.shape[0]
    L = np.zeros_like(A)
    for j in range(n):
        pivot = A[j, j] - np.dot(L[j, :j], L[j, :j])
        if not (np.isfinite(pivot) and pivot > 0.0):
            return None
        L[j, j] = math.sqrt(pivot)
        if j + 1 < n:
            L[j + 1:, j] = (A[j + 1:, j] - L[j + 1:, :j] @ L[j, :j]) / L[j, j]
    return L


def forward_sub(L, B):
    """Solve L V = B for lower-triangular L (B may be a vector or n x m)."""
    L = np.asarray(L, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    V = np.zeros_like(B)
    for i in range(L.shape[0]):
        V[i] = (B[i] - L[i, :i] @ V[:i]) / L[i, i]
    return V


def back_sub_transposed(L, B):
    """Solve L^T V = B for lower-triangular L."""
    L = np.asarray(L, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    n = L.shape[0]
    V = np.zeros_like(B)
    for i in range(n - 1, -1, -1):
        V[i] = (B[i] - L[i + 1:, i] @ V[i + 1:]) / L[i, i]
    return V


@dataclass
class GpModel:
    """D4: one fitted sub-search."""
    X: np.ndarray            # n x d encoded training inputs (float64 copy of the float32 input)
    lengthscale: np.ndarray  # d
    sf2: float
    sn2: float
    kind: int
    ytilde: np.ndarray       # standardised targets
    mean: float
    std: float
    best: float              # min y~ (reading R3)
    L: np.ndarray | None     # Cholesky factor of K + (sn2 + jitter) I
    alpha: np.ndarray | None
    jitter_k: int            # index k of the jitter that succeeded (-1 on failure)
    jitter: float
    status: int


def fit(X, y, lengthscale, sf2, sn2, kind=MATERN52):
    """H1-H4 for one sub-search ("trained using ... configurations"; P:L249 O(N^3))."""
    X = np.asarray(X, dtype=np.float32).astype(np.float64)
    ls = np.asarray(lengthscale, dtype=np.float32).astype(np.float64)
    sf2 = float(np.float32(sf2))
    sn2 = float(np.float32(sn2))
    ytilde, mean, std, degenerate = standardize(y)
    n = X.shape[0]
    K0 = kernel_from_sq_dist(sq_dist(X, X, ls), sf2, kind)
    L = None
    jitter_k, jitter = -1, float("nan")
    for k in range(JITTER_STEPS):
        j = JITTER_BASE * (10.0 ** k) * sf2
        L = cholesky_lower(K0 + (sn2 + j) * np.eye(n))
        if L is not None:
            jitter_k, jitter = k, j
            break
    if L is None:
        return GpModel(X, ls, sf2, sn2, kind, ytilde, mean, std, float(np.min(ytilde)),
                       None, None, -1, float("nan"), STATUS_ENOTPD)
    alpha = back_sub_transposed(L, forward_sub(L, ytilde))
    status = STATUS_WDEGENERATE if degenerate else STATUS_OK
    return GpModel(X, ls, sf2, sn2, kind, ytilde, mean, std, float(np.min(ytilde)),
                   L, alpha, jitter_k, jitter, status)


def posterior(model: GpModel, Xstar, chunk=4096):
    """H6-H7: standardised posterior mean mu~ and latent variance s2~ at every row of X*.

    mu~ = k*^T alpha;  s2~ = max(sf2 - |L^-1 k*|^2, 0)  (reading R5).
    """
    Xstar = np.asarray(Xstar, dtype=np.float32).astype(np.float64)
    M = Xstar.shape[0]
    mu = np.empty(M)
    var = np.empty(M)
    for a in range(0, M, chunk):
        b = min(M, a + chunk)
        Ks = kernel_from_sq_dist(sq_dist(model.X, Xstar[a:b], model.lengthscale), model.sf2, model.kind)
        mu[a:b] = Ks.T @ model.alpha
        V = forward_sub(model.L, Ks)
        var[a:b] = np.maximum(model.sf2 - np.sum(V * V, axis=0), 0.0)
    return mu, var


def tau(z):
    """tau(z) = phi(z) + z Phi(z) with Phi(z) = erfc(-z / sqrt 2) / 2 (standard normal)."""
    z = np.asarray(z, dtype=np.float64)
    phi = np.exp(-0.5 * z * z) / math.sqrt(2.0 * math.pi)
    Phi = 0.5 * erfc(-z / math.sqrt(2.0))
    return phi + z * Phi


def expected_improvement(mu, var, best):
    """H8: EI for minimisation with xi = 0 (readings R3, R4).

    EI = s * tau((best - mu) / s) for s > 0, max(best - mu, 0) for s == 0.
    """
    mu = np.asarray(mu, dtype=np.float64)
    s = np.sqrt(np.asarray(var, dtype=np.float64))
    out = np.maximum(best - mu, 0.0)
    pos = s > 0.0
    z = (best - mu[pos]) / s[pos]
    out[pos] = s[pos] * tau(z)
    return out


def argmax_lowest(ei):
    """H9: index of the maximum, ties -> lowest index (reading R10)."""
    ei = np.asarray(ei)
    return int(np.flatnonzero(ei == ei.max())[0])


@dataclass
class ScoreResult:
    idx: int            # global index of the suggestion
    ei: float           # max EI, standardised units
    ei_raw: float       # std * ei (H11)
    gap_rel: float      # (EI_(1) - EI_(2)) / EI_(1), for the argmax rule R11
    ei_all: np.ndarray  # standardised EI of every candidate
    mu: np.ndarray
    var: np.ndarray


def score(model: GpModel, Xstar, best=None, chunk=4096):
    """H6-H9 + H11 for one sub-search: posterior, EI and the argmax with lowest-index ties.

    ``best`` is in raw units (None -> min observed y, reading R3).
    """
    b = model.best if best is None else (float(best) - model.mean) / model.std
    mu, var = posterior(model, Xstar, chunk)
    ei = expected_improvement(mu, var, b)
    i = argmax_lowest(ei)
    top = ei[i]
    if ei.size > 1:
        rest = np.delete(ei, i)
        second = rest.max()
        gap = (top - second) / top if top > 0 else 0.0
    else:
        gap = 1.0
    return ScoreResult(i, float(top), float(model.std * top), float(gap), ei, mu, var)


def raw_posterior(model: GpModel, mu, var):
    """H11: mu = mean + std mu~, var = std^2 s2~ (raw units)."""
    return model.mean + model.std * np.asarray(mu), model.std ** 2 * np.asarray(var)
