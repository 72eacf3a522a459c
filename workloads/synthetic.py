"""The paper's synthetic objective functions (Fig. 1 + Table I), used to generate observed y.

These are workload generators, not part of the GP/EI method: neither the oracle nor the CUDA
path calls them; they only produce the objective values y that both sides then read.

PAPER.md (Fig. 1; Table I; P:L116 domain [-50, 50]; P:L144 log|.|):

    F(x_0..x_19) = G1 + G2 + G3 + G4, each group value passed through log(|.| + delta)
    G1 = sum_{i=0..3} (x_i - x_{i+1})^2 + sum_{i=0..4} A_i
    G2 = sum_{k=5..8} (x_k - x_{k+1})^4 + sum_{k=5..9} A_k
    G3 = Table I row for the case
    G4 = sum_{v=15..19} 1/x_v + eps
    A_i = 10 cos(2 pi (x_i - 1)) + eps

Readings: delta = 1e-12; eps ~ N(0, sigma^2) drawn once per
occurrence (5 in G1, 5 in G2, 1 in G3, 1 in G4 -> 12 per evaluation); "A_j" in G2 is A_k;
Table I rows 4-5 pair (u, v) zipped: (10,15), (11,16), ..., (14,19).
"""
from __future__ import annotations

import numpy as np

DELTA = 1e-12
N_EPS = 12  # eps draws per 20-D evaluation: A_0..A_4, A_5..A_9, G3, G4


def _eps(eps, n, j):
    return 0.0 if eps is None else eps[:, j]


def _log_abs(v):
    return np.log(np.abs(v) + DELTA)


def group1(x, eps=None):
    """x: (n, >=5) raw values; returns raw (un-logged) G1."""
    s = np.zeros(x.shape[0])
    for i in range(4):
        s += (x[:, i] - x[:, i + 1]) ** 2
    for i in range(5):
        s += 10.0 * np.cos(2.0 * np.pi * (x[:, i] - 1.0)) + _eps(eps, x.shape[0], i)
    return s


def group2(x, eps=None):
    """x: (n, >=10) raw values; uses x_5..x_9."""
    s = np.zeros(x.shape[0])
    for k in range(5, 9):
        s += (x[:, k] - x[:, k + 1]) ** 4
    for k in range(5, 10):
        s += 10.0 * np.cos(2.0 * np.pi * (x[:, k] - 1.0)) + _eps(eps, x.shape[0], k)
    return s


def group3(x, case, eps=None):
    """Table I row ``case`` (1..5) on x_10..x_14 (u) and x_15..x_19 (v)."""
    u = x[:, 10:15]
    v = x[:, 15:20]
    if case == 1:
        s = u.sum(1) + np.cos(2.0 * np.pi * v).sum(1)
    elif case == 2:
        s = (u ** 2).sum(1) + v.sum(1)
    elif case == 3:
        s = (u ** 2).sum(1) + (v ** 2).sum(1)
    elif case == 4:
        s = ((u * v ** 4) ** 2).sum(1)
    elif case == 5:
        s = ((u * v ** 8) ** 2).sum(1)
    else:
        raise ValueError(case)
    return s + _eps(eps, x.shape[0], 10)


def group4(x, eps=None):
    return (1.0 / x[:, 15:20]).sum(1) + _eps(eps, x.shape[0], 11)


def f20(x, case, eps=None):
    """The 20-D synthetic function of Fig. 1 with Group 3 from Table I; x raw in [-50, 50]."""
    x = np.asarray(x, dtype=np.float64)
    return (_log_abs(group1(x, eps)) + _log_abs(group2(x, eps))
            + _log_abs(group3(x, case, eps)) + _log_abs(group4(x, eps)))


def f20_groups(x, case, eps=None):
    x = np.asarray(x, dtype=np.float64)
    return (_log_abs(group1(x, eps)), _log_abs(group2(x, eps)),
            _log_abs(group3(x, case, eps)), _log_abs(group4(x, eps)))


def f2_slice(x):
    """Config 1 objective: the Group-1 term on 2 variables, noise free (SURVEY.md §8(d) cfg 1).
    f2(x0, x1) = log(|(x0 - x1)^2 + 10 cos 2pi(x0 - 1) + 10 cos 2pi(x1 - 1)| + delta)."""
    x = np.asarray(x, dtype=np.float64)
    g = ((x[:, 0] - x[:, 1]) ** 2 + 10.0 * np.cos(2 * np.pi * (x[:, 0] - 1.0))
         + 10.0 * np.cos(2 * np.pi * (x[:, 1] - 1.0)))
    return _log_abs(g)


def f2_slice_raw(x):
    """Un-logged config-1 slice, used by the sub-box known-optimum check (P12)."""
    x = np.asarray(x, dtype=np.float64)
    return ((x[:, 0] - x[:, 1]) ** 2 + 10.0 * np.cos(2 * np.pi * (x[:, 0] - 1.0))
            + 10.0 * np.cos(2 * np.pi * (x[:, 1] - 1.0)))


def sub5(x5, group, case=3, eps=None):
    """Config 3 five-parameter sub-search objectives (SURVEY.md §8(d) cfg 3).

    group 0: G1 on x_0..x_4;  group 1: G2 on x_5..x_9;  group 2: G3 of ``case`` on x_10..x_14
    with x_15..x_19 frozen at 1;  group 3: G4 on x_15..x_19.  Each returns log(|.| + delta).
    """
    x5 = np.asarray(x5, dtype=np.float64)
    n = x5.shape[0]
    x = np.ones((n, 20))
    x[:, 5 * group:5 * group + 5] = x5
    if group == 0:
        return _log_abs(group1(x, eps))
    if group == 1:
        return _log_abs(group2(x, eps))
    if group == 2:
        return _log_abs(group3(x, case, eps))
    return _log_abs(group4(x, eps))


def f60(x, eps=None):
    """Config 4 block-interdependent 60-D function: Case 3, Case 4, Case 5 blocks of 20."""
    x = np.asarray(x, dtype=np.float64)
    e = [None, None, None] if eps is None else [eps[:, 0:12], eps[:, 12:24], eps[:, 24:36]]
    return f20(x[:, 0:20], 3, e[0]) + f20(x[:, 20:40], 4, e[1]) + f20(x[:, 40:60], 5, e[2])
