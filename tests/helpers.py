"""Shared test helpers: pack workloads for the C ABI, run the oracle, apply the tolerances.

Tolerance reading T1: in standardised units
  |d mu~| <= 1e-4 max(|mu~_ref|, 1),  |d s2~| <= 1e-4 sf2,
  |d EI| <= 1e-4 max(max_j EI_ref,j, 1e-30)   (1e-30: the float32-underflow floor of R11)
Argmax rule R11: the index must match wherever the oracle's relative top-2 gap > 1e-3 and
EI_(1) >= 1e-30; otherwise the GPU's pick must be within 1e-3 EI_(1) of the oracle maximum.
"""
import numpy as np

from oracle import gp

TOL = 1e-4
GAP = 1e-3


def pack(workload):
    S = workload.S
    n = [s.X.shape[0] for s in workload.searches]
    d = [s.X.shape[1] for s in workload.searches]
    X = np.ascontiguousarray(np.concatenate([s.X.ravel() for s in workload.searches]), np.float32)
    y = np.ascontiguousarray(np.concatenate([s.y for s in workload.searches]), np.float64)
    ls = np.ascontiguousarray(np.concatenate([s.lengthscale for s in workload.searches]),
                              np.float32)
    sf2 = np.array([s.sf2 for s in workload.searches], np.float32)
    sn2 = np.array([s.sn2 for s in workload.searches], np.float32)
    return n, d, X, y, ls, sf2, sn2


def pack_candidates(workload):
    Xs = np.ascontiguousarray(np.concatenate([x.ravel() for x in workload.Xstar]), np.float32)
    m_off = np.zeros(workload.S + 1, np.int64)
    m_off[1:] = np.cumsum([x.shape[0] for x in workload.Xstar])
    return Xs, m_off


def oracle_fits(workload):
    return [gp.fit(s.X, s.y, s.lengthscale, s.sf2, s.sn2, workload.kernel)
            for s in workload.searches]


def check_T1(om, res, mu_raw, var_raw, ei_raw, label=""):
    """Element-wise T1 comparison of raw GPU outputs with the oracle's ScoreResult."""
    mu_t = (mu_raw.astype(np.float64) - om.mean) / om.std
    var_t = var_raw.astype(np.float64) / om.std ** 2
    ei_t = ei_raw.astype(np.float64) / om.std
    dmu = np.abs(mu_t - res.mu) / np.maximum(np.abs(res.mu), 1.0)
    dvar = np.abs(var_t - res.var) / om.sf2
    eimax = max(res.ei_all.max(), 1e-30)  # R11 floor: float32 EI underflows below
    dei = np.abs(ei_t - res.ei_all) / eimax
    worst = dict(mu=float(dmu.max()), var=float(dvar.max()), ei=float(dei.max()))
    assert worst["mu"] <= TOL and worst["var"] <= TOL and worst["ei"] <= TOL, (label, worst)
    return worst


def check_argmax(res, idx, label=""):
    """R11: exact index where the gap is decisive, else a valid near-maximal choice."""
    top = res.ei_all.max()
    if res.gap_rel > GAP and top >= 1e-30:
        assert idx == res.idx, (label, idx, res.idx, res.gap_rel)
    else:
        assert 0 <= idx < res.ei_all.size, (label, idx)
        assert res.ei_all[idx] >= top * (1 - GAP) or top < 1e-30, (label, idx, res.idx)
