"""Pins of the oracle's remaining parts (VERDICT r1 "weak #1"), each against something other
than the oracle itself:

* P12 known optimum (Fig. 1 Group-1 term): a BO loop
  driven by the oracle (fit + EI + argmax with the history masked) on the 64 x 64 lattice of the
  [0, 3]^2 sub-box reaches the brute-force lattice minimum of the raw 2-D slice.  A dropped term,
  a wrong sign or a transposed operand anywhere in fit/posterior/EI/argmax stops the search from
  converging (the random-search baseline needs ~4096/2 evaluations on average).
* score(): the standardised incumbent (raw best -> (best - mean)/std), EI_raw = std EI and the
  relative top-2 gap (reading R11) on a constructed case whose EI values follow from closed forms
  (interpolation at a training point, prior reversion far away, 40-digit tau).
* Space.encode_values: ordinal rank/(K-1) and the one-hot column order of categoricals on a
  hand-encoded example (reading R8).
* Space.words: the 64-bit seed's key split (key = (seed_lo32, seed_hi32))
  for a seed >= 2^32, against the KAT-pinned scalar Philox.
"""
import numpy as np
import pytest

from oracle import gp
from oracle import space as sp
from workloads import synthetic

# ---------------------------------------------------------------- P12 known optimum
LATTICE = 64
BOX = 3.0


def _lattice():
    u = np.arange(LATTICE) / (LATTICE - 1)
    U = np.stack(np.meshgrid(u, u, indexing="ij"), axis=-1).reshape(-1, 2)  # idx = 64 i0 + i1
    return U.astype(np.float32)


def _oracle_bo(seed, ell, iters=100, n0=5):
    """Sequential BO with the oracle as the engine (S:L404 run_bo protocol: 5 random initial
    points, then fit -> EI over the candidate pool -> argmax (ties first) -> evaluate), the pool
    being the lattice with already-evaluated points masked (reading R14)."""
    U = _lattice()
    f = synthetic.f2_slice_raw(BOX * U.astype(np.float64))
    target = f.min()
    rng = np.random.default_rng(seed)
    hist = list(rng.choice(U.shape[0], n0, replace=False))
    for it in range(iters):
        if f[hist].min() == target:
            return it
        X = U[hist]
        m = gp.fit(X, f[hist], np.full(2, ell, np.float32), 1.0, 1e-6, gp.MATERN52)
        mu, var = gp.posterior(m, U)
        ei = gp.expected_improvement(mu, var, m.best)
        ei[hist] = -np.inf
        hist.append(gp.argmax_lowest(ei))
    return iters if f[hist].min() == target else None


@pytest.mark.parametrize("ell", [0.2])
def test_p12_oracle_bo_reaches_lattice_minimum(ell):
    """P12: 5/5 seeds reach the exact brute-force lattice minimum within 100 BO iterations
    (measured: 15-69).  A blind search of the 4096-point lattice finds that one point within
    105 evaluations with probability 105/4096 = 2.6 % per seed, so 5/5 is no accident; the
    three wells x0 = x1 in {0.5, 1.5, 2.5} are near-ties, so the search must also pick the
    right one (SURVEY.md's scratch quoted <= 60 iterations for its seeds)."""
    its = [_oracle_bo(seed, ell) for seed in range(5)]
    assert all(i is not None for i in its), its


def test_p12_lattice_minimum_is_near_known_minimisers():
    """The brute-force lattice minimum sits next to one of the analytic minimisers
    x0 = x1 = k + 1/2 (value -20) of the Group-1 slice (P12)."""
    U = _lattice().astype(np.float64) * BOX
    f = synthetic.f2_slice_raw(U)
    x = U[np.argmin(f)]
    assert f.min() < -19.5
    assert np.abs(x - np.round(x - 0.5) - 0.5).max() <= 0.5 * BOX / (LATTICE - 1) + 1e-12


# ---------------------------------------------------------------- score(): best, EI_raw, gap
TAU_HALF = 0.6977965574013060295935327469  # mpmath 40 digits: phi(0.5) + 0.5 Phi(0.5)


def test_score_raw_best_ei_raw_and_gap():
    """y = (0, 4) at x = 0, 1 (mean 2, std 2, y~ = -1, +1), raw best 3 -> standardised 0.5.
    Candidates: the training point x = 0 (mu~ = -1, s~ ~ 0: EI = 0.5 + 1 = 1.5), the training
    point x = 1 (EI ~ 0), two far points (mu~ = 0, s~^2 = sf2 = 1: EI = tau(0.5)).
    => idx 0, EI_raw = 2 * 1.5 = 3, gap_rel = (1.5 - tau(0.5)) / 1.5."""
    X = np.array([[0.0], [1.0]], np.float32)
    y = np.array([0.0, 4.0])
    m = gp.fit(X, y, np.array([0.05], np.float32), 1.0, 1e-12, gp.MATERN52)
    assert (m.mean, m.std) == (2.0, 2.0)
    Xs = np.array([[0.0], [1.0], [40.0], [-40.0]], np.float32)
    r = gp.score(m, Xs, best=3.0)
    exp = np.array([1.5, 0.0, TAU_HALF, TAU_HALF])
    assert np.allclose(r.ei_all, exp, rtol=0, atol=1e-5), r.ei_all
    assert r.idx == 0
    assert abs(r.ei - 1.5) <= 1e-5 and abs(r.ei_raw - 3.0) <= 2e-5
    assert abs(r.gap_rel - (1.5 - TAU_HALF) / 1.5) <= 1e-5
    # default best = min observed y~ = -1: the training point x = 0 gives EI ~ 0, the far
    # points EI = tau(-1) (40-digit value 0.0833154705876864...)
    r2 = gp.score(m, Xs)
    assert abs(r2.ei_all[2] - 0.08331547058768629) <= 1e-12 and r2.idx == 2
    # exact tie between the two far points -> gap 0, the lower index wins
    assert r2.gap_rel == 0.0


# ---------------------------------------------------------------- encoding (H0, reading R8)
def test_encoding_hand_example():
    """INT 0..10 at 5 -> 0.5; ORDINAL (2, 4, 8, 16) at 8 (rank 2 of 4) -> 2/3; CATEGORICAL K = 3
    at label 2 -> one-hot columns (0, 0, 1) in label order; REAL [-50, 50) at u = 0.75."""
    params = [{"kind": sp.INT, "lo": 0, "hi": 10}, {"kind": sp.ORDINAL, "values": [2, 4, 8, 16]},
              {"kind": sp.CATEGORICAL, "K": 3}, {"kind": sp.REAL, "lo": -50.0, "hi": 50.0},
              {"kind": sp.ORDINAL, "values": [7]}]
    S = sp.Space(params)
    vals = np.array([[5, 2, 2, 0.75, 0], [0, 0, 0, 0.0, 0], [10, 3, 1, 0.5, 0]], np.float64)
    enc = S.encode_values(vals)
    exp = np.array([[0.5, 2 / 3, 0, 0, 1, 0.75, 0], [0, 0, 1, 0, 0, 0, 0],
                    [1, 1, 0, 1, 0, 0.5, 0]], np.float32)
    assert enc.dtype == np.float32 and np.array_equal(enc, exp), enc
    raw = S.raw_values(vals)
    assert np.array_equal(raw[0], [5, 8, 2, 25.0, 7]) and np.array_equal(raw[2], [10, 16, 1, 0.0, 7])


# ---------------------------------------------------------------- P16 seed key split
@pytest.mark.parametrize("seed", [0x299F31D0A4093822, 0xFFFFFFFFFFFFFFFF, 1 << 32])
def test_seed_high_word_key_split(seed):
    """Word u of candidate i = output[u % 4] of Philox(key = (seed_lo32, seed_hi32),
    ctr = (i, s, t, u // 4)) for seeds >= 2^32 (the high word must reach the key)."""
    params = [{"kind": sp.REAL, "lo": 0.0, "hi": 1.0}] * 6
    S = sp.Space(params)
    idx = np.array([0, 1, 0x243F6A88, 2 ** 32 - 1], np.uint64)
    W = S.words(seed, 0x85A308D3, 0x13198A2E, idx)
    for j, i in enumerate(idx):
        for u in range(6):
            ref = sp.philox4x32_10((int(i), 0x85A308D3, 0x13198A2E, u // 4),
                                   (seed & 0xFFFFFFFF, seed >> 32))
            assert int(W[u][j]) == ref[u % 4]
    # and the high word matters: dropping it changes the stream
    lo_only = S.words(seed & 0xFFFFFFFF, 0x85A308D3, 0x13198A2E, idx)
    assert not np.array_equal(W, lo_only)
