"""Oracle for H0 (encoding) and H5 (constrained candidate generation) -- TEST INFRASTRUCTURE ONLY.

Written from the specification in SURVEY.md §8(a) H5 / §8(c) P16, independently of the CUDA
path (no shared code, tables or constants; only the documented algorithm):

* Philox4x32-10 (Salmon et al., SC'11): M0 = 0xD2511F53, M1 = 0xCD9E8D57, W0 = 0x9E3779B9,
  W1 = 0xBB67AE85, 10 rounds, key = (seed_lo32, seed_hi32).  Word u of candidate i of search s at
  iteration t is output[u mod 4] of Philox(key, ctr = (i, s, t, u div 4)).
* Draw units: free parameters in declaration order, then constrained blocks in order; one word each.
  Real: u = (w >> 8) 2^-24 (exact in float32).  Discrete with K values: index (u64(w >> 8) K) >> 24.
  Block with T valid tuples: tuple index (u64(w >> 8) T) >> 24 -- uniform over the valid set with
  no rejection loop (GPTune could not even suggest candidates for the constrained searches).
* Encoding (H0, reading R8): real/int (v - lo)/(hi - lo); ordinal rank/(K - 1);
  categorical one-hot; K = 1 -> 0.  Each encoded value is computed in float64 and rounded once to
  float32.
* Fixed parameters (SURVEY.md §8(a) H0 "fixed params dropped"; parameters a
  search does not tune keep their default or an earlier stage's value): no encoded column, no
  Philox word (they are not free parameters); their raw value is the given constant.
"""
from __future__ import annotations

import numpy as np

REAL, INT, ORDINAL, CATEGORICAL, FIXED = 0, 1, 2, 3, 4

M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK = 0xFFFFFFFF


def philox4x32_10(ctr, key):
    """Scalar Philox4x32-10 on python ints: ctr = (c0, c1, c2, c3), key = (k0, k1)."""
    c0, c1, c2, c3 = ctr
    k0, k1 = key
    for r in range(10):
        if r:
            k0 = (k0 + W0) & MASK
            k1 = (k1 + W1) & MASK
        p0 = M0 * c0
        p1 = M1 * c2
        c0, c1, c2, c3 = ((p1 >> 32) ^ c1 ^ k0) & MASK, p1 & MASK, ((p0 >> 32) ^ c3 ^ k1) & MASK, p0 & MASK
    return c0, c1, c2, c3


def philox_vec(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10 (numpy uint64 arithmetic on 32-bit lanes)."""
    c0, c1, c2, c3 = (np.asarray(c, dtype=np.uint64) & MASK for c in (c0, c1, c2, c3))
    k0, k1 = np.uint64(k0), np.uint64(k1)
    m0, m1 = np.uint64(M0), np.uint64(M1)
    for r in range(10):
        if r:
            k0 = (k0 + np.uint64(W0)) & np.uint64(MASK)
            k1 = (k1 + np.uint64(W1)) & np.uint64(MASK)
        p0 = m0 * c0
        p1 = m1 * c2
        c0, c1, c2, c3 = ((p1 >> np.uint64(32)) ^ c1 ^ k0) & np.uint64(MASK), p1 & np.uint64(MASK), \
            ((p0 >> np.uint64(32)) ^ c3 ^ k1) & np.uint64(MASK), p0 & np.uint64(MASK)
    return c0, c1, c2, c3


class Space:
    """A search space: parameters (kind, range / value list) plus constrained blocks given by
    their enumerated valid tuples (value indices)."""

    def __init__(self, params, blocks=()):
        # params: list of dicts {kind, lo, hi} (REAL/INT) or {kind, values} (ORDINAL) or
        #         {kind, K} (CATEGORICAL) or {kind, lo} (FIXED: the constant)
        self.params = params
        self.blocks = [(list(b["params"]), np.asarray(b["tuples"], dtype=np.int64)) for b in blocks]
        inblock = {p for ps, _ in self.blocks for p in ps}
        self.free = [i for i in range(len(params))
                     if i not in inblock and params[i]["kind"] != FIXED]
        self.units = len(self.free) + len(self.blocks)

    def nvals(self, i):
        p = self.params[i]
        if p["kind"] == INT:
            return int(p["hi"] - p["lo"]) + 1
        if p["kind"] == ORDINAL:
            return len(p["values"])
        if p["kind"] == CATEGORICAL:
            return int(p["K"])
        return 0

    @property
    def dim(self):
        return sum(self.nvals(i) if p["kind"] == CATEGORICAL else 0 if p["kind"] == FIXED else 1
                   for i, p in enumerate(self.params))

    def words(self, seed, search, iteration, idx):
        """Philox words (units x len(idx)) for global candidate indices idx."""
        idx = np.asarray(idx, dtype=np.uint64)
        k0, k1 = seed & MASK, (seed >> 32) & MASK
        out = []
        for b in range((self.units + 3) // 4):
            w = philox_vec(idx, np.full_like(idx, search), np.full_like(idx, iteration),
                           np.full_like(idx, b), k0, k1)
            out.extend(w)
        return np.stack(out[:self.units]).astype(np.uint64)

    def sample_values(self, seed, search, iteration, idx):
        """Per candidate: real parameters as u in [0,1), discrete ones as value indices."""
        W = self.words(seed, search, iteration, idx)
        P = len(self.params)
        vals = np.zeros((P, W.shape[1]))
        for u, i in enumerate(self.free):
            w8 = W[u] >> np.uint64(8)
            if self.params[i]["kind"] == REAL:
                vals[i] = w8.astype(np.float64) * 2.0 ** -24
            else:
                vals[i] = ((w8 * np.uint64(self.nvals(i))) >> np.uint64(24)).astype(np.float64)
        for b, (ps, tup) in enumerate(self.blocks):
            w8 = W[len(self.free) + b] >> np.uint64(8)
            t = ((w8 * np.uint64(len(tup))) >> np.uint64(24)).astype(np.int64)
            for j, i in enumerate(ps):
                vals[i] = tup[t, j]
        return vals.T  # (count, P): u for real params, value index for discrete ones

    def encode_values(self, vals):
        """Encoded float32 rows from sample_values output (H0)."""
        vals = np.atleast_2d(vals)
        cols = []
        for i, p in enumerate(self.params):
            v = vals[:, i]
            if p["kind"] == FIXED:
                continue
            if p["kind"] == REAL:
                cols.append(v.astype(np.float32))
            elif p["kind"] == CATEGORICAL:
                K = self.nvals(i)
                for k in range(K):
                    cols.append((v == k).astype(np.float32))
            else:
                K = self.nvals(i)
                cols.append((v / (K - 1) if K > 1 else 0.0 * v).astype(np.float32))
        return np.stack(cols, axis=1)

    def raw_values(self, vals):
        """Raw parameter values (float64) from sample_values output (H11 decode)."""
        vals = np.atleast_2d(vals)
        out = np.zeros_like(vals, dtype=np.float64)
        for i, p in enumerate(self.params):
            v = vals[:, i]
            if p["kind"] == REAL:
                out[:, i] = p["lo"] + (p["hi"] - p["lo"]) * v
            elif p["kind"] == INT:
                out[:, i] = p["lo"] + v
            elif p["kind"] == ORDINAL:
                out[:, i] = np.asarray(p["values"], dtype=np.float64)[v.astype(np.int64)]
            elif p["kind"] == FIXED:
                out[:, i] = float(p["lo"])
            else:
                out[:, i] = v
        return out

    def sample(self, seed, search, iteration, idx):
        """Encoded candidates (float32, count x dim) -- the H5 oracle."""
        return self.encode_values(self.sample_values(seed, search, iteration, idx))
