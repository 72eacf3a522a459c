"""Config 5 workload: the RT-TDDFT tuning space of Table IV and its objective.

Readings:
* nstb in divisors(64), nkpb in divisors(36), nspb in {1, 2}; per kernel X in (DSCAL, PAIR, ZCOPY,
  VEC, ZVEC): u_X categorical {1, 2, 4, 8}, tb_X in {32, 64, ..., 1024}, tb_sm_X in 1..32;
  nstreams, nbatches in 1..32 ("4 x 32 x 32" per kernel, "32 x 32").
* Constraints: nstb * nkpb * nspb <= 40 (10 nodes x 4 tasks) and
  tb_X * tb_sm_X <= 2048 (threads per SM), enforced by enumerating each block's valid tuples.
* Objective: Fig. 1 Case 4 at x_i = -50 + 100 rank_i / (K_i - 1), parameters in Table IV row order
  (noise free).

This module only builds the description (data) and the objective; the encoding and sampling
arithmetic live in oracle/space.py (test side) and csrc/space.cu (CUDA side).
"""
from __future__ import annotations

import numpy as np

from . import synthetic as syn

REAL, INT, ORDINAL, CATEGORICAL = 0, 1, 2, 3
KERNELS = ("DSCAL", "PAIR", "ZCOPY", "VEC", "ZVEC")


def _divisors(n):
    return [k for k in range(1, n + 1) if n % k == 0]


def table_iv():
    """Parameter list (Table IV row order) and constrained blocks of valid value-index tuples."""
    params, names = [], []

    def add(name, **p):
        names.append(name)
        params.append(p)

    add("nstb", kind=ORDINAL, values=_divisors(64))
    add("nkpb", kind=ORDINAL, values=_divisors(36))
    add("nspb", kind=ORDINAL, values=[1, 2])
    for k in KERNELS:
        add(f"u_{k}", kind=CATEGORICAL, K=4, labels=[1, 2, 4, 8])
        add(f"tb_{k}", kind=ORDINAL, values=list(range(32, 1025, 32)))
        add(f"tb_sm_{k}", kind=INT, lo=1, hi=32)
    add("nstreams", kind=INT, lo=1, hi=32)
    add("nbatches", kind=INT, lo=1, hi=32)
    blocks = []
    mpi = [(a, b, c) for a, x in enumerate(params[0]["values"]) for b, y in enumerate(params[1]["values"])
           for c, z in enumerate(params[2]["values"]) if x * y * z <= 40]
    blocks.append({"params": [0, 1, 2], "tuples": mpi})
    for j in range(5):
        tb, tbsm = 4 + 3 * j, 5 + 3 * j
        tup = [(a, b) for a, x in enumerate(params[tb]["values"]) for b in range(32)
               if x * (b + 1) <= 2048]
        blocks.append({"params": [tb, tbsm], "tuples": tup})
    return params, blocks, names


def nvals(p):
    if p["kind"] == INT:
        return int(p["hi"] - p["lo"]) + 1
    if p["kind"] == ORDINAL:
        return len(p["values"])
    if p["kind"] == CATEGORICAL:
        return int(p["K"])
    return 0


def objective(vidx, params):
    """R18: Case 4 of Fig. 1 at x_i = -50 + 100 rank_i/(K_i - 1); vidx: (n, 20) value indices."""
    vidx = np.atleast_2d(vidx)
    K = np.array([nvals(p) for p in params], dtype=np.float64)
    x = -50.0 + 100.0 * vidx / (K - 1.0)
    return syn.f20(x, 4)


def initial_design(params, blocks, count, seed):
    """`count` uniformly random valid configurations (value indices), seeded (5 in P:L254)."""
    g = np.random.Generator(np.random.Philox(key=(5 << 32) | (0 << 16) | seed))
    out = np.zeros((count, len(params)), dtype=np.int64)
    inblock = {i for b in blocks for i in b["params"]}
    for i, p in enumerate(params):
        if i not in inblock:
            out[:, i] = g.integers(0, nvals(p), count)
    for b in blocks:
        t = np.asarray(b["tuples"])[g.integers(0, len(b["tuples"]), count)]
        for j, i in enumerate(b["params"]):
            out[:, i] = t[:, j]
    return out
