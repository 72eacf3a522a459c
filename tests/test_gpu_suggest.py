"""H0/H5 + bo_suggest_batch on the GPU against the oracle (oracle/space.py, oracle/gp.py).

Candidate coordinates are compared bit-exactly (both sides implement the documented Philox
mapping independently); the suggestion follows the argmax rule R11 on the same candidates.
"""
import numpy as np
import pytest

from oracle import gp
from oracle import space as osp
from tests import helpers as H
from workloads import rttddft

pytestmark = pytest.mark.gpu

MIXED = [{"kind": 0, "lo": -50.0, "hi": 50.0}, {"kind": 1, "lo": 1, "hi": 32},
         {"kind": 2, "values": [1, 2, 4, 8, 16]}, {"kind": 3, "K": 4},
         {"kind": 0, "lo": 0.0, "hi": 1.0}]
MIXED_BLOCKS = [{"params": [1, 2], "tuples": [(a, b) for a in range(32) for b in range(5)
                                              if (a + 1) * [1, 2, 4, 8, 16][b] <= 64]}]


@pytest.fixture(scope="module")
def G():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2403_08131_b200 import gpbo
    ctx = gpbo.Context(device=0)
    yield gpbo, ctx
    ctx.close()


@pytest.mark.parametrize("which", ["table_iv", "mixed"])
def test_generation_is_bit_exact(G, which):
    gpbo, ctx = G
    if which == "table_iv":
        params, blocks, _ = rttddft.table_iv()
    else:
        params, blocks = MIXED, MIXED_BLOCKS
    sp = gpbo.Space(ctx, params, blocks)
    ref = osp.Space(params, blocks)
    assert sp.dim == ref.dim
    for seed, s, t, first in ((1, 0, 0, 0), (0xDEADBEEF12345678, 3, 17, 123456), (7, 1, 2, 2 ** 31)):
        got = sp.sample(seed, s, t, first, 3000)
        exp = ref.sample(seed, s, t, np.arange(first, first + 3000))
        assert np.array_equal(got.view(np.uint32), exp.view(np.uint32)), (seed, s, t)
    # host-side encoding of decoded raw values reproduces the generator's encoding (H0)
    vals = ref.sample_values(5, 0, 1, np.arange(200))
    raw = ref.raw_values(vals)
    assert np.array_equal(sp.encode(raw), ref.encode_values(vals))


def _history(params, blocks, n0, seed):
    vidx = rttddft.initial_design(params, blocks, n0, seed)
    y = rttddft.objective(vidx, params)
    ref = osp.Space(params, blocks)
    return vidx, y, ref.encode_values(vidx.astype(float))


def test_suggest_matches_oracle_and_decodes(G):
    gpbo, ctx = G
    params, blocks, _ = rttddft.table_iv()
    sp = gpbo.Space(ctx, params, blocks)
    ref = osp.Space(params, blocks)
    vidx, y, X = _history(params, blocks, 24, 3)
    d = X.shape[1]
    ls = np.full(d, 0.4 * np.sqrt(d), np.float32)
    m = ctx.fit([len(y)], [d], np.ascontiguousarray(X.ravel()), y, ls, np.ones(1, np.float32),
                np.full(1, 1e-4, np.float32))
    M, seed, it = 8192, 42, 7
    idx, xr, ei = gpbo.suggest(ctx, m, [sp], [M], seed, it, dedup=True)
    cand = ref.sample(seed, 0, it, np.arange(M))
    om = gp.fit(X, y, ls, 1.0, 1e-4)
    res = gp.score(om, cand)
    H.check_argmax(res, int(idx[0]), "suggest")
    assert abs(ei[0] / om.std - res.ei) <= H.TOL * max(res.ei, 1e-30)
    vals = ref.sample_values(seed, 0, it, [int(idx[0])])
    assert np.array_equal(xr[0], ref.raw_values(vals)[0])
    # the suggestion satisfies the Table IV constraints
    nstb, nkpb, nspb = xr[0][0], xr[0][1], xr[0][2]
    assert nstb * nkpb * nspb <= 40
    for j in range(5):
        assert xr[0][4 + 3 * j] * xr[0][5 + 3 * j] <= 2048


def test_dedup_masks_observed_configurations(G):
    """R14 / S:L432: a candidate identical to an observation is skipped (next-best EI)."""
    gpbo, ctx = G
    sp = gpbo.Space(ctx, MIXED, MIXED_BLOCKS)
    ref = osp.Space(MIXED, MIXED_BLOCKS)
    seed, it, M = 11, 2, 2048
    cand = ref.sample(seed, 0, it, np.arange(M))
    g = np.random.default_rng(0)
    X = np.concatenate([g.random((10, ref.dim)).astype(np.float32), cand[[5, 900]]])
    y = g.standard_normal(12)
    y[10:] = y.min() - 1.0  # the duplicated points are the best observations
    ls = np.full(ref.dim, 0.5, np.float32)
    m = ctx.fit([12], [ref.dim], np.ascontiguousarray(X.ravel()), y, ls, np.ones(1, np.float32),
                np.full(1, 1e-4, np.float32))
    idx, _, _ = gpbo.suggest(ctx, m, [sp], [M], seed, it, dedup=True)
    om = gp.fit(X, y, ls, 1.0, 1e-4)
    mu, var = gp.posterior(om, cand)
    ei = gp.expected_improvement(mu, var, om.best)
    ei[[5, 900]] = -1.0  # masked
    assert int(idx[0]) not in (5, 900)
    top = int(np.argmax(ei))
    srt = np.sort(ei)[::-1]
    if (srt[0] - srt[1]) > 1e-3 * srt[0]:
        assert int(idx[0]) == top


def test_replay_teacher_forced(G):
    """Config-5 style replay (reduced): 12 BO iterations on the Table IV space; at every iteration
    the oracle scores the same candidates from the same history (teacher forcing)."""
    gpbo, ctx = G
    params, blocks, _ = rttddft.table_iv()
    sp = gpbo.Space(ctx, params, blocks)
    ref = osp.Space(params, blocks)
    vidx, y, X = _history(params, blocks, 5, 9)
    d = X.shape[1]
    ls = np.full(d, 0.4 * np.sqrt(d), np.float32)
    M, seed = 2048, 1234
    for it in range(12):
        m = ctx.fit([len(y)], [d], np.ascontiguousarray(X.ravel()), y, ls,
                    np.ones(1, np.float32), np.full(1, 1e-4, np.float32))
        idx, xr, _ = gpbo.suggest(ctx, m, [sp], [M], seed, it, dedup=True)
        cand = ref.sample(seed, 0, it, np.arange(M))
        om = gp.fit(X, y, ls, 1.0, 1e-4)
        mu, var = gp.posterior(om, cand)
        ei = gp.expected_improvement(mu, var, om.best)
        dup = (cand[:, None, :] == X[None, :, :]).all(-1).any(-1)
        ei[dup] = -1.0
        srt = np.sort(ei)[::-1]
        if srt[0] >= 1e-30 and (srt[0] - srt[1]) > 1e-3 * srt[0]:
            assert int(idx[0]) == int(np.argmax(ei)), it
        v = ref.sample_values(seed, 0, it, [int(idx[0])]).astype(np.int64)
        X = np.concatenate([X, ref.encode_values(v.astype(float))])
        y = np.concatenate([y, rttddft.objective(v, params)])


@pytest.mark.parametrize("n_dup", [1, 400])
def test_dedup_with_a_full_hash_table(G, n_dup):
    """The generator's dedup (space.cu: a shared-memory hash table of the training encodings,
    exact comparison on hash hits) with up to 500 training rows, n_dup of them equal to
    candidates of this call: no masked candidate is suggested, and the suggestion is the oracle's
    argmax over the unmasked candidates (R14 / S:L432; R11 where the gap is decisive)."""
    gpbo, ctx = G
    sp = gpbo.Space(ctx, MIXED, MIXED_BLOCKS)
    ref = osp.Space(MIXED, MIXED_BLOCKS)
    seed, it, M = 5, 3, 4096
    cand = ref.sample(seed, 0, it, np.arange(M))
    g = np.random.default_rng(n_dup)
    dup = np.sort(g.choice(M, n_dup, replace=False))
    X = np.concatenate([g.random((500 - n_dup, ref.dim)).astype(np.float32), cand[dup]])
    y = g.standard_normal(500)
    y[500 - n_dup:] -= 1.0  # the duplicated configurations are among the best observations
    ls = np.full(ref.dim, 0.5, np.float32)
    m = ctx.fit([500], [ref.dim], np.ascontiguousarray(X.ravel()), y, ls, np.ones(1, np.float32),
                np.full(1, 1e-4, np.float32))
    idx, _, _ = gpbo.suggest(ctx, m, [sp], [M], seed, it, dedup=True)
    om = gp.fit(X, y, ls, 1.0, 1e-4)
    mu, var = gp.posterior(om, cand)
    ei = gp.expected_improvement(mu, var, om.best)
    masked = np.zeros(M, bool)
    for r in X:  # the oracle's definition: exact equality with any observed configuration
        masked |= np.all(cand == r, axis=1)
    assert masked.sum() == n_dup
    ei[masked] = -1.0
    assert not masked[int(idx[0])]
    srt = np.sort(ei)[::-1]
    if (srt[0] - srt[1]) > 1e-3 * srt[0]:
        assert int(idx[0]) == int(np.argmax(ei))
    m.free()


def test_suggest_right_after_an_async_device_fit(G):
    """bo_suggest_batch draws its candidates on a side stream that waits only for the latest Gram
    pre-pass (which copies the caller's device X into the model -- the dedup's input): after an
    asynchronous fit from device arrays, with training rows that equal candidates of the call,
    the masked set and the suggestion must still be the oracle's, on every one of several
    back-to-back fits (a stale or unfinished X copy would leak a duplicate or mask a wrong row)."""
    import torch
    gpbo, ctx = G
    sp = gpbo.Space(ctx, MIXED, MIXED_BLOCKS)
    ref = osp.Space(MIXED, MIXED_BLOCKS)
    M = 4096
    dev = torch.device("cuda", 0)
    for rep in range(4):
        seed, it = 21 + rep, rep
        cand = ref.sample(seed, 0, it, np.arange(M))
        g = np.random.default_rng(100 + rep)
        dup = np.sort(g.choice(M, 150, replace=False))
        X = np.concatenate([g.random((50, ref.dim)).astype(np.float32), cand[dup]])
        y = g.standard_normal(200)
        y[50:] -= 1.5
        ls = np.full(ref.dim, 0.5, np.float32)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        m = ctx.fit([200], [ref.dim], t(X.ravel()), t(y), t(ls), t(np.ones(1, np.float32)),
                    t(np.full(1, 1e-4, np.float32)), wait=False)
        idx, _, _ = gpbo.suggest(ctx, m, [sp], [M], seed, it, dedup=True)
        om = gp.fit(X, y, ls, 1.0, 1e-4)
        mu, var = gp.posterior(om, cand)
        ei = gp.expected_improvement(mu, var, om.best)
        ei[dup] = -1.0
        assert int(idx[0]) not in set(dup.tolist()), rep
        srt = np.sort(ei)[::-1]
        if (srt[0] - srt[1]) > 1e-3 * srt[0]:
            assert int(idx[0]) == int(np.argmax(ei)), rep
        m.free()


def test_fixed_parameters_in_generation_encoding_and_decode(G):
    """GPBO_P_FIXED: no encoded column and no Philox word (bit-exact against the oracle's space
    with the same fixed parameters), gpbo_space_encode drops them, and bo_suggest_batch decodes
    them to their constant."""
    gpbo, ctx = G
    params = [MIXED[0], {"kind": 4, "lo": 64.0}] + MIXED[1:] + [{"kind": 4, "lo": -1.25}]
    nfix = len(MIXED) + 1  # index of the second fixed parameter
    shift = lambda b: {"params": [p + 1 for p in b["params"]], "tuples": b["tuples"]}
    blocks = [shift(b) for b in MIXED_BLOCKS]
    sp = gpbo.Space(ctx, params, blocks)
    ref = osp.Space(params, blocks)
    ref0 = osp.Space(MIXED, MIXED_BLOCKS)
    assert sp.dim == ref.dim == ref0.dim
    got = sp.sample(99, 0, 4, 0, 2048)
    assert np.array_equal(got.view(np.uint32), ref.sample(99, 0, 4, np.arange(2048)).view(np.uint32))
    assert np.array_equal(got.view(np.uint32), ref0.sample(99, 0, 4, np.arange(2048)).view(np.uint32))
    raw = ref.raw_values(ref.sample_values(99, 0, 4, np.arange(3)))
    assert np.array_equal(sp.encode(raw), got[:3])
    g = np.random.default_rng(5)
    X = g.random((30, ref.dim)).astype(np.float32)
    y = g.standard_normal(30)
    ls = np.full(ref.dim, 0.5, np.float32)
    m = ctx.fit([30], [ref.dim], np.ascontiguousarray(X.ravel()), y, ls, np.ones(1, np.float32),
                np.full(1, 1e-4, np.float32))
    idx, xr, _ = gpbo.suggest(ctx, m, [sp], [4096], 99, 4, dedup=True)
    assert xr[0][1] == 64.0 and xr[0][nfix] == -1.25
    exp = ref.raw_values(ref.sample_values(99, 0, 4, np.array([int(idx[0])])))[0]
    assert np.array_equal(xr[0], exp)
    m.free()
