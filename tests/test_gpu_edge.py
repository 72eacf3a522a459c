"""GPU: the H10 all-reduce path on a 1-rank NCCL communicator, and invalid-row handling of the
small-problem float64 direct kernel (NaN rows must never become suggestions).

Tolerances / argmax rule: tests/helpers.py (T1 / R11)."""
import numpy as np
import pytest

from oracle import gp
from tests import helpers as H
from workloads import gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2403_08131_b200 import gpbo
    ctx = gpbo.Context(device=0)
    yield gpbo, ctx
    ctx.close()


@pytest.mark.parametrize("case", ["cfg2", "cfg3"])
def test_one_rank_nccl_allreduce_matches_plain(G, case):
    """H10 (ncclAllReduce(max, u64) of the packed keys) runs on a 1-rank communicator and leaves
    the result bit-identical to the call without a communicator; the oracle agrees (R11)."""
    gpbo, ctx = G
    w = gen.make(2, M=1 << 16) if case == "cfg2" else gen.make(3, S=8, M=4096)
    nctx = gpbo.Context(device=0, nranks=1, rank=0, nccl_id=gpbo.nccl_unique_id())
    try:
        m0 = ctx.fit(*H.pack(w), kernel=w.kernel)
        m1 = nctx.fit(*H.pack(w), kernel=w.kernel)
        Xs, off = H.pack_candidates(w)
        i0, e0 = ctx.score_argmax(m0, Xs, off)
        c0 = nctx.collectives
        i1, e1 = nctx.score_argmax(m1, Xs, off)
        assert nctx.collectives == c0 + 1 and ctx.collectives == 0
        assert np.array_equal(i0, i1) and np.array_equal(e0.view(np.uint32), e1.view(np.uint32))
        for s, om in enumerate(H.oracle_fits(w)[:4]):
            H.check_argmax(gp.score(om, w.Xstar[s]), int(i1[s]), f"nccl1[{s}]")
        m0.free()
        m1.free()
    finally:
        nctx.close()


@pytest.mark.parametrize("impl", [0, 1, 2, 4])
def test_fully_masked_pool_returns_no_candidate(G, impl):
    """Every candidate of search 0 is NaN (as a fully dedup-masked pool): idx -1 on every
    implementation, while search 1 is unaffected."""
    gpbo, ctx = G
    ctx.set_score_impl(impl)
    try:
        w = gen.random_case(51, [20, 24], [3, 3], [300, 300], S=2)
        m = ctx.fit(*H.pack(w), kernel=w.kernel)
        Xs0 = np.full_like(w.Xstar[0], np.nan)
        Xs = np.ascontiguousarray(np.concatenate([Xs0.ravel(), w.Xstar[1].ravel()]), np.float32)
        idx, ei = ctx.score_argmax(m, Xs, [0, 300, 600])
        assert int(idx[0]) == -1 and float(ei[0]) == 0.0
        om = H.oracle_fits(w)[1]
        H.check_argmax(gp.score(om, w.Xstar[1]), int(idx[1]), "masked[1]")
        m.free()
    finally:
        ctx.set_score_impl(0)


@pytest.mark.parametrize("impl", [0, 4])
def test_nan_rows_on_direct_path(G, impl):
    """Direct float64 kernel (impl 4; also auto at this size): a NaN row is never chosen and its
    posterior outputs are NaN; every other row still meets T1."""
    gpbo, ctx = G
    ctx.set_score_impl(impl)
    try:
        w = gen.random_case(13, 20, 3, 256)
        m = ctx.fit(*H.pack(w), kernel=w.kernel)
        om = H.oracle_fits(w)[0]
        Xs = w.Xstar[0].copy()
        best = gp.score(om, Xs).idx
        Xs[best, 0] = np.nan
        Xs = np.ascontiguousarray(Xs)
        idx, _ = ctx.score_argmax(m, Xs, [0, 256])
        assert ctx.last_impl == 4
        assert int(idx[0]) != best and int(idx[0]) >= 0
        mu, var, ei = ctx.posterior(m, 0, Xs)
        assert np.isnan(mu[best]) and np.isnan(var[best]) and np.isnan(ei[best])
        keep = np.arange(256) != best
        res = gp.score(om, w.Xstar[0][keep])
        H.check_T1(om, res, mu[keep], var[keep], ei[keep], "direct-nan")
        m.free()
    finally:
        ctx.set_score_impl(0)

