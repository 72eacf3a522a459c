"""GPU parity: libgpbo (through the C ABI) against the float64 oracle on seeded inputs.

Tolerances and the argmax rule are the readings T1 / R11 in tests/helpers.py.
"""
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


def _fit(G, w):
    gpbo, ctx = G
    return ctx.fit(*H.pack(w), kernel=w.kernel)


IMPLS = [0, 1, 2, 3, 4]  # auto, CUDA-core, tcgen05, tcgen05 streamed, float64 direct (n <= 64)
FAST_IMPLS = [0, 1, 2, 3]  # implementations with a bracketed fast phase


# ------------------------------------------------------------------ fit (H1-H4)
@pytest.mark.parametrize("n,d", [(1, 1), (2, 3), (8, 2), (9, 3), (16, 2), (17, 5), (33, 8), (64, 4),
                                 (100, 5), (160, 20), (161, 9), (200, 20), (224, 12), (225, 7),
                                 (255, 35), (500, 60)])
@pytest.mark.parametrize("kernel", [gp.MATERN52, gp.RBF])
def test_fit_matches_oracle(G, n, d, kernel):
    w = gen.random_case(n * 7 + d, n, d, 4, kernel=kernel)
    m = _fit(G, w)
    om = H.oracle_fits(w)[0]
    assert m.status[0] in (0, 3) and m.jitter_k[0] == om.jitter_k
    L, Li, a = m.export(0)
    st = m.stats(0)
    assert abs(st["mean"] - om.mean) <= 1e-12 * max(1, abs(om.mean))
    assert abs(st["std"] - om.std) <= 1e-12 * om.std
    assert abs(st["best"] - om.best) <= 1e-12 * max(1, abs(om.best))
    np.testing.assert_allclose(L, om.L, rtol=0, atol=1e-12 * np.abs(om.L).max())
    Li_ref = np.linalg.inv(om.L)  # LAPACK inverse of the oracle's factor
    np.testing.assert_allclose(Li, Li_ref, rtol=0, atol=1e-9 * np.abs(Li_ref).max())
    np.testing.assert_allclose(a, om.alpha, rtol=0, atol=1e-7 * np.abs(om.alpha).max())


@pytest.mark.parametrize("ns", [[230, 17, 400], [217, 8, 1, 300, 64]])
def test_mixed_fit_batch_on_the_cluster_kernel(G, ns):
    """A batch whose largest search has n > 216 runs every search on the cluster fit (multicast G
    rows, per-search staging, CTAs that own no row of a small search): each search matches the
    oracle as in test_fit_matches_oracle, and its LML the oracle's."""
    w = gen.random_case(77 + len(ns), ns, [5 + (i % 3) for i in range(len(ns))], 4)
    m = _fit(G, w)
    oms = H.oracle_fits(w)
    lml = m.lml()
    for s, om in enumerate(oms):
        assert m.status[s] in (0, 3) and m.jitter_k[s] == om.jitter_k, s
        L, Li, a = m.export(s)
        np.testing.assert_allclose(L, om.L, rtol=0, atol=1e-12 * np.abs(om.L).max())
        Li_ref = np.linalg.inv(om.L)
        np.testing.assert_allclose(Li, Li_ref, rtol=0, atol=1e-9 * np.abs(Li_ref).max())
        np.testing.assert_allclose(a, om.alpha, rtol=0, atol=1e-7 * np.abs(om.alpha).max())
        from oracle import ml2 as oml2
        assert abs(lml[s] - oml2.lml(om)) <= 1e-9 * max(1.0, abs(lml[s])), s


def test_fit_jitter_escalation_and_failures(G):
    gpbo, ctx = G
    rng = np.random.default_rng(0)
    X = np.repeat(rng.random((6, 2)).astype(np.float32), 3, axis=0)
    y = rng.standard_normal(18)
    ls = np.array([0.3, 0.4], np.float32)
    m = ctx.fit([18], [2], X.ravel().copy(), y, ls, np.ones(1, np.float32),
                np.zeros(1, np.float32), kernel=gp.RBF)
    om = gp.fit(X, y, ls, 1.0, 0.0, gp.RBF)
    assert m.jitter_k[0] == om.jitter_k  # FP64 rounding never needs k > 0 here
    # no jitter can repair a negative noise variance -> rejected up front (EINVAL)
    with pytest.raises(gpbo.GpboError) as e:
        ctx.fit([3], [1], np.zeros(3, np.float32), np.arange(3.0), np.ones(1, np.float32),
                np.ones(1, np.float32), -np.ones(1, np.float32))
    assert e.value.status == gpbo.EINVAL
    y2 = y.copy()
    y2[3] = np.nan
    with pytest.raises(gpbo.GpboError) as e:
        ctx.fit([18], [2], X.ravel().copy(), y2, ls, np.ones(1, np.float32),
                np.full(1, 1e-4, np.float32))
    assert e.value.status == gpbo.EINVAL


def test_fit_degenerate(G):
    gpbo, ctx = G
    w = gen.random_case(3, 12, 2, 300)
    w.searches[0].y[:] = 4.2
    m = _fit(G, w)
    assert m.status[0] == gpbo.WDEGENERATE
    om = H.oracle_fits(w)[0]
    res = gp.score(om, w.Xstar[0])
    mu, var, ei = ctx_post(G, m, 0, w.Xstar[0])
    H.check_T1(om, res, mu, var, ei, "degenerate")


def ctx_post(G, m, s, Xs):
    gpbo, ctx = G
    return ctx.posterior(m, s, np.ascontiguousarray(Xs))


# ------------------------------------------------------------------ posterior (H6-H8)
CASES = [
    ("cfg1", lambda: gen.make(1)),
    ("cfg1_rbf", lambda: gen.make(1, kernel=gp.RBF)),
    ("cfg2", lambda: gen.make(2, M=8192)),
    ("cfg3", lambda: gen.make(3, S=8, M=2048)),
    ("cfg4", lambda: gen.make(4, M=2048)),
    ("n2", lambda: gen.random_case(1, 2, 3, 777)),
    ("n17_d9", lambda: gen.random_case(2, 17, 9, 1000)),
    ("n129_d33", lambda: gen.random_case(4, 129, 33, 1000)),
    ("n255_d64", lambda: gen.random_case(5, 255, 64, 600)),
    ("n511_d20", lambda: gen.random_case(6, 511, 20, 400)),
    # config-5 late-iteration shape (d = 35 encoded, n ~ 200): streamed tcgen05 layout
    ("n200_d35", lambda: gen.random_case(7, 200, 35, 1500)),
]


@pytest.mark.parametrize("impl", IMPLS)
@pytest.mark.parametrize("name,make", CASES, ids=[c[0] for c in CASES])
def test_posterior_matches_oracle(G, name, make, impl):
    gpbo, ctx = G
    ctx.set_score_impl(impl)
    try:
        w = make()
        if impl == 2 and max(x.X.shape[1] for x in w.searches) + 2 > 64:
            pytest.skip("outside the tcgen05 envelope (d + 2 > 64)")
        m = _fit(G, w)
        oms = H.oracle_fits(w)
        for s in range(w.S):
            res = gp.score(oms[s], w.Xstar[s])
            mu, var, ei = ctx.posterior(m, s, w.Xstar[s])
            H.check_T1(oms[s], res, mu, var, ei, f"{name}[{s}]")
            # the implementation that ran: forced stream, or auto -> streamed tcgen05 whenever
            # the resident image cannot hold the search (n16 > 256 or large d); d + 2 > 64 is
            # outside both tcgen05 envelopes (CUDA-core kernel)
            # (gp_posterior: the float64 direct kernel for small problems, else the float64
            # dense refine of every row -- implementation 5, no fast phase)
            n, d = w.searches[s].X.shape
            n16 = (n + 15) // 16 * 16
            if impl == 4 and n <= 64:
                assert ctx.last_impl == 4
            elif impl == 0 and n <= 64 and w.Xstar[s].shape[0] * n16 * n16 <= 1 << 24:
                assert ctx.last_impl == 4, (name, ctx.last_impl)
            else:
                assert ctx.last_impl == 5, (name, ctx.last_impl)
    finally:
        ctx.set_score_impl(0)


# ------------------------------------------------------------------ argmax (H9)
@pytest.mark.parametrize("impl", IMPLS)
@pytest.mark.parametrize("name,make", [
    ("cfg1", lambda: gen.make(1)),
    ("cfg2", lambda: gen.make(2, M=65536)),
    ("cfg3", lambda: gen.make(3, M=4096)),
    ("ragged", lambda: gen.random_case(9, [5, 64, 130], [3, 3, 3], [1, 129, 1000])),
    ("ragged_d", lambda: gen.random_case(10, [40, 7, 90], [2, 11, 5], [300, 64, 65])),
], ids=["cfg1", "cfg2", "cfg3", "ragged", "ragged_d"])
def test_argmax_matches_oracle(G, name, make, impl):
    gpbo, ctx = G
    ctx.set_score_impl(impl)
    try:
        w = make()
        m = _fit(G, w)
        Xs, off = H.pack_candidates(w)
        idx, ei = ctx.score_argmax(m, Xs, off)
        print(f"{name} impl={impl}: refined {ctx.last_refine_count} of {off[-1]}")
        oms = H.oracle_fits(w)
        for s in range(w.S):
            res = gp.score(oms[s], w.Xstar[s])
            H.check_argmax(res, int(idx[s]), f"{name}[{s}]")
            assert abs(ei[s] / oms[s].std - res.ei) <= H.TOL * max(res.ei, 1e-30)
    finally:
        ctx.set_score_impl(0)


@pytest.mark.parametrize("name,make", [
    # every search n > 112: the CTA-pair kernel (n16 + 16 > 128); ragged sizes give odd tile
    # counts (the pair tile's second half empty) and a 1-candidate search
    ("pair_multi", lambda: gen.random_case(21, [130, 200, 113], [3, 20, 7], [1, 300, 4097])),
    ("pair_cfg2", lambda: gen.make(2, M=65536 + 200)),
], ids=["pair_multi", "pair_cfg2"])
def test_pair_kernel_argmax_matches_oracle(G, name, make):
    """The CTA-pair tcgen05 kernel (cta_group::2) against the oracle, with the pair asserted."""
    gpbo, ctx = G
    ctx.set_score_impl(2)
    try:
        w = make()
        m = _fit(G, w)
        Xs, off = H.pack_candidates(w)
        idx, ei = ctx.score_argmax(m, Xs, off)
        assert ctx.last_impl == 2 and ctx.last_tc_pair == 1
        assert ctx.last_violations == 0
        oms = H.oracle_fits(w)
        for s in range(w.S):
            res = gp.score(oms[s], w.Xstar[s])
            H.check_argmax(res, int(idx[s]), f"{name}[{s}]")
            assert abs(ei[s] / oms[s].std - res.ei) <= H.TOL * max(res.ei, 1e-30)
    finally:
        ctx.set_score_impl(0)


def test_exact_tie_resolves_to_lowest_global_index(G):
    """R10 / S:L407: identical candidates tie bit-exactly; the lowest global index wins."""
    gpbo, ctx = G
    w = gen.random_case(11, 30, 4, 500)
    m = _fit(G, w)
    Xs = w.Xstar[0].copy()
    om = H.oracle_fits(w)[0]
    best = gp.score(om, Xs).idx
    Xs[400] = Xs[best]   # a later duplicate of the maximiser
    Xs[best // 2] = Xs[best]  # an earlier duplicate
    idx, _ = ctx.score_argmax(m, np.ascontiguousarray(Xs), [0, 500])
    assert idx[0] == best // 2


def test_sharded_scoring_is_bit_identical(G):
    """P13 (G-shard simulator): scoring contiguous shards separately with their global bases and
    taking the host-side max of (EI, -idx) reproduces the unsharded result bit-exactly."""
    gpbo, ctx = G
    w = gen.make(2, M=20000)
    m = _fit(G, w)
    Xs = w.Xstar[0]
    idx0, ei0 = ctx.score_argmax(m, Xs, [0, 20000])
    for shards in (2, 3, 8):
        per = -(-20000 // shards)
        picks = []
        for r in range(shards):
            a, b = r * per, min(20000, (r + 1) * per)
            i, e = ctx.score_argmax(m, np.ascontiguousarray(Xs[a:b]), [0, b - a], [a])
            picks.append((e[0], -i[0]))
        e, negi = max(picks)
        assert -negi == idx0[0] and e == ei0[0]


def test_device_and_host_memory_agree(G):
    import torch
    gpbo, ctx = G
    w = gen.make(3, S=4, M=1000)
    n, d, X, y, ls, sf2, sn2 = H.pack(w)
    mh = ctx.fit(n, d, X, y, ls, sf2, sn2)
    t = lambda a: torch.from_numpy(a).cuda()
    md = ctx.fit(n, d, t(X), t(y), t(ls), t(sf2), t(sn2))
    Xs, off = H.pack_candidates(w)
    ih, eh = ctx.score_argmax(mh, Xs, off)
    idv, edv = ctx.score_argmax(md, t(Xs), off)
    assert np.array_equal(ih, idv) and np.array_equal(eh, edv)
    mu_h, var_h, ei_h = ctx.posterior(mh, 1, w.Xstar[1])
    mu_d, var_d, ei_d = ctx.posterior(md, 1, t(w.Xstar[1]))
    assert np.array_equal(mu_h, mu_d.cpu().numpy()) and np.array_equal(ei_h, ei_d.cpu().numpy())


@pytest.mark.parametrize("case", ["cfg2", "cfg3", "cfg4"])
def test_chunked_host_feed_matches_device(G, case):
    """Host candidates large enough for the chunked feed (>= 2048 tiles: copies of chunk c + 1
    overlap the scoring of chunk c, one launch per chunk) give bit-identical keys to the
    device-resident single launch -- including chunk boundaries inside a search and between
    searches of a ragged batch, and the streamed kernel (cfg4)."""
    import torch
    gpbo, ctx = G
    w = {"cfg2": lambda: gen.make(2, M=1 << 19),
         "cfg3": lambda: gen.random_case(31, [100, 60, 100, 37], [5, 5, 7, 5],
                                         [70001, 1, 131072, 99999]),
         "cfg4": lambda: gen.make(4, M=300000)}[case]()
    n, d, X, y, ls, sf2, sn2 = H.pack(w)
    m = ctx.fit(n, d, X, y, ls, sf2, sn2, kernel=w.kernel)
    Xs, off = H.pack_candidates(w)
    Xp = torch.from_numpy(Xs).pin_memory()
    ih, eh = ctx.score_argmax(m, Xp, off)
    impl_h = ctx.last_impl
    idv, edv = ctx.score_argmax(m, torch.from_numpy(Xs).cuda(), off)
    assert impl_h == ctx.last_impl and impl_h in (2, 3)
    assert np.array_equal(ih, idv) and np.array_equal(eh, edv), (ih, idv, eh, edv)
    m.free()


@pytest.mark.parametrize("impl", IMPLS)
def test_empty_and_single_candidate_searches(G, impl):
    """A search with no candidates returns idx -1 (key 0 = "no candidate"); a one-candidate search
    returns that candidate; the others are unaffected -- on every implementation."""
    gpbo, ctx = G
    ctx.set_score_impl(impl)
    try:
        w = gen.random_case(41, [30, 12, 50, 7], [4, 4, 6, 3], [500, 0, 1, 300], S=4)
        m = _fit(G, w)
        Xs, off = H.pack_candidates(w)
        idx, ei = ctx.score_argmax(m, Xs, off)
        assert int(idx[1]) == -1
        assert int(idx[2]) == 0
        oms = H.oracle_fits(w)
        for s in (0, 2, 3):
            res = gp.score(oms[s], w.Xstar[s])
            H.check_argmax(res, int(idx[s]), f"empty[{s}]")
    finally:
        ctx.set_score_impl(0)


def test_nan_candidate_is_never_chosen(G):
    gpbo, ctx = G
    w = gen.random_case(12, 20, 3, 256)
    m = _fit(G, w)
    Xs = w.Xstar[0].copy()
    om = H.oracle_fits(w)[0]
    best = gp.score(om, Xs).idx
    Xs[best, 1] = np.nan
    idx, _ = ctx.score_argmax(m, np.ascontiguousarray(Xs), [0, 256])
    assert idx[0] != best and idx[0] >= 0


# ------------------------------------------------------------------ fast-phase bracket
BRACKET_CASES = [
    ("cfg1", lambda: gen.make(1)),
    ("cfg1_rbf", lambda: gen.make(1, kernel=gp.RBF)),
    ("cfg2", lambda: gen.make(2, M=16384)),
    ("cfg2_bo", lambda: gen.make(2, M=8192, layout="bo")),
    ("cfg3", lambda: gen.make(3, S=16, M=4096)),
    ("cfg4", lambda: gen.make(4, M=2048)),
    ("clustered", lambda: gen.random_case(21, 150, 10, 4096, clustered=True, sn2=1e-6)),
    ("rbf_clustered", lambda: gen.random_case(22, 80, 4, 4096, clustered=True, sn2=1e-6,
                                              kernel=gp.RBF)),
]


@pytest.mark.parametrize("impl", FAST_IMPLS)
@pytest.mark.parametrize("name,make", BRACKET_CASES, ids=[c[0] for c in BRACKET_CASES])
def test_fast_phase_brackets_contain_oracle(G, name, make, impl):
    """The argmax filter is sound only if, for EVERY candidate, the fast phase's bounds contain
    the oracle: |mu32 - mu| <= dmu, |var32 - var| <= dvar, EI_lo <= EI <= EI_hi."""
    import json
    import os
    import torch
    gpbo, ctx = G
    ctx.set_score_impl(impl)
    try:
        w = make()
        m = _fit(G, w)
        oms = H.oracle_fits(w)
        stats = []
        for s in range(w.S):
            res = gp.score(oms[s], w.Xstar[s])
            o = {k: v.cpu().numpy().astype(np.float64) for k, v in
                 ctx.debug_fast_phase(m, s, torch.from_numpy(w.Xstar[s]).cuda()).items()}
            emu = np.abs(o["mu"] - res.mu)
            evar = np.abs(o["var"] - res.var)
            stats.append(dict(s=s, mu_ratio=float((emu / o["dmu"]).max()),
                              var_ratio=float((evar / o["dvar"]).max()),
                              mu_err=float(emu.max()), var_err=float(evar.max()),
                              alpha_l1=float(np.abs(oms[s].alpha).sum())))
            # (the debug output stores mu~ as float32: its rounding, 2^-24 |mu~|, is not part of
            # the fast phase's bound -- the precise-mean tier's float64 mean has dmu ~ 1e-12)
            assert np.all(emu <= o["dmu"] + 6e-8 * np.abs(res.mu)), (name, s, stats[-1])
            assert np.all(evar <= o["dvar"]), (name, s, stats[-1])
            live = res.ei_all >= 1e-30  # below, float32 EI underflows on both sides (R11)
            assert np.all(o["ei_lo"][live] <= res.ei_all[live] * (1 + 1e-12)), (name, s)
            assert np.all(o["ei_hi"][live] >= res.ei_all[live] * (1 - 1e-12)), (name, s)
        os.makedirs("gpurun_out", exist_ok=True)
        with open(f"gpurun_out/bracket_{name}_{impl}.json", "w") as f:
            json.dump(stats, f)
    finally:
        ctx.set_score_impl(0)


# ------------------------------------------------------------------ asynchronous fit
def test_async_fit_matches_sync(G):
    """gp_fit_async + ei_score_argmax == gp_fit + ei_score_argmax bit for bit (incl. a raw-unit
    incumbent standardised on the device), and gp_model_sync reports the fit's statuses."""
    gpbo, ctx = G
    w = gen.make(3, M=4096)
    Xs = np.ascontiguousarray(np.concatenate(w.Xstar), np.float32)
    off = np.zeros(w.S + 1, np.int64)
    off[1:] = np.cumsum([x.shape[0] for x in w.Xstar])
    ms = ctx.fit(*H.pack(w), kernel=w.kernel)
    ma = ctx.fit(*H.pack(w), kernel=w.kernel, wait=False)
    i0, e0 = ctx.score_argmax(ms, Xs, off)
    i1, e1 = ctx.score_argmax(ma, Xs, off)
    assert np.array_equal(i0, i1) and np.array_equal(e0.view(np.uint32), e1.view(np.uint32))
    best = np.array([s.y.min() - 0.1 for s in w.searches])
    ma2 = ctx.fit(*H.pack(w), kernel=w.kernel, wait=False)
    i2, e2 = ctx.score_argmax(ma2, Xs, off, best=best)
    i3, e3 = ctx.score_argmax(ms, Xs, off, best=best)
    assert np.array_equal(i2, i3) and np.array_equal(e2.view(np.uint32), e3.view(np.uint32))
    assert np.array_equal(ma.status, ms.status) and np.array_equal(ma.jitter_k, ms.jitter_k)
    for s in range(w.S):
        assert ma.stats(s) == ms.stats(s)
    for m in (ms, ma, ma2):
        m.free()


def test_async_fit_failed_search_scores_nothing(G):
    """A non-finite input in one search: the asynchronous fit is enqueued (no host error), that
    search returns idx -1 on the device path, the other searches are unaffected, and
    gp_model_sync reports EINVAL."""
    gpbo, ctx = G
    w = gen.make(3, M=2048)
    n, d, X, y, ls, sf2, sn2 = H.pack(w)
    y = y.copy()
    y[n[0] + 3] = np.nan  # search 1
    Xs = np.ascontiguousarray(np.concatenate(w.Xstar), np.float32)
    off = np.zeros(w.S + 1, np.int64)
    off[1:] = np.cumsum([x.shape[0] for x in w.Xstar])
    ma = ctx.fit(n, d, X, y, ls, sf2, sn2, kernel=w.kernel, wait=False)
    idx, ei = ctx.score_argmax(ma, Xs, off)
    assert idx[1] == -1 and ei[1] == 0.0
    y_ok = H.pack(w)[3]
    ms = ctx.fit(n, d, X, y_ok, ls, sf2, sn2, kernel=w.kernel)
    i0, _ = ctx.score_argmax(ms, Xs, off)
    keep = [s for s in range(w.S) if s != 1]
    assert np.array_equal(idx[keep], i0[keep])
    st = np.zeros(w.S, np.int32)
    rc = gpbo.load().gp_model_sync(ctx.handle, ma.handle, st.ctypes.data, None)
    assert rc == gpbo.EINVAL and st[1] == gpbo.EINVAL
    ma.free()
    ms.free()
