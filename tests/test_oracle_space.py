"""Pins of the H0/H5 oracle (oracle/space.py): Philox known-answer vectors, the value mappings,
uniformity over the valid set, encoding, and the Table IV space counts."""
import numpy as np

from oracle import space as sp
from workloads import rttddft


def test_p16_philox_known_answer_vectors():
    """P16: Random123 philox4x32-10 KATs (also reproduced in SURVEY.md §8(c))."""
    assert sp.philox4x32_10((0, 0, 0, 0), (0, 0)) == (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)
    m = 0xFFFFFFFF
    assert sp.philox4x32_10((m, m, m, m), (m, m)) == (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)
    assert sp.philox4x32_10((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344),
                            (0xa4093822, 0x299f31d0)) == (0xd16cfe09, 0x94fdcceb, 0x5001e420,
                                                          0x24126ea1)


def test_vectorised_philox_matches_scalar():
    rng = np.random.default_rng(0)
    c = rng.integers(0, 2 ** 32, size=(4, 50), dtype=np.uint64)
    out = sp.philox_vec(*c, 0x12345678, 0x9abcdef0)
    for j in range(50):
        ref = sp.philox4x32_10(tuple(int(x) for x in c[:, j]), (0x12345678, 0x9abcdef0))
        assert tuple(int(o[j]) for o in out) == ref


def test_table_iv_counts():
    """R16 counts: 51 valid MPI triples of 126, 216 valid (tb, tb_sm) of 1024, d_enc = 35."""
    params, blocks, names = rttddft.table_iv()
    assert len(params) == 20 and names[0] == "nstb" and names[-1] == "nbatches"
    assert len(blocks[0]["tuples"]) == 51 and 7 * 9 * 2 == 126
    assert all(len(b["tuples"]) == 216 for b in blocks[1:])
    S = sp.Space(params, blocks)
    assert S.dim == 35 and S.units == 7 + 6


def test_sampling_is_uniform_over_valid_tuples_and_valid():
    params, blocks, _ = rttddft.table_iv()
    S = sp.Space(params, blocks)
    v = S.sample_values(seed=7, search=0, iteration=3, idx=np.arange(200000))
    # every sample satisfies the constraints
    nstb = np.asarray(params[0]["values"])[v[:, 0].astype(int)]
    nkpb = np.asarray(params[1]["values"])[v[:, 1].astype(int)]
    nspb = np.asarray(params[2]["values"])[v[:, 2].astype(int)]
    assert np.all(nstb * nkpb * nspb <= 40)
    for j in range(5):
        tb = np.asarray(params[4 + 3 * j]["values"])[v[:, 4 + 3 * j].astype(int)]
        assert np.all(tb * (v[:, 5 + 3 * j] + 1) <= 2048)
    # the MPI tuple index is uniform over its 51 valid tuples (chi-square, 50 dof, p ~ 1e-6 bound)
    tup = {tuple(t): i for i, t in enumerate(blocks[0]["tuples"])}
    ids = np.array([tup[(int(a), int(b), int(c))] for a, b, c in v[:, :3]])
    cnt = np.bincount(ids, minlength=51)
    exp = len(ids) / 51
    assert ((cnt - exp) ** 2 / exp).sum() < 110


def test_value_mappings_and_encoding():
    """u = (w >> 8) 2^-24 for reals; index (w >> 8) K >> 24 for K values; one-hot categoricals."""
    params = [{"kind": sp.REAL, "lo": -50.0, "hi": 50.0}, {"kind": sp.INT, "lo": 1, "hi": 5},
              {"kind": sp.ORDINAL, "values": [1, 2, 4]}, {"kind": sp.CATEGORICAL, "K": 3}]
    S = sp.Space(params)
    idx = np.arange(64)
    W = S.words(99, 2, 5, idx)
    v = S.sample_values(99, 2, 5, idx)
    assert np.array_equal(v[:, 0], (W[0] >> np.uint64(8)).astype(np.float64) / 2 ** 24)
    assert np.array_equal(v[:, 1], ((W[1] >> np.uint64(8)) * np.uint64(5) >> np.uint64(24)).astype(float))
    enc = S.encode_values(v)
    assert enc.shape == (64, 1 + 1 + 1 + 3) and enc.dtype == np.float32
    assert np.array_equal(enc[:, 0], v[:, 0].astype(np.float32))
    assert np.array_equal(enc[:, 1], (v[:, 1] / 4).astype(np.float32))
    assert np.all(enc[:, 3:].sum(1) == 1)
    raw = S.raw_values(v)
    assert np.all((raw[:, 0] >= -50) & (raw[:, 0] < 50)) and set(raw[:, 2]) <= {1, 2, 4}
    # counters: word u of block b is output[u % 4] of Philox(ctr = (i, s, t, u // 4))
    ref = sp.philox4x32_10((5, 2, 5, 0), (99, 0))
    assert int(W[1][5]) == ref[1]


def test_fixed_parameters_draw_nothing_and_encode_nothing():
    """H0 'fixed params dropped': inserting FIXED parameters
    anywhere leaves every other parameter's draw and encoding unchanged (they take no Philox word
    and no column), and their raw value is the given constant."""
    base = [{"kind": sp.REAL, "lo": -50.0, "hi": 50.0}, {"kind": sp.INT, "lo": 1, "hi": 32},
            {"kind": sp.CATEGORICAL, "K": 4}, {"kind": sp.ORDINAL, "values": [1, 2, 4, 8]}]
    fixed = [base[0], {"kind": sp.FIXED, "lo": 64.0}, base[1], base[2],
             {"kind": sp.FIXED, "lo": -3.5}, base[3]]
    a, b = sp.Space(base), sp.Space(fixed)
    assert b.dim == a.dim == 1 + 1 + 4 + 1
    idx = np.arange(2000)
    for seed, s, t in ((7, 0, 0), (2 ** 40 + 5, 3, 11)):
        ea, eb = a.sample(seed, s, t, idx), b.sample(seed, s, t, idx)
        assert np.array_equal(ea.view(np.uint32), eb.view(np.uint32))
        ra = a.raw_values(a.sample_values(seed, s, t, idx))
        rb = b.raw_values(b.sample_values(seed, s, t, idx))
        assert np.array_equal(rb[:, [0, 2, 3, 5]], ra)
        assert np.all(rb[:, 1] == 64.0) and np.all(rb[:, 4] == -3.5)
