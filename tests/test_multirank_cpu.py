"""World-size-2 gloo test of the multi-GPU protocol on CPU.

Each rank takes its contiguous shard of the candidate pool (workloads.gen sharding, the same
rows bench.py hands to the library), scores it with the oracle, packs the per-search argmax into
the library's 64-bit key (float32 bits of EI~ << 32 | 2^32-1-global_idx), and the ranks combine
keys with a MAX all-reduce -- the operation the library performs with ncclAllReduce(ncclMax) on
GPUs.  The decoded result must equal the unsharded oracle argmax bit-exactly, and the NCCL unique
id travels with broadcast_object_list as in bench.py.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import gp
from workloads import gen


def pack_key(ei, gidx):
    e = np.float32(ei if ei > 0 else 0.0)
    bits = int(np.frombuffer(e.tobytes(), dtype=np.uint32)[0])
    return (bits << 32) | (0xFFFFFFFF - int(gidx))


def decode_key(k):
    idx = 0xFFFFFFFF - (k & 0xFFFFFFFF)
    ei = np.frombuffer(np.uint32(k >> 32).tobytes(), dtype=np.float32)[0]
    return idx, float(ei)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, M, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    obj = [bytes(range(128)) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    assert obj[0] == bytes(range(128))
    w = gen.make(cfg, n=30, M=M, S=3 if cfg == 3 else None, rank=rank, world=world)
    keys = []
    for s, (srch, Xs) in enumerate(zip(w.searches, w.Xstar)):
        m = gp.fit(srch.X, srch.y, srch.lengthscale, srch.sf2, srch.sn2)
        if Xs.shape[0] == 0:
            keys.append(0)
            continue
        ei = gp.expected_improvement(*gp.posterior(m, Xs), m.best).astype(np.float32)
        top = max(range(len(ei)), key=lambda i: (ei[i], -i))
        keys.append(pack_key(ei[top], w.m_global_base[s] + top))
    # keys < 2^63 (EI bits of a non-negative float32 < 2^31), so a signed int64 MAX is exact
    t = torch.tensor(keys, dtype=torch.int64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    out[rank] = t.tolist()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg,M", [(2, 3001), (3, 1000)])
def test_two_rank_max_allreduce_matches_unsharded(cfg, M):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), cfg, M, out), nprocs=world, join=True)
    assert out[0] == out[1]
    full = gen.make(cfg, n=30, M=M, S=3 if cfg == 3 else None)
    for s, (srch, Xs) in enumerate(zip(full.searches, full.Xstar)):
        m = gp.fit(srch.X, srch.y, srch.lengthscale, srch.sf2, srch.sn2)
        ei = gp.expected_improvement(*gp.posterior(m, Xs), m.best).astype(np.float32)
        top = max(range(len(ei)), key=lambda i: (ei[i], -i))
        idx, e = decode_key(out[0][s])
        assert idx == top and e == float(ei[top])


def test_key_order_is_ei_then_lowest_index():
    assert pack_key(0.5, 7) > pack_key(0.25, 1)
    assert pack_key(0.5, 3) > pack_key(0.5, 4)       # tie -> lower global index wins
    assert pack_key(0.0, 0) > pack_key(-0.0, 5) > 0  # -0 canonicalised to +0, still > 0
    assert decode_key(pack_key(1.5, 12345)) == (12345, 1.5)


def _search_worker(rank, world, port, cfg, S, M, out):
    """bench.py --shard searches: rank r owns searches r, r + world, ... whole (no collective on
    the data path); the ranks' argmaxes only meet when gathered for the report."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ids = list(range(rank, S, world))
    w = gen.make(cfg, n=30, M=M, S=S, search_ids=ids)
    res = {}
    for s, srch, Xs in zip(ids, w.searches, w.Xstar):
        m = gp.fit(srch.X, srch.y, srch.lengthscale, srch.sf2, srch.sn2)
        ei = gp.expected_improvement(*gp.posterior(m, Xs), m.best).astype(np.float32)
        top = max(range(len(ei)), key=lambda i: (ei[i], -i))
        res[s] = (top, float(ei[top]))
    got = [None] * world
    dist.all_gather_object(got, res)
    out[rank] = {k: v for r in got for k, v in r.items()}
    dist.destroy_process_group()


def test_two_rank_search_shard_matches_unsharded():
    world, cfg, S, M = 2, 3, 5, 700
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_search_worker, args=(world, _free_port(), cfg, S, M, out), nprocs=world, join=True)
    assert out[0] == out[1] and sorted(out[0]) == list(range(S))
    full = gen.make(cfg, n=30, M=M, S=S)
    for s, (srch, Xs) in enumerate(zip(full.searches, full.Xstar)):
        m = gp.fit(srch.X, srch.y, srch.lengthscale, srch.sf2, srch.sn2)
        ei = gp.expected_improvement(*gp.posterior(m, Xs), m.best).astype(np.float32)
        top = max(range(len(ei)), key=lambda i: (ei[i], -i))
        assert out[0][s] == (top, float(ei[top]))
