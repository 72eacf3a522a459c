"""Config 5 of BASELINE.json: a full tuning-campaign replay on the Table IV space (RT-TDDFT-shaped
mixed integer / ordinal / categorical parameters with the paper's constraint blocks, R16-R18).

5 random initial configurations, then ITERS sequential BO iterations: gp_fit on the history
(n = 5 .. 5 + ITERS - 1, d = 35 encoded), bo_suggest_batch (on-device constrained candidate
generation, M candidates, dedup against the history, scoring, argmax), the suggestion decoded to
raw values and evaluated by the synthetic objective on the host (rttddft.objective), appended.
SURVEY.md §8(d) asks for iterations/s and candidates/s for this config.

    python tools/replay_bench.py [--iters 200] [--M 262144] [--seed 5]

Prints one JSON line: iterations/s (wall clock, everything included), the device time per
iteration (CUDA events around fit + suggest), candidates/s, the scoring kernel used as n grows,
and the best objective found.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_08131_b200 import gpbo  # noqa: E402
from workloads import rttddft  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--M", type=int, default=1 << 18)
    ap.add_argument("--seed", type=int, default=5)
    ap.add_argument("--update", default="append", choices=["append", "refit"],
                    help="append: O(n^2) gp_fit_append per iteration (§8(f)2); refit: gp_fit")
    args = ap.parse_args()
    params, blocks, _ = rttddft.table_iv()
    stream = torch.cuda.current_stream()
    ctx = gpbo.Context(device=0, stream=stream)
    sp = gpbo.Space(ctx, params, blocks)
    d = sp.dim
    vidx = rttddft.initial_design(params, blocks, 5, args.seed)
    y = rttddft.objective(vidx, params)
    # encoded history: the library's own encoder on the decoded raw values of the initial design
    X = np.concatenate([sp.encode(_raw(params, row)[None, :]) for row in vidx]).astype(np.float32)
    ls = np.full(d, 0.4 * np.sqrt(d), np.float32)
    sf2 = np.ones(1, np.float32)
    sn2 = np.full(1, 1e-4, np.float32)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # untimed warm-up (library load, first launches) on a throw-away copy of the history
    for _ in range(3):
        m = ctx.fit([len(y)], [d], np.ascontiguousarray(X.ravel()), y, ls, sf2, sn2)
        gpbo.suggest(ctx, m, [sp], [args.M], args.seed + 1, 0, dedup=True)
        m.free()
    torch.cuda.synchronize()
    dev_ms, impls, refits = [], {}, 0
    m = None
    t0 = time.perf_counter()
    for it in range(args.iters):
        e0.record(stream)
        if m is None or args.update == "refit":
            if m is not None:
                m.free()
            m = ctx.fit([len(y)], [d], np.ascontiguousarray(X.ravel()), y, ls, sf2, sn2)
        else:  # the surrogate update: one new observation, O(n^2) (gp_fit_append)
            m2 = ctx.fit_append(m, np.ascontiguousarray(X[-1]), y[-1:].copy())
            refits += ctx.last_append_refit
            m.free()
            m = m2
        idx, xr, ei = gpbo.suggest(ctx, m, [sp], [args.M], args.seed, it, dedup=True)
        e1.record(stream)
        e1.synchronize()
        dev_ms.append(e0.elapsed_time(e1))
        impls[ctx.last_impl] = impls.get(ctx.last_impl, 0) + 1
        raw = np.asarray(xr[0], np.float64)
        vnew = _vidx(params, raw)
        X = np.concatenate([X, sp.encode(raw[None, :]).astype(np.float32)])
        y = np.concatenate([y, rttddft.objective(vnew[None, :], params)])
    m.free()
    wall = time.perf_counter() - t0
    names = {1: "cuda-core", 2: "tcgen05", 3: "tcgen05-stream"}
    line = {"metric": "BO iterations/s (config 5 replay)", "value": args.iters / wall,
            "unit": "iterations/s", "iters": args.iters, "M_per_iter": args.M,
            "n_final": int(len(y)), "d_enc": d,
            "device_ms_per_iter": {"mean": float(np.mean(dev_ms)), "first": float(dev_ms[0]),
                                   "last": float(dev_ms[-1])},
            "candidates_per_s_device": args.M * args.iters / (np.sum(dev_ms) / 1e3),
            "scoring_kernels": {names.get(k, str(k)): v for k, v in impls.items()},
            "update": args.update, "append_refits": refits,
            "best_y": float(np.min(y)), "initial_best_y": float(np.min(y[:5]))}
    print(json.dumps(line), flush=True)
    ctx.close()


def _raw(params, row):
    """raw values of one configuration given per-parameter value indices"""
    out = []
    for v, p in zip(row, params):
        if p["kind"] == 2:
            out.append(float(p["values"][int(v)]))
        elif p["kind"] == 1:
            out.append(float(p["lo"] + int(v)))
        else:
            out.append(float(v))
    return np.array(out)


def _vidx(params, raw):
    """value indices of one configuration given its raw values (inverse of _raw)"""
    out = []
    for v, p in zip(raw, params):
        if p["kind"] == 2:
            out.append(int(np.argmin(np.abs(np.asarray(p["values"], float) - v))))
        elif p["kind"] == 1:
            out.append(int(round(v - p["lo"])))
        else:
            out.append(int(round(v)))
    return np.array(out, np.int64)


if __name__ == "__main__":
    main()
