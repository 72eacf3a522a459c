"""bo_suggest_batch at a config's shape (d REAL parameters in [0, 1], M on-device candidates per
search): time per call next to ei_score_argmax on the same model.  python tools/suggest_bench.py [cfg]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_08131_b200 import gpbo  # noqa: E402
from workloads import gen  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = gen.make(cfg)
ctx = gpbo.Context(0, torch.cuda.current_stream())
n = [s.X.shape[0] for s in w.searches]
d = [s.X.shape[1] for s in w.searches]
X = np.ascontiguousarray(np.concatenate([s.X.ravel() for s in w.searches]), np.float32)
y = np.concatenate([s.y for s in w.searches])
ls = np.ascontiguousarray(np.concatenate([s.lengthscale for s in w.searches]), np.float32)
sf2 = np.array([s.sf2 for s in w.searches], np.float32)
sn2 = np.array([s.sn2 for s in w.searches], np.float32)
m = ctx.fit(n, d, X, y, ls, sf2, sn2, kernel=w.kernel)
spaces = [gpbo.Space(ctx, [{"kind": 0, "lo": 0.0, "hi": 1.0}] * dd) for dd in d]
M = np.array([x.shape[0] for x in w.Xstar], np.int64)
out = {"cfg": cfg, "M": int(M.sum())}
for dedup in (True, False):
    for it in range(3):
        gpbo.suggest(ctx, m, spaces, M, 7, it, dedup=dedup)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for it in range(10):
        gpbo.suggest(ctx, m, spaces, M, 7, 100 + it, dedup=dedup)
    out["suggest_ms_dedup" if dedup else "suggest_ms"] = (time.perf_counter() - t0) / 10 * 1e3
print(json.dumps(out))
