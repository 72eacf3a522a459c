"""Fit S copies of a config's first search in one batched gp_fit (profiling the fit kernels with
enough CTAs for ncu's stall sampling).  python tools/fit_many.py [cfg] [S]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_08131_b200 import gpbo  # noqa: E402
from workloads import gen  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
S = int(sys.argv[2]) if len(sys.argv) > 2 else 148
w = gen.make(cfg, M=1024)
s0 = w.searches[0]
ctx = gpbo.Context(device=0)
n = [s0.X.shape[0]] * S
d = [s0.X.shape[1]] * S
X = np.ascontiguousarray(np.tile(s0.X.ravel(), S), np.float32)
y = np.tile(s0.y, S)
ls = np.ascontiguousarray(np.tile(s0.lengthscale, S), np.float32)
sf2 = np.full(S, s0.sf2, np.float32)
sn2 = np.full(S, s0.sn2, np.float32)
for it in range(4):
    t0 = time.perf_counter()
    m = ctx.fit(n, d, X, y, ls, sf2, sn2, kernel=w.kernel)
    dt = time.perf_counter() - t0
    m.free()
print(f"cfg {cfg} S {S} n {n[0]} fit wall {dt * 1e3:.3f} ms")
ctx.close()
