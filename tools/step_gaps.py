"""Where the time of one bench step (config 2) goes: CUDA-event spans around each API call and
the host time of each call.  python tools/step_gaps.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_08131_b200 import gpbo  # noqa: E402
from workloads import gen  # noqa: E402

dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
CFG = int(next((a for a in sys.argv[1:] if a.isdigit()), "2"))
w = gen.make(CFG, M=1 << 20 if CFG == 2 else None)
ctx = gpbo.Context(device=0, stream=stream)
n = [s.X.shape[0] for s in w.searches]
d = [s.X.shape[1] for s in w.searches]
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
Xd = t(np.concatenate([s.X.ravel() for s in w.searches]).astype(np.float32))
yd = t(np.concatenate([s.y for s in w.searches]))
lsd = t(np.concatenate([s.lengthscale for s in w.searches]).astype(np.float32))
sf2d = t(np.array([s.sf2 for s in w.searches], np.float32))
sn2d = t(np.array([s.sn2 for s in w.searches], np.float32))
Xsd = t(np.concatenate([x.ravel() for x in w.Xstar]).astype(np.float32))
m_off = np.zeros(w.S + 1, np.int64)
m_off[1:] = np.cumsum([x.shape[0] for x in w.Xstar])
base = np.array(w.m_global_base, np.int64)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
acc = np.zeros(6)
K = 30
WAIT = "--sync" in sys.argv  # default: the bench's asynchronous fit
for it in range(K + 5):
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    ev[0].record(stream)
    m = ctx.fit(n, d, Xd, yd, lsd, sf2d, sn2d, kernel=w.kernel, wait=WAIT)
    h1 = time.perf_counter()
    ev[1].record(stream)
    idx, ei = ctx.score_argmax(m, Xsd, m_off, base)
    h2 = time.perf_counter()
    ev[2].record(stream)
    m.free()
    ev[3].record(stream)
    h3 = time.perf_counter()
    ev[3].synchronize()
    if it >= 5:
        acc += [ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3]),
                (h1 - h0) * 1e3, (h2 - h1) * 1e3, (h3 - h2) * 1e3]
acc /= K
print("device spans ms: fit %.4f  score %.4f  free %.4f | host ms: fit %.4f  score %.4f  free %.4f"
      % tuple(acc))
ctx.set_profiling(True)
for _ in range(10):
    m = ctx.fit(n, d, Xd, yd, lsd, sf2d, sn2d, kernel=w.kernel)
    ctx.score_argmax(m, Xsd, m_off, base)
    m.free()
torch.cuda.synchronize()
print("kernel ms:", {k: ctx.kernel_time(k) for k in ctx.KERNELS})
