import time, sys, os
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2403_08131_b200 import gpbo
from workloads import gen
w = gen.make(1)
s = w.searches[0]
ctx = gpbo.Context(0, torch.cuda.current_stream())
dev = torch.device("cuda", 0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
Xd, yd, lsd = t(s.X.ravel()), t(s.y), t(s.lengthscale)
sf2d, sn2d = t(np.array([s.sf2], np.float32)), t(np.array([s.sn2], np.float32))
Xsd = t(w.Xstar[0].ravel())
moff = np.array([0, 4096], np.int64); base = np.zeros(1, np.int64)
for _ in range(20):
    m = ctx.fit([20], [2], Xd, yd, lsd, sf2d, sn2d, kernel=w.kernel, wait=False)
    ctx.score_argmax(m, Xsd, moff, base); m.free()
torch.cuda.synchronize()
N = 200
tf = ts = tfree = 0.0
t0 = time.perf_counter()
for _ in range(N):
    a = time.perf_counter()
    m = ctx.fit([20], [2], Xd, yd, lsd, sf2d, sn2d, kernel=w.kernel, wait=False)
    b = time.perf_counter()
    ctx.score_argmax(m, Xsd, moff, base)
    c = time.perf_counter()
    m.free()
    d = time.perf_counter()
    tf += b - a; ts += c - b; tfree += d - c
tt = time.perf_counter() - t0
print(f"per step: total {tt/N*1e6:.1f} us, fit call {tf/N*1e6:.1f}, score call {ts/N*1e6:.1f}, free {tfree/N*1e6:.1f}")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(100):
    m = ctx.fit([20], [2], Xd, yd, lsd, sf2d, sn2d, kernel=w.kernel, wait=False)
    ctx.score_argmax(m, Xsd, moff, base); m.free()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(8)
