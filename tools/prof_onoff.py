import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2403_08131_b200 import gpbo
from workloads import gen
dev = torch.device("cuda", 0); stream = torch.cuda.current_stream()
w = gen.make(2, M=1 << 20)
ctx = gpbo.Context(device=0, stream=stream)
n = [s.X.shape[0] for s in w.searches]; d = [s.X.shape[1] for s in w.searches]
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
X = t(np.concatenate([s.X.ravel() for s in w.searches]).astype(np.float32)); y = t(np.concatenate([s.y for s in w.searches]))
ls = t(np.concatenate([s.lengthscale for s in w.searches]).astype(np.float32))
sf2 = t(np.array([s.sf2 for s in w.searches], np.float32)); sn2 = t(np.array([s.sn2 for s in w.searches], np.float32))
Xs = t(np.concatenate([x.ravel() for x in w.Xstar]).astype(np.float32))
off = np.array([0, Xs.numel() // 20], np.int64)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
def run(prof, K=40):
    ctx.set_profiling(prof)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tot = 0
    for i in range(K + 5):
        flush.zero_()
        e0.record(stream)
        m = ctx.fit(n, d, X, y, ls, sf2, sn2, wait=False)
        ctx.score_argmax(m, Xs, off)
        m.free()
        e1.record(stream); e1.synchronize()
        if i >= 5: tot += e0.elapsed_time(e1)
    ctx.set_profiling(False)
    return tot / K
for _ in range(2):
    print("profiling off %.4f  on %.4f ms" % (run(False), run(True)))
