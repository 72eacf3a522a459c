"""gp_posterior throughput (raw mu / var / EI of every candidate, device-resident) at a config's
shape, next to the argmax path on the same model and candidates.
    python tools/posterior_bench.py [cfg] [M]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_08131_b200 import gpbo  # noqa: E402
from workloads import gen  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
M = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 18
w = gen.make(cfg, M=M, S=1 if cfg == 3 else None)
s = w.searches[0]
stream = torch.cuda.current_stream()
ctx = gpbo.Context(0, stream)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
m = ctx.fit([s.X.shape[0]], [s.X.shape[1]], t(s.X.ravel()), t(s.y), t(s.lengthscale),
            t(np.array([s.sf2], np.float32)), t(np.array([s.sn2], np.float32)), kernel=w.kernel)
Xs = t(w.Xstar[0])
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
out = {"cfg": cfg, "M": M, "n": int(s.X.shape[0]), "d": int(s.X.shape[1])}
for name, fn in (("posterior", lambda: ctx.posterior(m, 0, Xs)),
                 ("argmax", lambda: ctx.score_argmax(m, Xs, [0, M]))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(5):
        fn()
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 5
    out[name] = {"ms": ms, "candidates_per_s": M / (ms / 1e3), "impl": ctx.last_impl}
out["posterior_over_argmax"] = out["posterior"]["ms"] / out["argmax"]["ms"]
print(json.dumps(out))
