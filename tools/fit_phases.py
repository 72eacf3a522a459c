"""Print the fit kernel's phase clocks (CTA 0) for a config's fit; needs a GPBO_FIT_TIMING build:
    GPBO_FIT_TIMING=1 python paper_2403_08131_b200/build.py && python tools/fit_phases.py 2"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_08131_b200 import gpbo  # noqa: E402
from workloads import gen  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = gen.make(cfg, M=1024)
ctx = gpbo.Context(device=0)
n = [s.X.shape[0] for s in w.searches]
d = [s.X.shape[1] for s in w.searches]
X = np.ascontiguousarray(np.concatenate([s.X.ravel() for s in w.searches]), np.float32)
y = np.concatenate([s.y for s in w.searches])
ls = np.ascontiguousarray(np.concatenate([s.lengthscale for s in w.searches]), np.float32)
sf2 = np.array([s.sf2 for s in w.searches], np.float32)
sn2 = np.array([s.sn2 for s in w.searches], np.float32)
for _ in range(3):
    m = ctx.fit(n, d, X, y, ls, sf2, sn2, kernel=w.kernel)
    m.free()
ctx.close()
