"""Run one scoring call (config argv[2], default 2; config 3: its first search only) with the tcgen05 event trace on and print CTA 0's timeline."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2403_08131_b200 import gpbo
from workloads import gen

cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = gen.make(cfg, M=1 << 20 if cfg == 2 else None, S=1 if cfg == 3 else None)
s = w.searches[0]
ctx = gpbo.Context(0, torch.cuda.current_stream())
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
m = ctx.fit([s.X.shape[0]], [s.X.shape[1]], t(s.X.ravel()), t(s.y), t(s.lengthscale),
            t(np.array([s.sf2], np.float32)), t(np.array([s.sn2], np.float32)))
Xs = t(w.Xstar[0])
ctx.score_argmax(m, Xs, [0, Xs.shape[0]])
buf = torch.zeros(6 * 16384, dtype=torch.int64, device="cuda")
ctx.debug_trace(buf)
ctx.score_argmax(m, Xs, [0, Xs.shape[0]])
ctx.debug_trace(None)
b = buf.cpu().numpy().astype(np.uint64)
ev = []
for sl in range(5):
    for i in range(8191):
        key, clk = int(b[sl * 16384 + 2 * i]), int(b[sl * 16384 + 2 * i + 1])
        if key == 0 and clk == 0:
            break
        ev.append((clk, key >> 56, (key >> 48) & 0xFF, key & 0xFFFFFFFFFFFF))
n = len(ev)
ev.sort()
t0 = ev[0][0] if ev else 0
names = {1: "mma:wait_kf", 2: "mma:kf_ok", 3: "mma:V_issued", 4: "mma:dist_issued",
         5: "epi:df_arrived", 6: "epi:df_ok", 7: "epi:ke_ok", 8: "epi:kf_arrive",
         9: "ld:wait", 10: "ld:go", 11: "ld:A_full", 12: "mma:wait_de", 13: "mma:de_ok",
         14: "mma:V_mmas_done", 15: "mma:V_start",
         16: "drn:start", 17: "drn:v_done", 18: "drn:pf_ok", 19: "drn:finished",
         20: "mma:V_k0", 21: "mma:V_k1", 22: "mma:V_k2", 23: "mma:V_k3", 24: "mma:dist_start"}
lim = int(sys.argv[1]) if len(sys.argv) > 1 else 400
for clk, tag, role, idx in ev[:lim]:
    print(f"{clk - t0:9d} {names.get(tag, tag):16s} r{role:<3d} #{idx}")
print("events", n, "span cycles", ev[-1][0] - t0 if ev else 0)
cta = b[5 * 16384:5 * 16384 + 2 * 8192].reshape(-1, 2).astype(np.int64)
cta = cta[cta[:, 1] > 0]
if len(cta):
    g0 = cta[:, 0].min()
    st, en = (cta[:, 0] - g0) / 1e3, (cta[:, 1] - g0) / 1e3
    print(f"CTAs {len(cta)}: start us min/med/max {st.min():.1f}/{np.median(st):.1f}/{st.max():.1f}"
          f"  end us min/med/max {en.min():.1f}/{np.median(en):.1f}/{en.max():.1f}"
          f"  dur med {np.median(en - st):.1f}  slowest CTAs {np.argsort(-(en - st))[:6].tolist()}")
