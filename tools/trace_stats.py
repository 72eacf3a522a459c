"""Per-panel / per-tile statistics of a tools/trace_tc.py dump (gpurun_out/trace.txt)."""
import collections
import statistics
import sys

f = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/trace.txt"
npan = int(sys.argv[2]) if len(sys.argv) > 2 else 7
ev = []
for line in open(f):
    p = line.split()
    if len(p) >= 4 and p[0].isdigit():
        ev.append((int(p[0]), p[1], p[2], int(p[3][1:])))
V = [(c, i) for c, n, r, i in ev if n == "mma:V_issued"]
tiles = [V[i][0] for i in range(0, len(V), npan)]
td = [tiles[i + 1] - tiles[i] for i in range(len(tiles) - 1)]
print("tile cycles median", statistics.median(td), "tiles", len(tiles))
bypd = collections.defaultdict(list)
for i in range(len(V) - 1):
    bypd[V[i][1] % npan].append(V[i + 1][0] - V[i][0])
print("V issue interval by panel", {k: int(statistics.mean(v)) for k, v in sorted(bypd.items())})
for role in sorted({x[2] for x in ev if x[1] == "epi:kf_arrive"}):
    e = [x for x in ev if x[2] == role]
    by = collections.defaultdict(dict)
    for c, n, r, i in e:
        by[i][n] = c
    keys = sorted(by)
    comp = [by[i]["epi:kf_arrive"] - by[i]["epi:ke_ok"] for i in keys
            if "epi:kf_arrive" in by[i] and "epi:ke_ok" in by[i]]
    wke = [by[i]["epi:ke_ok"] - by[i]["epi:df_ok"] for i in keys
           if "epi:ke_ok" in by[i] and "epi:df_ok" in by[i]]
    bp = collections.defaultdict(list)
    for j in range(len(keys) - 1):
        if "epi:df_ok" in by[keys[j + 1]] and "epi:kf_arrive" in by[keys[j]]:
            bp[keys[j] % npan].append(by[keys[j + 1]]["epi:df_ok"] - by[keys[j]]["epi:kf_arrive"])
    if comp:
        print(role, "K* compute", statistics.median(comp), "wait KE", statistics.median(wke),
              "arrive->next df_ok by panel", {k: int(statistics.mean(v)) for k, v in sorted(bp.items())})
wk = {i: c for c, n, r, i in ev if n == "mma:wait_kf"}
ko = {i: c for c, n, r, i in ev if n == "mma:kf_ok"}
byp = collections.defaultdict(list)
for i in ko:
    if i in wk:
        byp[i % npan].append(ko[i] - wk[i])
print("MMA wait for K* by panel", {k: int(statistics.mean(v)) for k, v in sorted(byp.items())})
