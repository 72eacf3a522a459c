"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.
usage: python tools/launch_summary.py launches.csv "<command line>" > profiles/rNN_launches_summary.txt"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ix = {h: j for j, h in enumerate(hdr)}
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.OrderedDict()
lst = []
for r in rows[start + 1:]:
    if len(r) < len(hdr):
        continue
    t = float(r[ix["Metric Value"]].replace(",", "")) * scale.get(r[ix["Metric Unit"]], 1.0)
    name = r[ix["Kernel Name"]]
    short = name.split("(")[0].split("::")[-1]
    if "at::native" in name or "vectorized_elementwise" in name or short.startswith("array<"):
        short = "[torch] L2 flush (zero_ of 256 MiB, outside the timed step)"
    lst.append((r[ix["ID"]], short, t))
    a = agg.setdefault(short, [0, 0.0])
    a[0] += 1
    a[1] += t
ours = {k: v for k, v in agg.items() if not k.startswith("[torch]")}
tot = sum(v[1] for v in ours.values())
print(f"# ncu --metrics gpu__time_duration.sum --clock-control none: {sys.argv[2] if len(sys.argv) > 2 else ''}")
print("# cold-cache, serialised launches: compare SHARES of the step, not absolute times")
print(f"{'kernel':44s} {'launches':>8s} {'total_us':>10s} {'mean_us':>9s} {'share':>7s}")
for k, (c, t) in sorted(agg.items(), key=lambda a: -a[1][1]):
    sh = f"{100 * t / tot:6.1f}%" if k in ours else "     -"
    print(f"{k:44s} {c:8d} {t:10.1f} {t / c:9.1f} {sh}")
print("\n# per launch (us)")
for i, k, t in lst:
    print(f"{i:>4s} {k:44s} {t:9.1f}")

# one timed step of bench.py (the launches between the first two L2 flushes: the value's pass --
# gp_fit + ei_score_argmax; the later passes of the same run time e2e, e2e_suggest, score-only and
# gp_posterior, whose kernels appear in the totals above)
groups, cur, seen = [], [], False
for i, k, t in lst:
    if k.startswith("[torch]"):
        if seen:
            groups.append(cur)
        cur, seen = [], True
    elif seen:
        cur.append((k, t))
if groups:
    g = groups[0]
    st = sum(t for _, t in g)
    print("\n# one timed step (first flush-delimited group): kernel, us, share of the step")
    for k, t in g:
        print(f"  {k:44s} {t:9.1f} {100 * t / st:6.1f}%")
    print(f"  {'total':44s} {st:9.1f}")
