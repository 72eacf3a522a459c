"""Aggregate an ncu source page (--page source --csv --print-source=cuda,sass) by CUDA line:
instructions executed and warp-stall samples.  usage: ncu -i rep --page source --csv
--print-source=cuda,sass | python tools/ncu_lines.py [top]"""
import csv
import sys

top = int(sys.argv[1]) if len(sys.argv) > 1 else 30
rows = list(csv.reader(sys.stdin))
hdr = next(r for r in rows if r and r[0] == "Line No")
ix = {h: i for i, h in enumerate(hdr)}
i_inst = ix["Instructions Executed"]
i_st = ix["Warp Stall Sampling (All Samples)"]
agg = []
for r in rows:
    if r and r[0].isdigit() and len(r) > i_inst:
        try:
            inst = float(r[i_inst] or 0)
            st = float(r[i_st] or 0)
        except ValueError:
            continue
        if inst or st:
            agg.append((inst, st, int(r[0]), r[1][:90]))
tot_i = sum(a[0] for a in agg) or 1
tot_s = sum(a[1] for a in agg) or 1
print(f"total warp instructions {tot_i:.0f}, stall samples {tot_s:.0f}")
for inst, st, ln, src in sorted(agg, key=lambda a: -a[1])[:top]:
    print(f"{ln:5d} inst {inst:9.0f} ({100*inst/tot_i:5.1f}%) stall {100*st/tot_s:5.1f}%  {src}")
