"""Stall-reason totals and the top SASS instructions by stall samples from an ncu source page
(--page source --csv --print-source=cuda,sass).  usage: ... | python tools/ncu_stalls.py [top]"""
import csv
import sys

top = int(sys.argv[1]) if len(sys.argv) > 1 else 25
rows = list(csv.reader(sys.stdin))
hdr = next(r for r in rows if r and r[0] == "Line No")
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {h: 0.0 for h in reasons}
sass = []
line = None
for r in rows:
    if not r or len(r) < len(hdr):
        continue
    if r[0].isdigit():
        line = int(r[0])
        continue
    if r[0] == "" and r[2].startswith("0x"):
        st = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        for h in reasons:
            tot[h] += float(r[ix[h]] or 0)
        det = sorted(((float(r[ix[h]] or 0), h[6:]) for h in reasons), reverse=True)[:3]
        sass.append((st, line, r[3][:60], det))
T = sum(tot.values()) or 1
print("stall reasons:", ", ".join(f"{h[6:]} {100*v/T:.1f}%" for h, v in sorted(tot.items(), key=lambda a: -a[1]) if v))
for st, ln, ins, det in sorted(sass, key=lambda a: -a[0])[:top]:
    print(f"{100*st/T:5.1f}% line {ln}: {ins:60s} " + " ".join(f"{n}:{v:.0f}" for v, n in det if v))
