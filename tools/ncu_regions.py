"""Stall samples of an ncu SASS source page (--page source --csv --print-source=sass) grouped by
code region: usage python tools/ncu_regions.py src.csv [window]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
win = int(sys.argv[2]) if len(sys.argv) > 2 else 80
hdr = next(r for r in rows if r and r[0] == "Address")
ix = {h: i for i, h in enumerate(hdr)}
st_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ins = []
for r in rows:
    if len(r) == len(hdr) and r[0].startswith("0x"):
        ins.append(r)
tot = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in ins)
print("instructions", len(ins), "samples", tot)
for w0 in range(0, len(ins), win):
    chunk = ins[w0:w0 + win]
    smp = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in chunk)
    if smp < 0.01 * tot:
        continue
    ops = {}
    for r in chunk:
        op = r[1].split()[0] if r[1].split() else ""
        if op.startswith("@"):
            op = r[1].split()[1]
        op = op.split(".")[0]
        ops[op] = ops.get(op, 0) + 1
    key = [o for o in ("UTCHMMA", "MUFU", "LDTM", "STTM", "STS", "SYNCS", "ATOMG", "REDG", "BAR", "DFMA") if o in ops]
    st = {h[6:]: sum(float(r[ix[h]] or 0) for r in chunk) for h in st_cols}
    top = sorted(st.items(), key=lambda a: -a[1])[:4]
    print(f"{w0:5d}-{w0 + len(chunk):5d} {100 * smp / tot:5.1f}%  [{' '.join(key)}]  " +
          " ".join(f"{k}:{100 * v / tot:.1f}" for k, v in top if v))
