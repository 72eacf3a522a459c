"""Summarise an ncu report: key throughput metrics and the top stall sites (SASS)."""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
        "Registers Per Thread", "Achieved Occupancy", "Issue Slots Busy", "L2 Cache Throughput"]
RAW = ["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"]


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main(rep, top=25, ctx=0):
    out = []
    for row in csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))):
        if len(row) > 14 and row[-4] in KEYS:
            out.append(f"{row[-4]}: {row[-2]} {row[-3]}")
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    if len(rows) >= 3:
        h, v = rows[0], rows[2]
        for k in RAW:
            if k in h:
                out.append(f"{k}: {v[h.index(k)]}")
    print("\n".join(out))
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv",
                                           "--print-source=sass"]))))
    if len(rows) < 3:
        return
    h = rows[1]
    ia, isrc = h.index("Address"), h.index("Source")
    iall = h.index("Warp Stall Sampling (All Samples)")
    data = []
    for i, r in enumerate(rows[2:]):
        try:
            data.append((int(r[iall]), i, r[ia][-5:], r[isrc]))
        except (ValueError, IndexError):
            pass
    tot = sum(d[0] for d in data)
    print(f"stall samples: {tot}")
    for smp, i, a, src in sorted(data, reverse=True)[:top]:
        print(f"{smp:7d} {100.0 * smp / tot:5.1f}% {a} {src[:100]}")
        for j in range(max(0, i - ctx), i):
            print(f"{'':21s}{data[j][2]} {data[j][3][:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25,
         int(sys.argv[3]) if len(sys.argv) > 3 else 0)
