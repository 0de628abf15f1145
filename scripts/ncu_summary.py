"""Summarise an ncu --set full report: key throughputs, pipes, stalls, top SASS lines."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25


def page(p, *extra):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True,
                         text=True).stdout
    return list(csv.reader(io.StringIO(out)))


rows = page("raw")
hdr, r = rows[0], rows[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
print(r[hdr.index("Kernel Name")][:100])
for k in keys:
    if k in hdr:
        print(f"  {k:60s} {r[hdr.index(k)]} {rows[1][hdr.index(k)]}")
pipes = []
for i, h in enumerate(hdr):
    if h.startswith("sm__inst_executed_pipe_") and h.endswith(".avg.pct_of_peak_sustained_active"):
        try:
            pipes.append((float(r[i]), h))
        except ValueError:
            pass
print("  pipes:", ", ".join(f"{h.split('pipe_')[1].split('.')[0]} {v:.1f}" for v, h in sorted(pipes, reverse=True)[:6]))
s = page("source", "--print-source", "sass")
shdr, data = s[1], s[2:]
cols = [h for h in shdr if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
for d in data:
    for c in cols:
        tot[c] += int(d[shdr.index(c)] or 0)
T = sum(tot.values()) or 1
print("  stalls:", {k[6:]: round(v / T * 100, 1) for k, v in tot.most_common(8)})
si = shdr.index("Warp Stall Sampling (All Samples)")
ie = shdr.index("Instructions Executed")
op = collections.Counter()
for d in data:
    o = d[1].strip().split()
    if o:
        m = o[1] if o[0].startswith("@") else o[0]
        op[m.split(".")[0]] += int(d[ie] or 0)
print("  inst mix:", op.most_common(14))
S = sum(int(d[si]) for d in data) or 1
for d in sorted(data, key=lambda d: -int(d[si]))[:top]:
    print(f"   {int(d[si]) / S * 100:5.2f}% {d[0][-5:]} {d[1].strip()[:90]}")
