"""Summarise an ncu --set full report: headline metrics per kernel and the
hottest SASS opcodes / instruction windows by stall samples.
usage: python scripts/ncu_hot.py REPORT.ncu-rep KERNEL_REGEX"""
import collections
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv", "-k", f"regex:{kre}"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(io.StringIO(det)))
h = r[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
want = ["Duration", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Theoretical Occupancy", "Achieved Occupancy", "Warp Cycles Per Issued Instruction",
        "Avg. Active Threads Per Warp", "L1/TEX Hit Rate", "L2 Hit Rate", "DRAM Throughput"]
for x in r[1:]:
    if x[mi] in want:
        print(f"{x[ki][:28]:28s} {x[mi]:38s} {x[vi]} {x[ui]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kre}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
si, wi, ie = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
cnt, smp = collections.Counter(), collections.Counter()
data = []
for idx, x in enumerate(rows[2:]):
    if len(x) < len(h):
        continue
    try:
        w, n = int(x[wi]), int(x[ie] or 0)
    except ValueError:
        continue
    op = [o for o in x[si].split() if not o.startswith("@")]
    m = op[0].split(".")[0] if op else "?"
    cnt[m] += n
    smp[m] += w
    data.append((idx, w, n, x[si][:90]))
tot, ti = sum(smp.values()) or 1, sum(cnt.values()) or 1
print("samples", tot, "instructions", ti)
for m, v in sorted(smp.items(), key=lambda t: -t[1])[:16]:
    print(f"  {m:8s} {100 * v / tot:5.1f}% samples {100 * cnt[m] / ti:5.1f}% instr")
win = collections.Counter()
for d in data:
    win[d[0] // 24] += d[1]
for k, v in sorted(win.items(), key=lambda t: -t[1])[:8]:
    print(f"window {k * 24}-{k * 24 + 23}: {100 * v / tot:5.1f}% samples")
    for d in data[k * 24:k * 24 + 24]:
        if d[1] > 0.004 * tot:
            print("     ", d[0], d[1], d[2], d[3])
