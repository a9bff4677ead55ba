"""Summarise an ncu report: speed-of-light / occupancy / stalls + per-source-line
instruction and stall shares.   python tools/ncu_lines.py report.ncu-rep [topN]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


rows = list(csv.reader(io.StringIO(ncu("--page", "details", "--csv"))))
h = rows[0]
si, mi, vi, ui = (h.index(x) for x in ("Section Name", "Metric Name", "Metric Value", "Metric Unit"))
keep = {"Duration", "Compute (SM) Throughput", "Memory Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "DRAM Throughput", "Issue Slots Busy", "Executed Ipc Active",
        "Achieved Active Warps Per SM", "Theoretical Active Warps per SM", "Registers Per Thread",
        "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp", "Eligible Warps Per Scheduler",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Grid Size"}
for r in rows[1:]:
    if r[mi] in keep:
        print(f"{r[mi]:40s} {r[vi]} {r[ui]}")
rows = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source=cuda,sass"))))
for hi, r in enumerate(rows):
    if "Instructions Executed" in r:
        break
h = rows[hi]
ie = h.index("Instructions Executed")
ws = h.index("Warp Stall Sampling (All Samples)")
agg = {}
for r in rows[hi + 1:]:
    # source-line rows carry the line's aggregated metrics (SASS rows have an
    # empty first column)
    if not r or not r[0] or r[0].startswith("0x") or len(r) <= ie:
        continue
    try:
        agg[(r[0], r[1].strip())] = [float(r[ie] or 0), float(r[ws] or 0)]
    except ValueError:
        pass
tot = sum(v[0] for v in agg.values()) or 1
tots = sum(v[1] for v in agg.values()) or 1
print(f"total warp instructions: {tot:.3e}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0]/tot*100:5.1f}% inst {v[1]/tots*100:5.1f}% stall  L{k[0]}: {k[1][:95]}")
