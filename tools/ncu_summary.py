"""One-launch ncu --set full report -> the JSON summary kept under profiles/.

    python tools/ncu_summary.py rep.ncu-rep "<command>" "<workload>" > summary.json
"""
import csv
import io
import json
import subprocess
import sys

rep, command, workload = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, vals = rows[0], rows[1], rows[2]


def get(name, scale=1.0):
    idx = [i for i, x in enumerate(h) if x == name] + \
          [i for i, x in enumerate(h) if x.endswith("." + name)]
    for i in idx:
        if not vals[i].strip():
            continue
        if True:
            v = float(vals[i].replace(",", ""))
            u = units[i]
            if u == "Mbyte":
                v *= 1e6
            elif u == "Gbyte":
                v *= 1e9
            elif u == "Kbyte":
                v *= 1e3
            elif u == "us":
                v /= 1e3
            elif u == "ns":
                v /= 1e6
            return round(v * scale, 4)
    return None


rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
out = {
    "kernel": h and vals[h.index("Kernel Name")] if "Kernel Name" in h else None,
    "command": command,
    "workload": workload,
    "duration_ms": get("gpu__time_duration.sum"),
    "grid_size": get("launch__grid_size"),
    "dram_bytes_per_launch": int(rd + wr) if rd is not None and wr is not None else None,
    "dram_read_bytes": rd,
    "dram_write_bytes": wr,
    "issue_slots_busy_pct": get("sm__inst_issued.avg.pct_of_peak_sustained_active"),
    "executed_ipc_active": get("sm__inst_executed.avg.per_cycle_active"),
    "warp_instructions": get("smsp__inst_executed.sum"),
    "fp64_pipe_active_pct": get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    "achieved_warps_per_sm": get("sm__warps_active.avg.per_cycle_active"),
    "registers_per_thread": get("launch__registers_per_thread"),
    "avg_active_threads_per_warp": get("smsp__thread_inst_executed_per_inst_executed.ratio"),
    "l1_hit_rate_pct": get("l1tex__t_sector_hit_rate.pct"),
    "l2_hit_rate_pct": get("lts__t_sector_hit_rate.pct"),
    "dram_throughput_pct": get("dram__throughput.avg.pct_of_peak_sustained_elapsed"),
}
json.dump(out, sys.stdout, indent=1)
print()
