"""Summarise an ncu launch list of k_dp_level (one bench step) into
profiles/dp_level_profile.json, read by bench.py for the issue-rate roofline.

    ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,
        sm__inst_executed_pipe_fp64.sum,smsp__thread_inst_executed.sum,
        dram__bytes_read.sum,dram__bytes_write.sum --kernel-name regex:k_dp_level
        --clock-control none --csv --log-file launches.csv
        python bench.py --steps 1 --warmup 0 --no-sweep --no-latency --no-cpu-baseline
    python tools/ncu_inst_summary.py launches.csv NB D K > profiles/dp_level_profile.json

K = k_dp_level launches of one step (the bench line's roofline.launches_per_step):
the first K launches are that step's (the bench's later schedule-(i) runs follow).

The instruction counts are per step of that workload (deterministic up to
atomic ordering); bench.py divides them by the live k_dp_level time and checks
`dp_cu_sha` against the kernel source it runs.
"""
import csv
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path, nb, D, K = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
rows = [r for r in csv.reader(open(path)) if r]
hdr_i = next(i for i, r in enumerate(rows) if "Metric Name" in r)
h = rows[hdr_i]
ci = {k: h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
per = {}
for r in rows[hdr_i + 1:]:
    if len(r) < len(h) or "k_dp_level" not in r[ci["Kernel Name"]]:
        continue
    v = float(r[ci["Metric Value"]].replace(",", ""))
    u = r[ci["Metric Unit"]]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9,
             "usecond": 1e-6, "us": 1e-6, "ms": 1e-3,
             "msecond": 1e-3, "second": 1.0}.get(u, 1.0)
    per.setdefault(r[ci["ID"]], {})[r[ci["Metric Name"]]] = v * scale
launches = [per[k] for k in sorted(per, key=int)][:K]
assert len(launches) == K, (len(launches), K)
tot = {k: sum(l.get(k, 0.0) for l in launches) for k in launches[0]}
inst = tot["smsp__inst_executed.sum"]
sha = hashlib.sha256(open(os.path.join(ROOT, "paper_2103_16063_b200", "csrc", "dp.cu"), "rb").read())
out = {
    "workload": {"nb": nb, "D": D, "n_gpus": 1},
    "dp_cu_sha": sha.hexdigest()[:16],
    "launches": len(launches),
    "warp_inst_per_step": inst,
    "fp64_pipe_inst_per_step": tot.get("sm__inst_executed_pipe_fp64.sum"),
    "active_threads_per_warp": tot.get("smsp__thread_inst_executed.sum", 0.0) / inst if inst else None,
    "ncu_seconds_per_step": tot.get("gpu__time_duration.sum"),
    "dram_bytes_per_step": tot.get("dram__bytes_read.sum", 0.0) + tot.get("dram__bytes_write.sum", 0.0),
    "dram_bytes_per_launch": (tot.get("dram__bytes_read.sum", 0.0) +
                              tot.get("dram__bytes_write.sum", 0.0)) / len(launches),
    "source": os.path.basename(path),
    "note": "ncu --clock-control none, serialised launches (cold caches): counts are exact, "
            "times are not the bench's",
}
print(json.dumps(out, indent=1))
