"""Per-run phase times of partition_blocks + form_stage on C1-C4 (bench.py's
latency loop, every run printed): finds sporadic host stalls."""
import gc
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2103_16063_b200 import _lib, form_stage, partition_blocks  # noqa: E402
from paper_2103_16063_b200 import flatten as _flat  # noqa: E402
from paper_2103_16063_b200.workloads import config_partition  # noqa: E402

ctx = _lib.context(0)
for name in sys.argv[1:] or ["C1", "C2", "C3", "C4"]:
    part, model, k, batch, cl = config_partition(name)
    rows = []
    for i in range(11):
        _flat._ATOM_CACHE.clear()
        ctx.problem_owner = None
        ctx.lib.pc_reset_cache(ctx.h)
        gc.collect()
        t_pb, t_fs = {}, {}
        t0 = time.perf_counter()
        bs = partition_blocks(part, model, k, timings=t_pb)
        t1 = time.perf_counter()
        form_stage(cl.num_nodes, cl.devices_per_node, batch, bs, last_stats=t_fs)
        t2 = time.perf_counter()
        rows.append(((t1 - t0) * 1e3, (t2 - t1) * 1e3, t_pb["library_ms"], t_fs["library_ms"],
                     t_fs.get("span_ms", 0), t_fs.get("device_ms", 0), t_fs.get("post_ms", 0)))
    for r in rows:
        print(name, " ".join("%7.2f" % x for x in r), flush=True)
