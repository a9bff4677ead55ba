"""form_stage batching modes (pc_form_stage: 0 one batch per widening level,
1 all levels, 2 first level then the rest): warm median wall times on C1-C4
and C5 chains -- which one the default should be.

    python tools/form_stage_modes.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2103_16063_b200 import form_stage, partition_blocks  # noqa: E402
from paper_2103_16063_b200.workloads import c5_blockset, config_partition  # noqa: E402


def timeit(fn, reps=5):
    ts = []
    for _ in range(reps + 1):
        t0 = time.perf_counter()
        r = fn()
        ts.append((time.perf_counter() - t0) * 1e3)
    return sorted(ts[1:])[len(ts[1:]) // 2], r


cases = []
for c in ("C1", "C2", "C3", "C4"):
    part, model, k, batch, cl = config_partition(c)
    cases.append((c, partition_blocks(part, model, k), cl.num_nodes, cl.devices_per_node, batch))
for nb, D in ((1024, 256), (4096, 256), (4096, 1024)):
    cases.append((f"C5 {nb}x{D}", c5_blockset(nb, D, jitter_seed=0), max(1, D // 8), min(8, D), 8 * D))
for name, bs, N, dpn, BS in cases:
    row = [name]
    ref = None
    for label, spec in (("hybrid", None), ("per-level", False), ("all", True)):
        ms, r = timeit(lambda: form_stage(N, dpn, BS, bs, speculative=spec), reps=3 if "4096" in name else 5)
        assert ref is None or (r.plan == ref.plan and r.stats == ref.stats)
        ref = r
        row.append(f"{label} {ms:.1f} ms")
    print(" | ".join(row), flush=True)
