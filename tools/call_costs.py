"""Per-call device work (feasible pairs, DP ms) vs the closed-form visit
weight, for sharding weights.   python tools/call_costs.py --nb 1024 --D 256"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2103_16063_b200 import _lib  # noqa: E402
from paper_2103_16063_b200.search import call_weight, enumerate_calls, run_calls  # noqa: E402
from paper_2103_16063_b200.stages import bind_problem  # noqa: E402
from paper_2103_16063_b200.workloads import c5_blockset  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nb", type=int, default=1024)
ap.add_argument("--D", type=int, default=256)
a = ap.parse_args()
ctx = _lib.context(0)
bs = c5_blockset(a.nb, a.D, jitter_seed=0)
bind_problem(ctx, bs)
calls, levels = enumerate_calls(max(1, a.D // 8), min(8, a.D), 8 * a.D, a.nb)
out = []
for c in calls:
    b = run_calls(ctx, [c], 8 * a.D, False, False)
    out.append({"call": c, "weight": call_weight(a.nb, c), "pairs": int(b.stats.pairs),
                "dp_ms": float(b.stats.device_ms)})
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", f"call_costs_{a.nb}_{a.D}.json"), "w"))
tot = sum(o["dp_ms"] for o in out)
print(f"{len(out)} calls, sum of single-call DP ms {tot:.0f}")
