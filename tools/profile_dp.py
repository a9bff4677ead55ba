"""Profiling driver: one (or more) full C5 searches on cuda:0, for ncu.

    python tools/profile_dp.py --nb 512 --D 128 [--reps 2]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2103_16063_b200 import _lib  # noqa: E402
from paper_2103_16063_b200.search import enumerate_calls, run_calls  # noqa: E402
from paper_2103_16063_b200.stages import bind_problem  # noqa: E402
from paper_2103_16063_b200.workloads import c5_blockset, unpruned_visits  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nb", type=int, default=512)
ap.add_argument("--D", type=int, default=128)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--levels", default="all", help="'all' or a widening level index")
ap.add_argument("--call", default=None, help="S,D,R,MB: run only this call")
a = ap.parse_args()
ctx = _lib.context(0)
bs = c5_blockset(a.nb, a.D, jitter_seed=0)
bind_problem(ctx, bs)
calls, levels = enumerate_calls(max(1, a.D // 8), min(8, a.D), 8 * a.D, a.nb)
if a.levels != "all":
    calls = [c for c, l in zip(calls, levels) if l == int(a.levels)]
if a.call:
    calls = [tuple(int(x) for x in a.call.split(","))]
for r in range(a.reps):
    ctx.lib.pc_reset_cache(ctx.h)
    t0 = time.perf_counter()
    b = run_calls(ctx, calls, 8 * a.D)
    dt = time.perf_counter() - t0
    st = b.stats
    print(f"rep {r}: {dt*1e3:.1f} ms, dp {st.device_ms:.1f} ms ({st.dp_launches} launches), "
          f"span {st.span_ms:.1f} ms, visits {unpruned_visits(a.nb, calls):.3e}, "
          f"pairs {st.pairs:.3e}, cands {st.candidates:.3e}, "
          f"rate {unpruned_visits(a.nb, calls)/(st.device_ms/1e3):.3e}/s", flush=True)
