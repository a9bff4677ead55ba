"""Host-side breakdown of one bench step (N=1): run_calls / pack / decide."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2103_16063_b200 import _lib
from paper_2103_16063_b200.search import enumerate_calls, run_calls, _pack, exchange, decide, lpt_shard
from paper_2103_16063_b200.stages import bind_problem
from paper_2103_16063_b200.workloads import c5_blockset

nb, D = int(sys.argv[1]), int(sys.argv[2])
ctx = _lib.context(0)
bs = c5_blockset(nb, D, jitter_seed=0)
bind_problem(ctx, bs)
calls, levels = enumerate_calls(max(1, D // 8), min(8, D), 8 * D, nb)
owner = lpt_shard(nb, calls, 1)
idx = list(range(len(calls)))
for rep in range(3):
    ctx.lib.pc_reset_cache(ctx.h)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    b = run_calls(ctx, calls, 8 * D, False, True)
    t1 = time.perf_counter()
    rec, plan_w = _pack(nb, calls, levels, owner, 0, b, idx, max(levels) + 1, max(c[0] for c in calls))
    t2 = time.perf_counter()
    allrec = exchange(rec, None, torch.device("cuda", 0))
    t3 = time.perf_counter()
    out = decide(allrec, calls, levels, owner, plan_w, None, 8 * D)
    t4 = time.perf_counter()
    st = b.stats
    print(f"run_calls {1e3*(t1-t0):.1f} ms (dp {st.device_ms:.1f}, span {st.span_ms:.1f}), pack {1e3*(t2-t1):.1f}, "
          f"exchange {1e3*(t3-t2):.1f}, decide {1e3*(t4-t3):.1f}", flush=True)
