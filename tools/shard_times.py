"""Time each rank's shard of the C5 enumeration as one batch on one GPU."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2103_16063_b200 import _lib  # noqa: E402
from paper_2103_16063_b200.search import device_weights, enumerate_calls, lpt_shard, run_calls  # noqa: E402
from paper_2103_16063_b200.stages import bind_problem  # noqa: E402
from paper_2103_16063_b200.workloads import c5_blockset  # noqa: E402

nb, D = int(sys.argv[1]), int(sys.argv[2])
ctx = _lib.context(0)
bs = c5_blockset(nb, D, jitter_seed=0)
bind_problem(ctx, bs)
calls, levels = enumerate_calls(max(1, D // 8), min(8, D), 8 * D, nb)
run_calls(ctx, calls[:4], 8 * D)   # warm-up
dw = device_weights(ctx, calls, 8 * D)
for world, wname, w in [(1, "closed", None)] + [(k, m, x) for k in (2, 4, 8)
                                                for m, x in (("closed", None), ("device", dw))]:
    own = lpt_shard(nb, calls, world, w)
    ts = []
    for r in range(world):
        mine = [c for c, o in zip(calls, own) if o == r]
        ctx.lib.pc_reset_cache(ctx.h)
        b = run_calls(ctx, mine, 8 * D)
        st = b.stats
        ts.append(f"{st.device_ms:.0f}+{st.span_ms:.0f}ms/{len(mine)}c/{st.dp_launches}L/"
                  f"{st.pairs/1e6:.0f}Mp")
    print(world, wname, "per-rank DP+span:", ts, flush=True)
