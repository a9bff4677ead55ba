"""Schedule (i) (form_stage_sharded, speculative=False) on the C5 headline,
per-run wall time and per-level device times."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2103_16063_b200 import _lib  # noqa: E402
from paper_2103_16063_b200.search import form_stage_sharded  # noqa: E402
from paper_2103_16063_b200.workloads import c5_blockset  # noqa: E402

nb, D = 4096, 256
bs = c5_blockset(nb, D, jitter_seed=0)
ctx = _lib.context(0)
for i in range(6):
    ctx.lib.pc_reset_cache(ctx.h)
    t0 = time.perf_counter()
    r = form_stage_sharded(D // 8, 8, 8 * D, bs, speculative=False)
    torch.cuda.synchronize()
    print(f"run {i}: {(time.perf_counter() - t0) * 1e3:.1f} ms, visits {r.stats.visits}, calls {r.stats.dp_calls}",
          flush=True)
