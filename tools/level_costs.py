"""Per widening level of form_stage: closed-form unpruned visits, the
device sharding weight (pc_call_weights) and the one-GPU wall time of the
level's calls as one batch -- calibrates when schedule (i) shards a level
(search._sharded_by_level) instead of running it on every rank.

    python tools/level_costs.py [nb D ...]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2103_16063_b200 import _lib  # noqa: E402
from paper_2103_16063_b200.search import call_weight, device_weights, enumerate_calls, run_calls  # noqa: E402
from paper_2103_16063_b200.stages import bind_problem  # noqa: E402
from paper_2103_16063_b200.workloads import c5_blockset, config_partition  # noqa: E402
from paper_2103_16063_b200 import partition_blocks  # noqa: E402


def report(name, bs, nodes, dpn, BS):
    ctx = _lib.context(0)
    bind_problem(ctx, bs)
    nb = len(bs)
    calls, levels = enumerate_calls(nodes, dpn, BS, nb)
    w = device_weights(ctx, calls, BS)
    for lv in sorted(set(levels)):
        idx = [i for i in range(len(calls)) if levels[i] == lv]
        sub = [calls[i] for i in idx]
        ts = []
        for _ in range(3):
            ctx.lib.pc_reset_cache(ctx.h)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            b = run_calls(ctx, sub, BS, False, True)
            ts.append((time.perf_counter() - t0) * 1e3)
        feas = int(sum(b.results["feasible"]))
        print(f"{name} level {lv}: calls {len(sub)} feasible {feas} unpruned "
              f"{sum(call_weight(nb, c) for c in sub):.3e} weight {sum(w[i] for i in idx):.3e} "
              f"ms {min(ts):.2f}", flush=True)


if __name__ == "__main__":
    args = [int(x) for x in sys.argv[1:]] or [4096, 1024, 1024, 256, 4096, 256]
    for nb, D in zip(args[::2], args[1::2]):
        report(f"C5 nb={nb} D={D}", c5_blockset(nb, D, jitter_seed=0), max(1, D // 8),
               min(8, D), 8 * D)
    for c in ("C2", "C4"):
        part, model, k, batch, cl = config_partition(c)
        report(c, partition_blocks(part, model, k), cl.num_nodes, cl.devices_per_node, batch)
