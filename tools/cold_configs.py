"""Cold runs of C1..C4 in one process (bench latency order), phases timed."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2103_16063_b200 import _lib, form_stage, partition_blocks
from paper_2103_16063_b200 import flatten as F
from paper_2103_16063_b200.workloads import config_partition

ctx = _lib.context(0)
if "--after-c5" in sys.argv:                 # the bench's order: the big search first
    from paper_2103_16063_b200.search import enumerate_calls, run_calls
    from paper_2103_16063_b200.stages import bind_problem
    from paper_2103_16063_b200.workloads import c5_blockset
    bs5 = c5_blockset(1024, 256, jitter_seed=0)
    bind_problem(ctx, bs5)
    calls, _ = enumerate_calls(32, 8, 2048, 1024)
    run_calls(ctx, calls, 2048)
    print("ran the C5 search", flush=True)
for name in ("C1", "C2", "C3", "C4"):
    part, model, k, batch, cl = config_partition(name)
    for rep in range(2):
        F._ATOM_CACHE.clear()
        ctx.problem_owner = None
        ctx.lib.pc_reset_cache(ctx.h)
        t0 = time.perf_counter()
        fa = F.flatten_atoms(part, model)
        t1 = time.perf_counter()
        bs = partition_blocks(part, model, k)
        t2 = time.perf_counter()
        res = form_stage(cl.num_nodes, cl.devices_per_node, batch, bs)
        t3 = time.perf_counter()
        print(f"{name} rep {rep}: flatten {1e3*(t1-t0):.1f} blocks {1e3*(t2-t1):.1f} "
              f"form_stage {1e3*(t3-t2):.1f} ms", flush=True)
