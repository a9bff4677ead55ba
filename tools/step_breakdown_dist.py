"""Per-rank phases of one sharded step (torchrun, NCCL): run_calls / pack /
exchange / decide, each bracketed by cuda synchronize."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import torch.distributed as dist
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, world = dist.get_rank(), dist.get_world_size()
from paper_2103_16063_b200 import _lib
from paper_2103_16063_b200.search import (_pack, decide, device_weights, enumerate_calls, exchange,
                                          lpt_shard, run_calls)
from paper_2103_16063_b200.stages import bind_problem
from paper_2103_16063_b200.workloads import c5_blockset

ctx = _lib.context(local)
bs = c5_blockset(1024, 256, jitter_seed=0)
bind_problem(ctx, bs)
calls, levels = enumerate_calls(32, 8, 2048, 1024)
owner = lpt_shard(1024, calls, world, device_weights(ctx, calls, 2048))
idx = [i for i in range(len(calls)) if owner[i] == rank]
mine = [calls[i] for i in idx]
dev = torch.device("cuda", local)
for rep in range(4):
    ctx.lib.pc_reset_cache(ctx.h)
    torch.cuda.synchronize(); dist.barrier()
    t0 = time.perf_counter()
    b = run_calls(ctx, mine, 2048, False, True)
    t1 = time.perf_counter()
    rec, pw = _pack(1024, calls, levels, owner, rank, b, idx, max(levels) + 1, max(c[0] for c in calls))
    t2 = time.perf_counter()
    allrec = exchange(rec, None, dev)
    t3 = time.perf_counter()
    out = decide(allrec, calls, levels, owner, pw, None, 2048)
    t4 = time.perf_counter()
    if rep >= 2:
        print(f"[rank {rank}] run_calls {1e3*(t1-t0):.1f} (dp {b.stats.device_ms:.1f}) pack {1e3*(t2-t1):.1f} "
              f"exchange {1e3*(t3-t2):.1f} decide {1e3*(t4-t3):.1f} ms", flush=True)
dist.destroy_process_group()
