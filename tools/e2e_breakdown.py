"""Host-side phases of the public-API path (form_stage_sharded) at N=1."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2103_16063_b200 import _lib
from paper_2103_16063_b200 import flatten as F
from paper_2103_16063_b200 import abi
from paper_2103_16063_b200.search import device_weights, enumerate_calls, form_stage_sharded
from paper_2103_16063_b200.workloads import c5_blockset
import ctypes as C

ctx = _lib.context(0)
bs = c5_blockset(1024, 256, jitter_seed=0)
calls, levels = enumerate_calls(32, 8, 2048, 1024)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    flat = F.flatten_blockset(bs)
    t1 = time.perf_counter()
    st = abi.problem_struct(flat)
    ctx.check(ctx.lib.pc_set_problem(ctx.h, C.byref(st)), "set")
    t2 = time.perf_counter()
    w = device_weights(ctx, calls, 2048)
    t3 = time.perf_counter()
    ctx.problem_owner = None
    ctx.lib.pc_reset_cache(ctx.h)
    t4 = time.perf_counter()
    r = form_stage_sharded(32, 8, 2048, bs)
    t5 = time.perf_counter()
    print(f"flatten {1e3*(t1-t0):.1f} set_problem {1e3*(t2-t1):.1f} weights {1e3*(t3-t2):.1f} "
          f"form_stage_sharded {1e3*(t5-t4):.1f} ms", flush=True)
