"""First partition_blocks call of a process vs the next (C1), with the library
phase timers: where the one-time cost goes."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2103_16063_b200 import _lib, partition_blocks
from paper_2103_16063_b200 import flatten as F
from paper_2103_16063_b200.workloads import config_partition

t = time.perf_counter(); _lib.context(0); print(f"context {1e3*(time.perf_counter()-t):.0f} ms", flush=True)
part, model, k, batch, cl = config_partition("C1")
for rep in range(3):
    F._ATOM_CACHE.clear()
    t0 = time.perf_counter(); fa = F.flatten_atoms(part, model); t1 = time.perf_counter()
    partition_blocks(part, model, k); t2 = time.perf_counter()
    print(f"rep {rep}: flatten {1e3*(t1-t0):.1f} ms, partition_blocks (cached flatten) {1e3*(t2-t1):.1f} ms", flush=True)
