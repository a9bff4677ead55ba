"""partition_blocks phases on C1-C4: host atom flattening, the library call
(coarsening on device + host greedy), result objects."""
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2103_16063_b200 import _lib, abi  # noqa: E402
from paper_2103_16063_b200 import flatten as F  # noqa: E402
from paper_2103_16063_b200 import partition_blocks  # noqa: E402
from paper_2103_16063_b200.workloads import config_partition  # noqa: E402

ctx = _lib.context(0)
for name in sys.argv[1:] or ["C1", "C2", "C3", "C4"]:
    part, model, k, batch, cl = config_partition(name)
    partition_blocks(part, model, k)
    for rep in range(3):
        F._ATOM_CACHE.clear()
        t0 = time.perf_counter()
        fa = F.flatten_atoms(part, model)
        t1 = time.perf_counter()
        st = abi.atoms_struct(fa)
        n = fa.n
        nbk = C.c_int32()
        off = np.zeros(n + 1, np.int32)
        at = np.zeros(n, np.int32)
        tf, tb = np.zeros(n), np.zeros(n)
        mem = np.zeros(n, np.int64)
        err = np.zeros(2, np.int64)
        rc = ctx.lib.pc_partition_blocks(ctx.h, C.byref(st), k, C.byref(nbk), off.ctypes.data,
                                         at.ctypes.data, tf.ctypes.data, tb.ctypes.data,
                                         mem.ctypes.data, err.ctypes.data)
        t2 = time.perf_counter()
        F._ATOM_CACHE.clear()
        t3 = time.perf_counter()
        partition_blocks(part, model, k)
        t4 = time.perf_counter()
        print(f"{name}: flatten_atoms {1e3*(t1-t0):.1f} ms, pc_partition_blocks {1e3*(t2-t1):.1f} ms, "
              f"whole drop-in {1e3*(t4-t3):.1f} ms", flush=True)
