"""Time partition_blocks (GPU drop-in vs reference) on C1-C4."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2103_16063_b200 import partition_blocks  # noqa: E402
from paper_2103_16063_b200._host import pipecut as pc  # noqa: E402
from paper_2103_16063_b200.workloads import config_partition  # noqa: E402

for name in sys.argv[1:] or ["C1", "C2", "C3", "C4"]:
    part, model, k, batch, cl = config_partition(name)
    ts = []
    for _ in range(4):
        t0 = time.perf_counter()
        bs = partition_blocks(part, model, k)
        ts.append(time.perf_counter() - t0)
    t0 = time.perf_counter()
    ref = pc.partition_blocks(part, model, k)
    tr = time.perf_counter() - t0
    assert bs.block_atoms == ref.block_atoms and bs.costs == ref.costs
    print(f"{name}: gpu {min(ts)*1e3:.1f} ms (cold {ts[0]*1e3:.1f}), reference {tr*1e3:.1f} ms, "
          f"{len(part.atoms)} atoms -> {len(bs)} blocks", flush=True)
