"""cProfile of the partition_blocks drop-in (atom cache cleared, warm device)."""
import cProfile
import os
import pstats
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2103_16063_b200 import flatten as F  # noqa: E402
from paper_2103_16063_b200 import partition_blocks  # noqa: E402
from paper_2103_16063_b200.workloads import config_partition  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
part, model, k, batch, cl = config_partition(name)
partition_blocks(part, model, k)
F._ATOM_CACHE.clear()
pr = cProfile.Profile()
pr.enable()
partition_blocks(part, model, k)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(28)
