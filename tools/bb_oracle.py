"""Measurement only: the DP time of a full C5 enumeration with and without
the objective bound, the bound set to each call's own optimum
(PIPECUT_B200_BB_ORACLE) -- the most the bound can save.

    PIPECUT_B200_BB_ORACLE=1 python tools/bb_oracle.py nb D [nb D ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2103_16063_b200 import _lib  # noqa: E402
from paper_2103_16063_b200.search import enumerate_calls, run_calls  # noqa: E402
from paper_2103_16063_b200.stages import bind_problem  # noqa: E402
from paper_2103_16063_b200.workloads import c5_blockset  # noqa: E402

args = [int(x) for x in sys.argv[1:]] or [1024, 256, 4096, 256]
ctx = _lib.context(0)
for nb, D in zip(args[::2], args[1::2]):
    bs = c5_blockset(nb, D, jitter_seed=0)
    bind_problem(ctx, bs)
    calls, _ = enumerate_calls(max(1, D // 8), min(8, D), 8 * D, nb)
    for rep in range(2):
        print(f"nb={nb} D={D} rep {rep}", file=sys.stderr, flush=True)
        run_calls(ctx, calls, 8 * D, False, True)
