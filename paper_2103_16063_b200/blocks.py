"""Drop-in `partition_blocks` backed by the B200 coarsening kernels.

Same signature, results and exceptions as the reference
(pkg/src/pipecut/blocks.py:361-397): takes the reference's AtomicPartition and
CostModel, returns the reference's own BlockSet (blocks in dependency order,
costs = profile at microbatch 1 with checkpointing), raises ValueError for
k < 1, InfeasibleAtom and CompactionStuck.  The memory/convexity/traffic
predicates and all profiles run on the GPU (csrc/blocks.cu).
"""

from __future__ import annotations

import ctypes as C
import time

import numpy as np

from . import _lib, abi
from ._host import pipecut as _pc
from .flatten import flatten_atoms

BlockSet = _pc.blocks.BlockSet
InfeasibleAtom = _pc.blocks.InfeasibleAtom
CompactionStuck = _pc.blocks.CompactionStuck
CostRecord = _pc.costs.CostRecord


@_lib.serialized
def partition_blocks(partition, model, k: int = 32, *, timings: dict | None = None):
    """Group atoms into at most k convex, memory-feasible blocks (GPU).
    ``timings`` (optional) gets the host flatten, library call (coarsening,
    refinement, block profiles) and object-build times in ms."""
    if k < 1:
        raise ValueError("k must be at least 1")
    t0 = time.perf_counter()
    fa = flatten_atoms(partition, model)
    t1 = time.perf_counter()
    ctx = _lib.context()
    st = abi.atoms_struct(fa)
    n = fa.n
    nbk = C.c_int32()
    off = np.zeros(n + 1, np.int32)
    at = np.zeros(n, np.int32)
    tf = np.zeros(n, np.float64)
    tb = np.zeros(n, np.float64)
    mem = np.zeros(n, np.int64)
    err = np.zeros(2, np.int64)
    rc = ctx.lib.pc_partition_blocks(ctx.h, C.byref(st), k, C.byref(nbk), off.ctypes.data,
                                     at.ctypes.data, tf.ctypes.data, tb.ctypes.data,
                                     mem.ctypes.data, err.ctypes.data)
    if rc == abi.PC_ERR_ATOM:
        atom = partition.atoms[int(err[0])]
        raise InfeasibleAtom(atom.id, int(err[1]), fa.budget)
    if rc == abi.PC_ERR_STUCK:
        raise CompactionStuck(int(err[0]), k)
    ctx.check(rc, "partition_blocks")
    t2 = time.perf_counter()
    nb = int(nbk.value)
    glist = tuple(tuple(int(x) for x in at[off[b]:off[b + 1]]) for b in range(nb))
    width = max(3, len(str(nb)))
    blocks = tuple(partition.merged(grp, f"B{idx:0{width}d}") for idx, grp in enumerate(glist))
    costs = tuple(CostRecord(t_fwd_sec=float(tf[b]), t_bwd_sec=float(tb[b]), mem_bytes=int(mem[b]))
                  for b in range(nb))
    out = BlockSet(partition=partition, model=model, block_atoms=glist, blocks=blocks,
                   costs=costs)
    if timings is not None:
        timings.update(flatten_ms=(t1 - t0) * 1e3, library_ms=(t2 - t1) * 1e3,
                       build_ms=(time.perf_counter() - t2) * 1e3)
    return out
