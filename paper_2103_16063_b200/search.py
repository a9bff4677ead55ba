"""form_stage's candidate enumeration, run as device batches and sharded
across GPUs.

The reference's form_stage (pkg/src/pipecut/stages.py:372-413) walks widening
levels n = 1, 2, 4, ... (num_nodes % n == 0), and within a level every
(S, MB) pair is an independent `_run_dp` call; the first level with a feasible
plan wins and its candidates are ranked by (simulated iteration time,
objective, microbatches), first in (S, MB) order on ties.

Here the calls are independent device work units:
  * `run_calls` evaluates any list of them in one level-synchronous batch;
  * `form_stage_sharded` spreads them over the ranks of a torch.distributed
    group (one process per GPU, NCCL over NVLink) by LPT on the closed-form
    visit count and exchanges one fixed-size record per rank with a single
    `all_gather_into_tensor`; every rank then applies the reference's
    selection rule to the gathered records, so all ranks return the same
    `SearchResult`.
"""

from __future__ import annotations

import ctypes as C
import heapq
import time

import numpy as np

from . import _lib, abi
from .stages import (InvalidArgs, Plan, SearchBudgetExceeded, SearchOptions, SearchResult,
                     SearchStats, StagePlan, bind_overrides, bind_problem, call_shares,
                     checked_form_stage, times_nonneg)


def enumerate_calls(num_nodes: int, dpn: int, batch_size: int, nb: int):
    """(S, D, R, MB) calls and their widening-level index, in the reference's
    order (stages.py:389-403)."""
    calls, levels = [], []
    n, lv = 1, 0
    while n <= num_nodes:
        if num_nodes % n == 0:
            D, R = dpn * n, num_nodes // n
            for S in range(dpn * (n - 1) + 1, D + 1):
                if S > nb:
                    continue
                MB = 1
                while MB * R <= batch_size:
                    calls.append((S, D, R, MB))
                    levels.append(lv)
                    MB *= 2
            lv += 1
        n *= 2
    return calls, levels


def call_weight(nb: int, call) -> int:
    S, D, _, _ = call
    A, B = nb - S + 1, D - S + 1
    return S * (A * (A + 1) // 2) * (B * (B + 1) // 2)


def lpt_shard(nb: int, calls, world: int, weights=None):
    """Owner rank per call: longest-processing-time first, deterministic.
    ``weights`` (device_weights) default to the closed-form visit count."""
    w = list(weights) if weights is not None else [call_weight(nb, c) for c in calls]
    order = sorted(range(len(calls)), key=lambda i: (-w[i], i))
    heap = [(0, r) for r in range(world)]
    owner = [0] * len(calls)
    for i in order:
        load, r = heapq.heappop(heap)
        owner[i] = r
        heapq.heappush(heap, (load + int(w[i]) + 1, r))
    return owner


def device_weights(ctx: _lib.Context, calls, batch_size: int):
    """Feasible-pair sharding weights from the device key tables
    (pc_call_weights); identical on every rank."""
    n = len(calls)
    if ctx.problem_flat is not None:
        bind_overrides(ctx, ctx.problem_flat, call_shares(calls, batch_size))
    out = np.zeros(max(n, 1), np.int64)
    if n:
        arr = np.ascontiguousarray(np.asarray(calls, np.int32).reshape(n, 4))
        ctx.check(ctx.lib.pc_call_weights(ctx.h, n, arr.ctypes.data, batch_size, out.ctypes.data),
                  "pc_call_weights")
    return out[:n].tolist()


# the library bounds the DP of batches from this many closed-form visits up
# (api.cu: BOUND_MIN_VISITS); their per-call cost then follows the DP cells
BOUNDED_BATCH_VISITS = 2e8


def shard_weights(ctx: _lib.Context, calls, batch_size: int, nb: int):
    """LPT weights of the calls.  Unbounded searches: `device` -- feasible
    pairs from the key tables (pc_call_weights).  Searches large enough for the
    objective bound: `cells` -- S * A * B DP cells, which tracks the bounded
    kernel's per-call cost best (4096 x 256 on 4 GPUs: 367 ms per step vs 405 ms
    with either visit-based weight, r2n).  PIPECUT_B200_SHARD_WEIGHTS forces
    `device`, `visits` (closed-form unpruned visits) or `cells`."""
    import os
    kind = os.environ.get("PIPECUT_B200_SHARD_WEIGHTS")
    if kind is None:
        kind = "cells" if sum(call_weight(nb, c) for c in calls) >= BOUNDED_BATCH_VISITS \
            else "device"
    if kind == "visits":
        return [call_weight(nb, c) for c in calls]
    if kind == "cells":
        return [c[0] * (nb - c[0] + 1) * (c[1] - c[0] + 1) for c in calls]
    return device_weights(ctx, calls, batch_size)


class BatchResult:
    """Per-call records of one device batch: `results` is a structured array
    with the PcCallResult fields, `bufs[i]` the call's stage arrays."""

    def __init__(self, calls, results, bufs, stats):
        self.calls = calls
        self.results = results
        self.bufs = bufs
        self.stats = stats

    def feasible(self, i):
        return bool(self.results[i]["feasible"])

    def plan(self, i, batch_size) -> Plan | None:
        if not self.results[i]["feasible"]:
            return None
        S, D, R, MB = self.calls[i]
        buf = self.bufs[i]
        stages = tuple(
            StagePlan(blocks=(int(buf.lo[k]), int(buf.hi[k])), devices=int(buf.devices[k]),
                      replicas=int(buf.devices[k]) * R, t_fwd=float(buf.t_fwd[k]),
                      t_bwd=float(buf.t_bwd[k]), mem=int(buf.mem[k]))
            for k in range(S))
        return Plan(stages=stages, microbatches=MB, replica_factor=R,
                    objective=float(self.results[i]["objective"]), batch_size=batch_size,
                    devices_total=D)


def run_calls(ctx: _lib.Context, calls, batch_size: int, disable_pruning: bool = False,
              want_iteration: bool = True) -> BatchResult:
    n = len(calls)
    if ctx.problem_flat is not None:
        bind_overrides(ctx, ctx.problem_flat, call_shares(calls, batch_size))
    arr = np.ascontiguousarray(np.asarray(calls, np.int32).reshape(n, 4)) if n else np.zeros((1, 4), np.int32)
    res = np.zeros(max(n, 1), abi.CALL_RESULT_DTYPE)
    plans = abi.PlanArena([c[0] for c in calls])
    st = abi.PcStats()
    if n:
        rc = ctx.lib.pc_run_calls(ctx.h, n, arr.ctypes.data_as(C.POINTER(abi.PcCall)), batch_size,
                                  int(bool(disable_pruning)), int(bool(want_iteration)),
                                  res.ctypes.data_as(C.POINTER(abi.PcCallResult)), plans.ptr(),
                                  C.byref(st))
        ctx.check(rc, "pc_run_calls")
    return BatchResult(calls, res[:n], plans, st)


def rank_key(iteration, objective, MB, index):
    # min by (iteration_time, objective, microbatches), first wins (stages.py:407-411)
    return (iteration, objective, MB, index)


def select(levels, visits, feasible, keys, budget):
    """Reference selection over per-call records in call order.

    Returns (best index or -1, counted calls, visits, crossing call or -1,
    visits before the crossing call)."""
    running = 0
    counted = 0
    n = len(levels)
    i = 0
    while i < n:
        lv = levels[i]
        j = i
        best = -1
        while j < n and levels[j] == lv:
            counted += 1
            if budget is not None and running + visits[j] > budget:
                return -1, counted, running, j, running
            running += visits[j]
            if feasible[j] and (best < 0 or keys[j] < keys[best]):
                best = j
            j += 1
        if best >= 0:
            return best, counted, running, -1, running
        i = j
    return -1, counted, running, -1, running


# --------------------------------------------------------------------------- sharded
_REC = 4  # per call: visits, feasible, iteration, objective


def _pack(nb, calls, levels, owner, rank, batch, local_idx, n_levels, max_stages):
    """This rank's record: per-call (visits, feasible, iteration, objective)
    for the calls it owns (zeros elsewhere) + its best plan per level."""
    n = len(calls)
    plan_w = 4 + 6 * max_stages
    rec = np.zeros(n * _REC + n_levels * plan_w, np.float64)
    best = {}
    for li, gi in enumerate(local_idx):
        r = batch.results[li]
        rec[gi * _REC + 0] = r["visits"]
        rec[gi * _REC + 1] = r["feasible"]
        rec[gi * _REC + 2] = r["iteration_time"]
        rec[gi * _REC + 3] = r["objective"]
        if r["feasible"]:
            key = rank_key(float(r["iteration_time"]), float(r["objective"]), calls[gi][3], gi)
            lv = levels[gi]
            if lv not in best or key < best[lv][0]:
                best[lv] = (key, li, gi)
    base = n * _REC
    for lv, (_, li, gi) in best.items():
        o = base + lv * plan_w
        buf = batch.bufs[li]
        S = calls[gi][0]
        rec[o] = 1
        rec[o + 1] = gi
        rec[o + 2] = S
        rec[o + 3] = batch.results[li]["objective"]
        k = o + 4
        rec[k:k + S] = buf.lo[:S]
        rec[k + S:k + 2 * S] = buf.hi[:S]
        rec[k + 2 * S:k + 3 * S] = buf.devices[:S]
        rec[k + 3 * S:k + 4 * S] = buf.t_fwd[:S]
        rec[k + 4 * S:k + 5 * S] = buf.t_bwd[:S]
        rec[k + 5 * S:k + 6 * S] = buf.mem[:S]    # exact: mem < 2**53
    return rec, plan_w


def exchange(rec: np.ndarray, group=None, device=None) -> np.ndarray:
    """all_gather_into_tensor of one fixed-size float64 record per rank
    (NCCL on `device`, or gloo on CPU when device is None)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return rec.reshape(1, -1)
    world = dist.get_world_size(group)
    mine = torch.from_numpy(rec)
    if device is not None:
        mine = mine.to(device)
    if mine.is_cuda:
        out = torch.empty(world * rec.size, dtype=torch.float64, device=mine.device)
        dist.all_gather_into_tensor(out, mine, group=group)
        return out.view(world, rec.size).cpu().numpy()
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine, group=group)
    return torch.stack(parts).numpy()


def decide(allrec: np.ndarray, calls, levels, owner, plan_w: int, budget, batch_size: int,
           upto: int | None = None):
    """Apply the reference's selection to the gathered records (to the first
    `upto` calls when given: the levels evaluated so far).

    Returns ("plan", SearchResult) or ("budget", crossing call, visits before)."""
    n = len(calls)
    m = n if upto is None else upto
    world = allrec.shape[0]
    per = allrec[:, :n * _REC].reshape(world, n, _REC)
    own = np.asarray(owner[:m], dtype=np.int64)
    g = per[own, np.arange(m)] if m else np.zeros((0, _REC))
    visits = [int(v) for v in g[:, 0]]
    feasible = [bool(f) for f in g[:, 1]]
    keys = [rank_key(float(g[i, 2]), float(g[i, 3]), calls[i][3], i) for i in range(m)]
    best, counted, running, cross, before = select(levels[:m], visits, feasible, keys, budget)
    if cross >= 0:
        return ("budget", cross, before)
    stats = SearchStats(visits=running, dp_calls=counted)
    if best < 0:
        return ("plan", SearchResult(None, stats))
    o = n * _REC + levels[best] * plan_w
    row = allrec[owner[best]]
    if row[o] != 1 or int(row[o + 1]) != best:
        raise RuntimeError("inconsistent shard record")
    S, D, R, MB = calls[best]
    k = o + 4
    stages = tuple(
        StagePlan(blocks=(int(row[k + j]), int(row[k + S + j])), devices=int(row[k + 2 * S + j]),
                  replicas=int(row[k + 2 * S + j]) * R, t_fwd=float(row[k + 3 * S + j]),
                  t_bwd=float(row[k + 4 * S + j]), mem=int(row[k + 5 * S + j]))
        for j in range(S))
    plan = Plan(stages=stages, microbatches=MB, replica_factor=R, objective=float(row[o + 3]),
                batch_size=batch_size, devices_total=D)
    return ("plan", SearchResult(plan, stats))


@_lib.serialized
def form_stage_sharded(num_nodes: int, devices_per_node: int, batch_size: int, blocks,
                       options=None, *, group=None, timings: dict | None = None,
                       speculative: bool = True):
    """form_stage with its DP calls spread over every rank of a
    torch.distributed group (one GPU per rank, NCCL); all ranks return the
    reference's SearchResult.

    ``speculative`` (SURVEY.md §8e schedule ii) shards every widening level's
    calls at once and exchanges once; ``speculative=False`` (schedule i, the
    reference's latency order) runs the levels in order, sharding each level's
    calls and exchanging after each, and stops at the first level with a
    feasible plan (or at a budget crossing).  Results and stats are identical."""
    import torch
    import torch.distributed as dist

    if num_nodes < 1 or devices_per_node < 1 or batch_size < 1:
        raise InvalidArgs("node count, devices per node and batch size must be at least 1")
    opts = options or SearchOptions()
    dist_on = dist.is_initialized()
    world = dist.get_world_size(group) if dist_on else 1
    rank = dist.get_rank(group) if dist_on else 0
    ctx = _lib.context()
    tm = {} if timings is not None else None
    flat = bind_problem(ctx, blocks, tm)
    if not times_nonneg(flat):
        # negative span times: the reference can raise InvalidPlan while ranking
        # (stages.checked_form_stage); every rank runs that exact path itself
        return checked_form_stage(ctx, num_nodes, devices_per_node, batch_size, blocks, opts)
    if tm is not None:
        # device-resident part of the call: CUDA events on the library stream
        ctx.check(ctx.lib.pc_timer_start(ctx.h), "timer")
        t_res = time.perf_counter()
    nb = len(blocks)
    calls, levels = enumerate_calls(num_nodes, devices_per_node, batch_size, nb)
    n_levels = (max(levels) + 1) if levels else 0
    max_stages = max((c[0] for c in calls), default=1)
    dev = torch.device("cuda", ctx.device)
    weights = shard_weights(ctx, calls, batch_size, nb) if world > 1 else None
    if not speculative:
        return _sharded_by_level(ctx, calls, levels, n_levels, max_stages, nb, weights, world,
                                 rank, group, dev, opts, batch_size)
    owner = lpt_shard(nb, calls, world, weights)
    local_idx = [i for i in range(len(calls)) if owner[i] == rank]
    if tm is not None:
        t_calls = time.perf_counter()
    batch = run_calls(ctx, [calls[i] for i in local_idx], batch_size,
                      opts.disable_pruning, True)
    if tm is not None:
        t_pack = time.perf_counter()
    rec, plan_w = _pack(nb, calls, levels, owner, rank, batch, local_idx, n_levels, max_stages)
    if tm is not None:
        t_ex = time.perf_counter()
    allrec = exchange(rec, group, dev)
    if tm is not None:
        t_dec = time.perf_counter()
    out = decide(allrec, calls, levels, owner, plan_w, opts.visit_budget, batch_size)
    if tm is not None:
        t_end = time.perf_counter()
        ms = C.c_double()
        ctx.check(ctx.lib.pc_timer_stop(ctx.h, C.byref(ms)), "timer")
        st = batch.stats
        timings.update(
            tm, pairs=int(st.pairs), candidates=int(st.candidates),
            dp_ms=float(st.device_ms), span_ms=float(st.span_ms), post_ms=float(st.post_ms),
            dp_launches=int(st.dp_launches), kernel_launches=int(st.kernel_launches),
            local_unpruned=int(st.visits_unpruned),
            unpruned=sum(call_weight(nb, c) for c in calls),
            h2d_bytes=_flat_bytes(ctx.problem_flat), d2h_bytes=int(rec.nbytes),
            resident_ms=ms.value,
            weights_ms=(t_calls - t_res) * 1e3, run_calls_ms=(t_pack - t_calls) * 1e3,
            pack_ms=(t_ex - t_pack) * 1e3, exchange_ms=(t_dec - t_ex) * 1e3,
            decide_ms=(t_end - t_dec) * 1e3)
    if out[0] == "plan":
        return out[1]
    _, cross, before = out
    _raise_crossing(ctx, calls, owner, local_idx, cross, before, world, rank, group, dev, opts,
                    batch_size)


def crossing_visits(ctx, index, call, before, budget, batch_size, disable_pruning) -> int:
    """Visits at the first cell past `budget` inside `call`, position `index`
    of the last run_calls batch (stages.py:214-216); a call whose flags went
    with an earlier chunk of that batch is run again alone."""
    at = C.c_int64()
    ctx.check(ctx.lib.pc_last_crossing(ctx.h, index, before, budget, C.byref(at)),
              "pc_last_crossing")
    if at.value < -1:
        run_calls(ctx, [call], batch_size, disable_pruning, False)
        ctx.check(ctx.lib.pc_last_crossing(ctx.h, 0, before, budget, C.byref(at)),
                  "pc_last_crossing")
    return int(at.value)


def _raise_crossing(ctx, calls, owner, local_idx, cross, before, world, rank, group, dev, opts,
                    batch_size):
    """SearchBudgetExceeded with the exact visit count at the crossing cell,
    computed by the rank that owns the crossing call (its last batch)."""
    import torch
    import torch.distributed as dist

    v = np.zeros(1, np.float64)
    if owner[cross] == rank:
        v[0] = crossing_visits(ctx, local_idx.index(cross), calls[cross], before,
                               int(opts.visit_budget), batch_size, opts.disable_pruning)
    if world > 1:
        t = torch.from_numpy(v).to(dev)
        # owner[] holds ranks within `group`; broadcast's src is a global rank
        src = owner[cross] if group is None else dist.get_global_rank(group, owner[cross])
        dist.broadcast(t, src=src, group=group)
        v = t.cpu().numpy()
    raise SearchBudgetExceeded(int(v[0]), int(opts.visit_budget))


# Schedule (i): a widening level below this many closed-form unpruned visits
# runs whole on every rank instead of being sharded: such a level takes
# ~15 ms or less on one B200 (tools/level_costs.py, r2c: 1024 x 256 level 1,
# 5.3e9 visits, 15 ms), so splitting it saves less than the pack + all-gather
# + decide round it would cost.
REPLICATE_BELOW = 5e9


def _sharded_by_level(ctx, calls, levels, n_levels, max_stages, nb, weights, world, rank, group,
                      dev, opts, batch_size):
    """Schedule (i): widening levels in order, each level's calls sharded
    (LPT within the level) and one exchange per level -- or, for a light level,
    run whole on every rank with no exchange; the reference's rule is applied
    to the calls evaluated so far after every level."""
    n = len(calls)
    owner = [0] * n
    allrec = None
    end = 0
    plan_w = 4 + 6 * max_stages
    for lv in range(n_levels):
        start = end
        while end < n and levels[end] == lv:
            end += 1
        idx = list(range(start, end))
        replicated = world == 1 or sum(call_weight(nb, calls[i]) for i in idx) < REPLICATE_BELOW
        if replicated:
            for i in idx:
                owner[i] = rank        # every rank computes (and owns) every call
        else:
            lv_owner = lpt_shard(nb, [calls[i] for i in idx], world,
                                 None if weights is None else [weights[i] for i in idx])
            for i, o in zip(idx, lv_owner):
                owner[i] = o
        local_idx = [i for i in idx if owner[i] == rank]
        batch = run_calls(ctx, [calls[i] for i in local_idx], batch_size,
                          opts.disable_pruning, True)
        rec, plan_w = _pack(nb, calls, levels, owner, rank, batch, local_idx, n_levels,
                            max_stages)
        if replicated:
            got = np.zeros((max(world, 1), rec.size))
            got[rank] = rec                                    # this rank's row only
        else:
            got = exchange(rec, group, dev)
        allrec = got if allrec is None else allrec + got      # disjoint slots per level
        out = decide(allrec, calls, levels, owner, plan_w, opts.visit_budget, batch_size,
                     upto=end)
        if out[0] == "budget":
            _, cross, before = out
            _raise_crossing(ctx, calls, owner, local_idx, cross, before,
                            1 if replicated else world, rank, group, dev, opts, batch_size)
        result = out[1]
        if result.plan is not None or end == n:
            return result
    return decide(np.zeros((max(world, 1), n * _REC + n_levels * plan_w)), calls, levels,
                  owner, plan_w, opts.visit_budget, batch_size)[1]


def _flat_bytes(flat) -> int:
    if flat is None:
        return 0
    return int(sum(getattr(flat, f).nbytes for f in flat.__dataclass_fields__
                   if isinstance(getattr(flat, f), np.ndarray)))
