"""Drop-in `form_stage_dp` / `form_stage` backed by the B200 stage DP.

Same signatures, argument meaning, results and exceptions as the reference
(pkg/src/pipecut/stages.py:282-291 and 372-413): callers pass a reference
`BlockSet` and `SearchOptions`, and get the reference's own `SearchResult`,
`Plan`, `StagePlan` and `SearchStats` back; `InvalidArgs` and
`SearchBudgetExceeded` are the reference's classes.  All search arithmetic
runs on the GPU through libpipecut_b200.so.
"""

from __future__ import annotations

import ctypes as C
import time
import weakref

from . import _lib, abi
from ._host import pipecut as _pc
from .flatten import flatten_blockset, resolve_overrides

_stages = _pc.stages
InvalidArgs = _stages.InvalidArgs
SearchBudgetExceeded = _stages.SearchBudgetExceeded
TooLarge = _stages.TooLarge
SearchOptions = _stages.SearchOptions
SearchResult = _stages.SearchResult
SearchStats = _stages.SearchStats
StagePlan = _stages.StagePlan
Plan = _stages.Plan


def bind_problem(ctx: _lib.Context, blocks, timings: dict | None = None):
    """Upload the flattened BlockSet once per BlockSet object.  ``timings``
    gets flatten_ms (host) and upload_ms (pc_set_problem: host->device copy
    of the arrays and the span-input tables)."""
    owner = ctx.problem_owner() if ctx.problem_owner is not None else None
    if owner is blocks:
        if timings is not None:
            timings.update(flatten_ms=0.0, upload_ms=0.0)
        return ctx.problem_flat
    t0 = time.perf_counter()
    flat = flatten_blockset(blocks)
    t1 = time.perf_counter()
    st = abi.problem_struct(flat)
    ctx.check(ctx.lib.pc_set_problem(ctx.h, C.byref(st)), "pc_set_problem")
    if timings is not None:
        timings.update(flatten_ms=(t1 - t0) * 1e3, upload_ms=(time.perf_counter() - t1) * 1e3)
    ctx.problem_owner = weakref.ref(blocks)
    ctx.problem_flat = flat
    ctx.problem_shares = frozenset()
    return flat


def call_shares(calls, batch_size: int):
    """Microbatch shares m = batch // (MB * R * devices) the calls' span
    profiles are taken at (stages.py:201-206)."""
    out = set()
    for S, D, R, MB in calls:
        for dev in range(1, D - S + 2):
            m = batch_size // (MB * R * dev)
            if m >= 1:
                out.add(m)
    return out


def bind_overrides(ctx: _lib.Context, flat, shares) -> None:
    """Resolve measured cost-table entries (costs.py:130-148) for every share
    a search will touch; the device profiles take them from there.  Shares
    accumulate per bound BlockSet so cached span tables survive."""
    if not flat.has_cost_table:
        return
    want = ctx.problem_shares | frozenset(int(m) for m in shares)
    if want == ctx.problem_shares:
        return
    ms, has, tf, tb, act = resolve_overrides(flat.cost_config, flat.task_nodes, want)
    ctx.check(ctx.lib.pc_set_overrides(ctx.h, len(ms), ms.ctypes.data, has.ctypes.data,
                                       tf.ctypes.data, tb.ctypes.data, act.ctypes.data),
              "pc_set_overrides")
    ctx.problem_shares = want


def _check_args(blocks, S, D, batch_size, replica_factor, microbatches):
    # same messages as stages.py:160-168
    if S < 1 or D < 1 or batch_size < 1 or replica_factor < 1 or microbatches < 1:
        raise InvalidArgs("stage count, devices, batch size, replicas and "
                          "microbatches must all be at least 1")
    if S > D:
        raise InvalidArgs(f"cannot run {S} stages on {D} devices")
    if S > len(blocks):
        raise InvalidArgs(f"cannot cut {len(blocks)} blocks into {S} stages")


def plan_from_buffers(buf: abi.PlanBuffers, batch_size: int) -> Plan:
    s = buf.s
    R = int(s.R)
    stages = tuple(
        StagePlan(blocks=(int(buf.lo[i]), int(buf.hi[i])), devices=int(buf.devices[i]),
                  replicas=int(buf.devices[i]) * R, t_fwd=float(buf.t_fwd[i]),
                  t_bwd=float(buf.t_bwd[i]), mem=int(buf.mem[i]))
        for i in range(int(s.n_stages)))
    return Plan(stages=stages, microbatches=int(s.MB), replica_factor=R,
                objective=float(s.objective), batch_size=int(batch_size),
                devices_total=int(s.D))


def _budget(opts) -> int:
    return -1 if opts.visit_budget is None else int(opts.visit_budget)


@_lib.serialized
def form_stage_dp(blocks, S: int, D: int, batch_size: int, replica_factor: int,
                  microbatches: int, options=None):
    """Optimal S-stage assignment of the block list onto D devices (GPU)."""
    _check_args(blocks, S, D, batch_size, replica_factor, microbatches)
    opts = options or SearchOptions()
    ctx = _lib.context()
    flat = bind_problem(ctx, blocks)
    bind_overrides(ctx, flat, call_shares([(S, D, replica_factor, microbatches)], batch_size))
    buf = abi.PlanBuffers(S)
    st = abi.PcStats()
    rc = ctx.lib.pc_form_stage_dp(ctx.h, S, D, batch_size, replica_factor, microbatches,
                                  int(bool(opts.disable_pruning)), _budget(opts),
                                  C.byref(buf.s), C.byref(st))
    ctx.check(rc, "form_stage_dp")
    if rc == abi.PC_ERR_BUDGET:
        raise SearchBudgetExceeded(int(st.visits), int(opts.visit_budget))
    stats = SearchStats(visits=int(st.visits), dp_calls=int(st.dp_calls))
    plan = plan_from_buffers(buf, batch_size) if rc == abi.PC_OK else None
    return SearchResult(plan, stats)


@_lib.serialized
def form_stage(num_nodes: int, devices_per_node: int, batch_size: int, blocks,
               options=None, *, speculative: bool | None = None,
               last_stats: dict | None = None):
    """Search replica factor, stage count and microbatch count together (GPU).

    Batching of the widening levels: ``speculative=True`` evaluates every level
    in one device batch, ``False`` one batch per level, and the default
    (``None``) the first level alone and then, only while no level was
    feasible, the later ones in batches of consecutive levels up to 2e9
    closed-form visits each (small levels share a batch, large ones run alone
    so the search stops at the first feasible one).  The reference's
    first-feasible-level rule is applied afterwards, so the result and the
    stats are identical either way.
    """
    if num_nodes < 1 or devices_per_node < 1 or batch_size < 1:
        raise InvalidArgs("node count, devices per node and batch size must be at least 1")
    opts = options or SearchOptions()
    ctx = _lib.context()
    tm = {} if last_stats is not None else None
    flat = bind_problem(ctx, blocks, tm)
    if not times_nonneg(flat):
        return checked_form_stage(ctx, num_nodes, devices_per_node, batch_size, blocks, opts)
    if flat.has_cost_table:
        from .search import enumerate_calls
        calls, _ = enumerate_calls(num_nodes, devices_per_node, batch_size, len(blocks))
        bind_overrides(ctx, flat, call_shares(calls, batch_size))
    buf = abi.PlanBuffers(max(1, len(blocks)))
    st = abi.PcStats()
    t0 = time.perf_counter()
    rc = ctx.lib.pc_form_stage(ctx.h, num_nodes, devices_per_node, batch_size,
                               int(bool(opts.disable_pruning)), _budget(opts),
                               2 if speculative is None else int(bool(speculative)),
                               C.byref(buf.s), C.byref(st))
    ctx.check(rc, "form_stage")
    if last_stats is not None:
        last_stats.update(tm, library_ms=(time.perf_counter() - t0) * 1e3,
                          kernel_launches=int(st.kernel_launches),
                          visits=int(st.visits), dp_calls=int(st.dp_calls),
                          visits_unpruned=int(st.visits_unpruned), cells=int(st.cells),
                          device_ms=float(st.device_ms), span_ms=float(st.span_ms),
                          post_ms=float(st.post_ms))
    if rc == abi.PC_ERR_BUDGET:
        raise SearchBudgetExceeded(int(st.visits), int(opts.visit_budget))
    stats = SearchStats(visits=int(st.visits), dp_calls=int(st.dp_calls))
    plan = plan_from_buffers(buf, batch_size) if rc == abi.PC_OK else None
    return SearchResult(plan, stats)


def times_nonneg(flat) -> bool:
    """Every task time the search can see is >= 0 (FLOP model with
    non-negative FLOPs, cost-table entries with non-negative times)."""
    if not (flat.flops_per_sec > 0 and flat.bwd_fwd_ratio >= 0):
        return False
    if flat.task_flops.size and not (flat.task_flops >= 0).all():
        return False
    table = getattr(flat.cost_config, "cost_table", None) if flat.has_cost_table else None
    for e in (table or {}).values():
        if not (e.t_fwd >= 0) or (e.t_bwd is not None and not (e.t_bwd >= 0)):
            return False
    return True


def checked_form_stage(ctx, num_nodes: int, devices_per_node: int, batch_size: int, blocks,
                       opts):
    """form_stage (stages.py:372-413) when span times can be negative.  The
    reference ranks every feasible candidate of the first feasible level with
    simulate(), whose validate_plan (stages.py:416-492) recomputes the
    objective without the DP's 0.0 start entry: a plan whose stage times are
    all negative fails it and min() raises InvalidPlan at the first such
    candidate in call order.  Here the levels run in order as device batches
    (every call's plan kept), the visit budget is applied over the level as the
    reference's cells would cross it, and each feasible candidate is validated
    on the device (simulate.validate_plan) in call order before ranking."""
    from .search import enumerate_calls, rank_key, run_calls
    from .simulate import InvalidPlan, validate_plan
    nb = len(blocks)
    calls, levels = enumerate_calls(num_nodes, devices_per_node, batch_size, nb)
    budget = opts.visit_budget
    visits = counted = 0
    lv_all = sorted(set(levels))
    for lv in lv_all:
        idx = [i for i in range(len(calls)) if levels[i] == lv]
        batch = run_calls(ctx, [calls[i] for i in idx], batch_size, opts.disable_pruning, True)
        for j in range(len(idx)):
            v = int(batch.results[j]["visits"])
            counted += 1
            if budget is not None and visits + v > budget:
                from .search import crossing_visits
                raise SearchBudgetExceeded(
                    crossing_visits(ctx, j, calls[idx[j]], visits, int(budget), batch_size,
                                    opts.disable_pruning), int(budget))
            visits += v
        best = None
        for j, i in enumerate(idx):
            plan = batch.plan(j, batch_size)
            if plan is None:
                continue
            bad = validate_plan(plan, blocks)
            if bad:
                raise InvalidPlan(bad)
            key = rank_key(float(batch.results[j]["iteration_time"]), plan.objective,
                           plan.microbatches, i)
            if best is None or key < best[0]:
                best = (key, plan)
        if best is not None:
            return SearchResult(best[1], SearchStats(visits=visits, dp_calls=counted))
    return SearchResult(None, SearchStats(visits=visits, dp_calls=counted))


@_lib.serialized
def brute_force_partition(blocks, S: int, D: int, batch_size: int, replica_factor: int,
                          microbatches: int, options=None, *, guard: bool = True):
    """Exhaustive search over every (cut combination, device composition)
    pair on the GPU (stages.py:304-369): same candidate rules as the DP,
    objective max(t_fwd) + max(t_bwd), ties by (bounds, devices), visits =
    pairs enumerated.  ``guard`` keeps the reference's TooLarge limit
    (nb <= 12, D <= 8); with ``guard=False`` the device enumerates up to 1e12
    pairs (S <= 64)."""
    _check_args(blocks, S, D, batch_size, replica_factor, microbatches)
    nb = len(blocks)
    if guard and (nb > 12 or D > 8):
        raise TooLarge(f"{nb} blocks on {D} devices is past the enumeration guard")
    ctx = _lib.context()
    flat = bind_problem(ctx, blocks)
    bind_overrides(ctx, flat, call_shares([(S, D, replica_factor, microbatches)], batch_size))
    buf = abi.PlanBuffers(S)
    st = abi.PcStats()
    rc = ctx.lib.pc_brute_force(ctx.h, S, D, batch_size, replica_factor, microbatches,
                                C.byref(buf.s), C.byref(st))
    ctx.check(rc, "brute_force_partition")
    stats = SearchStats(visits=int(st.visits), dp_calls=0)
    plan = plan_from_buffers(buf, batch_size) if rc == abi.PC_OK else None
    return SearchResult(plan, stats)
