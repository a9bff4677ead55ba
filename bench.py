"""Benchmark: DP cells/s of RaNNC's partition search (form_stage) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1, NCCL)

Workload (config.workload): the C5 DP scaling sweep point of BASELINE.json
configs[4] -- an enlarged-BERT layer chain (one BERT-1024 layer per block,
+-10% seeded FLOP jitter), nb blocks on D devices (D/8 nodes x 8), batch 8*D,
every (n, S, MB) call of form_stage evaluated (full enumeration), the plan
chosen by the reference's first-feasible-level rule.  A step is one complete
search.  DP cells/s = the reference's unpruned SearchStats.visits unit
 / step time.  Multi-GPU: the calls are sharded (LPT) over the
ranks, one NCCL all-gather of fixed-size records per step: strong scaling.

value: problem resident on the device, span/cut tables rebuilt every step.
e2e:   the public API form_stage_sharded() per step, including host
       flattening, host->device upload of the problem and device->host results.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DEFAULT_NB = 1024
DEFAULT_D = 256
JITTER_SEED = 0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--nb", type=int, default=DEFAULT_NB)
    ap.add_argument("--D", type=int, default=DEFAULT_D)
    ap.add_argument("--cpu-sample-sec", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-latency", action="store_true")
    return ap.parse_args()


def workload_config(nb, D, calls, unpruned):
    nodes, dpn = max(1, D // 8), min(8, D)
    return {
        "workload": f"C5 enlarged-BERT layer chain: nb={nb} blocks, D={D} devices "
                    f"({nodes}x{dpn}), batch {8 * D}, full (n,S,MB) enumeration of form_stage",
        "nb": nb, "devices": D, "batch": 8 * D, "calls": len(calls),
        "unpruned_visits_per_step": unpruned, "jitter_seed": JITTER_SEED,
        "parallelism": "calls sharded over GPUs (LPT), one NCCL all-gather",
        "l2": "span/cut tables rebuilt each step (> L2); 512 MiB L2 flush between steps",
    }


# --------------------------------------------------------------------------- clocks
class Clocks:
    def __init__(self, index):
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")
        self.index = index

    def __enter__(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        try:
            rows = [l.split(",") for l in open(self.path) if l.strip()]
        except Exception:
            return None
        if not rows:
            return None
        sm = sorted(float(r[0]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4)
                          if len(r) > 4 + i and r[3 + i].strip() == "Active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(rows[0][1]),
                "reasons": reasons, "samples": len(rows)}


# --------------------------------------------------------------------------- CPU legs
def _ref_worker_init(nb, D):
    global _REF_BS
    from paper_2103_16063_b200.workloads import c5_blockset
    _REF_BS = c5_blockset(nb, D, jitter_seed=JITTER_SEED)


class _Deadline:
    """SearchOptions-compatible options for the unmodified reference: pruning
    off (the metric's unit) or on (its stock default), and `visit_budget` None
    until the deadline, then -1 -- the reference's own per-cell check
    (stages.py:214-216) then raises SearchBudgetExceeded carrying the exact
    visit count reached."""

    def __init__(self, seconds, disable_pruning=True):
        self._end = time.perf_counter() + seconds
        self.disable_pruning = disable_pruning

    @property
    def visit_budget(self):
        return None if time.perf_counter() < self._end else -1


def _ref_run(args):
    """The reference's own form_stage_dp on one call of the workload for about
    `seconds` of wall time; returns (visits, seconds)."""
    import pipecut
    (S, D, R, MB), bs_batch, seconds = args[:3]
    unpruned = args[3] if len(args) > 3 else True
    t0 = time.perf_counter()
    try:
        res = pipecut.form_stage_dp(_REF_BS, S, D, bs_batch, R, MB, _Deadline(seconds, unpruned))
        visits = res.stats.visits
    except pipecut.SearchBudgetExceeded as exc:
        visits = exc.visits
    return visits, time.perf_counter() - t0


def sample_calls(calls, k):
    step = max(1, len(calls) // k)
    return [calls[(i * step) % len(calls)] for i in range(k)]


class RefSampler:
    """Reference visits/s on `cores` host processes, each running one call of
    the workload (calls spread over the enumeration) for `seconds`."""

    def __init__(self, nb, D, calls, seconds, cores, unpruned=True):
        import multiprocessing as mp
        self.cores = cores
        self.calls = sample_calls(calls, cores)
        self.work = [(c, 8 * D, seconds, unpruned) for c in self.calls]
        if cores == 1:
            _ref_worker_init(nb, D)
            self.pool = None
        else:
            self.pool = mp.get_context("fork").Pool(cores, initializer=_ref_worker_init,
                                                    initargs=(nb, D))

    def rate(self):
        out = self.pool.map(_ref_run, self.work) if self.pool else [_ref_run(w) for w in self.work]
        return sum(o[0] for o in out) / max(o[1] for o in out)

    def close(self):
        if self.pool:
            self.pool.close()
            self.pool.join()


def run_reference_arm(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2103_16063_b200._host import pipecut  # noqa: F401  (baseline/_ref)
    from paper_2103_16063_b200.search import enumerate_calls
    from paper_2103_16063_b200.workloads import unpruned_visits
    nodes, dpn = max(1, a.D // 8), min(8, a.D)
    calls, _ = enumerate_calls(nodes, dpn, 8 * a.D, a.nb)
    cores = os.cpu_count() or 1
    per_step = max(2.0, min(a.cpu_sample_sec, 120.0 / max(1, a.steps + a.warmup)))
    sampler = RefSampler(a.nb, a.D, calls, per_step, cores)
    rates = []
    for i in range(a.warmup + a.steps):
        r = sampler.rate()
        if i >= a.warmup:
            rates.append(r)
    sampler.close()
    value = sorted(rates)[len(rates) // 2]
    stock_sampler = RefSampler(a.nb, a.D, calls, per_step, cores, unpruned=False)
    stock = stock_sampler.rate()
    stock_sampler.close()
    sample = (f"{cores} processes x one call of the workload each (calls spread over the "
              f"enumeration), the reference's pipecut.form_stage_dp with pruning off, each "
              f"stopped after ~{per_step:.0f} s by its own visit-budget check; "
              f"value = total visits / slowest worker")
    line = {
        "impl": "reference", "metric": "dp_cells_per_sec", "value": value,
        "unit": "visits/s", "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": None, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(a.nb, a.D, calls, unpruned_visits(a.nb, calls)),
        "cpu_baseline": {"value": value, "unit": "visits/s", "cores": cores,
                         "kind": "reference", "sample": sample,
                         "stock_path": {"pruned_visits_per_sec": stock,
                                        "note": "same workers, the reference's default options "
                                                "(pruning on); rate in its own pruned visits. "
                                                "Bounded samples start at level 1 (O(1) per cell, "
                                                "up to b*d visits), which favours the reference"}},
        "e2e": {"value": value, "unit": "visits/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU arm
def run_ours(a):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    from paper_2103_16063_b200 import _lib
    from paper_2103_16063_b200.search import (device_weights, _pack, decide, enumerate_calls,
                                              exchange, form_stage_sharded, lpt_shard,
                                              run_calls)
    from paper_2103_16063_b200.stages import bind_problem
    from paper_2103_16063_b200.workloads import c5_blockset, unpruned_visits
    import ctypes as C

    ctx = _lib.context(local)
    nodes, dpn = max(1, a.D // 8), min(8, a.D)
    BS = 8 * a.D
    bs = c5_blockset(a.nb, a.D, jitter_seed=JITTER_SEED)
    nb = len(bs)
    calls, levels = enumerate_calls(nodes, dpn, BS, nb)
    unpruned = unpruned_visits(nb, calls)
    bind_problem(ctx, bs)
    owner = lpt_shard(nb, calls, world, device_weights(ctx, calls, BS) if world > 1 else None)
    local_idx = [i for i in range(len(calls)) if owner[i] == rank]
    my_calls = [calls[i] for i in local_idx]
    n_levels = max(levels) + 1
    max_stages = max(c[0] for c in calls)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timer():
        ctx.check(ctx.lib.pc_timer_start(ctx.h), "timer")

    def stop():
        ms = C.c_double()
        ctx.check(ctx.lib.pc_timer_stop(ctx.h, C.byref(ms)), "timer")
        return ms.value

    # ---- device-resident step: span tables + DP + backtrack + simulate + exchange + select
    bind_problem(ctx, bs)
    last = {}

    def step_resident():
        ctx.check(ctx.lib.pc_reset_cache(ctx.h), "reset")
        flush.zero_()
        barrier()
        timer()
        batch = run_calls(ctx, my_calls, BS, False, True)
        rec, plan_w = _pack(nb, calls, levels, owner, rank, batch, local_idx, n_levels, max_stages)
        allrec = exchange(rec, None, dev)
        out = decide(allrec, calls, levels, owner, plan_w, None, BS)
        ms = stop()
        last.update(stats=batch.stats, result=out[1], stats_visits=batch.results["visits"].copy(),
                    own_ms=ms)
        return max_over_ranks(ms)

    for _ in range(a.warmup):
        step_resident()
    times = []
    pairs = cands = dp_ms = span_ms = launches = dp_launches = 0
    own_ms = 0.0
    with Clocks(local) as clk:
        for _ in range(a.steps):
            times.append(step_resident())
            own_ms += last["own_ms"]
            st = last["stats"]
            pairs += st.pairs
            cands += st.candidates
            dp_ms += st.device_ms
            span_ms += st.span_ms
            launches += st.kernel_launches
            dp_launches += st.dp_launches
    ms_per_step = sum(times) / len(times)
    if os.environ.get("PIPECUT_BENCH_VERBOSE"):
        print(f"[rank {rank}] own step ms {own_ms / a.steps:.1f}, max-over-ranks {ms_per_step:.1f}, "
              f"dp {dp_ms / a.steps:.1f}, span {span_ms / a.steps:.1f}, calls {len(my_calls)}",
              file=sys.stderr, flush=True)
    value = unpruned / (ms_per_step / 1e3)
    result = last["result"]

    # ---- e2e: public API from host objects every step
    e2e_times = []
    tim = {}
    for i in range(a.warmup + a.steps):
        ctx.problem_owner = None            # force flatten + H2D upload
        ctx.check(ctx.lib.pc_reset_cache(ctx.h), "reset")
        flush.zero_()
        barrier()
        timer()
        res = form_stage_sharded(nodes, dpn, BS, bs, timings=tim)
        ms = stop()
        if i >= a.warmup:
            e2e_times.append(max_over_ranks(ms))
        assert res.plan == result.plan and res.stats == result.stats
    e2e_ms = sum(e2e_times) / len(e2e_times)
    # schedule (i): widening levels in order, stop at the first
    # feasible level -- the time to the same answer under the reference's order
    lvl_times = []
    for i in range(a.warmup + a.steps):
        ctx.problem_owner = None
        ctx.check(ctx.lib.pc_reset_cache(ctx.h), "reset")
        flush.zero_()
        barrier()
        timer()
        res_l = form_stage_sharded(nodes, dpn, BS, bs, speculative=False)
        ms = stop()
        if i >= a.warmup:
            lvl_times.append(max_over_ranks(ms))
        assert res_l.plan == result.plan and res_l.stats == result.stats
    lvl_ms = sum(lvl_times) / len(lvl_times)
    plan_bytes = 0 if result.plan is None else 48 * len(result.plan.stages)

    # ---- roofline of the dominant kernel (DP level kernel)
    peak = C.c_double()
    ctx.check(ctx.lib.pc_measure_fp64_peak(ctx.h, C.byref(peak)), "peak")
    # Algorithmic fp64 work per SURVEY §8(d): 2 + 4*F ops per visit (2 comm
    # adds, stages.py:232-237, then per predecessor frontier entry 2 max,
    # stages.py:239, and 2 compares, _pareto) over the step's unpruned visits;
    # F = mean predecessor frontier size over the feasible pairs (cands/pairs).
    f_bar = cands / pairs if pairs else 0.0
    # per GPU: this rank's calls over this rank's DP time (rank 0 reports)
    local_unpruned = unpruned_visits(nb, my_calls)
    ops = local_unpruned * a.steps * (2.0 + 4.0 * f_bar)
    achieved = ops / (dp_ms / 1e3) / 1e9 if dp_ms > 0 else 0.0
    # what the kernel executes after its exact pruning (corner, window, prefix skip)
    ops_exec = 2.0 * pairs + 4.0 * cands
    achieved_exec = ops_exec / (dp_ms / 1e3) / 1e9 if dp_ms > 0 else 0.0
    traffic = None
    prof = os.path.join(ROOT, "profiles", "dp_level_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    line = {
        "metric": "dp_cells_per_sec", "value": value, "unit": "visits/s",
        "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": workload_config(nb, a.D, calls, unpruned),
        "e2e": {"value": unpruned / (e2e_ms / 1e3), "unit": "visits/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": int(tim.get("h2d_bytes", 0)),
                "d2h_bytes_per_step": int(tim.get("d2h_bytes", 0)) + plan_bytes},
        "gpu_launches": int(launches // max(1, a.steps)),
        "schedules_ms": {"speculative": e2e_ms, "level_by_level": lvl_ms,
                         "note": "public API, answer-equal; level by level stops at the first "
                                 "feasible widening level (the reference's order), the "
                                 "metric counts the full enumeration"},
        "breakdown_ms": {"dp_levels": dp_ms / a.steps, "span_tables": span_ms / a.steps,
                         "rest": ms_per_step - (dp_ms + span_ms) / a.steps},
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak.value,
                     "unit": "Gop/s", "frac": achieved / peak.value if peak.value else None,
                     "traffic": traffic,
                     "kernel": "k_dp_level", "avg_launch_ms": dp_ms / max(1, dp_launches),
                     "ops_per_step": ops / a.steps, "f_bar": f_bar,
                     "scope": "rank 0: its own calls' unpruned visits over its own DP time",
                     "basis": "SURVEY 8(d): (2 + 4*F_bar) fp64 ops per unpruned visit",
                     "executed": {"achieved": achieved_exec,
                                  "frac": achieved_exec / peak.value if peak.value else None,
                                  "ops_per_step": ops_exec / a.steps,
                                  "note": "ops the kernel actually runs after exact pruning; "
                                          "ncu: issue-bound on frontier bookkeeping"},
                     "peak_source": "measured on this GPU: pc_measure_fp64_peak "
                                    "(DADD+DSETP.MAX+DSETP chains, full occupancy)"},
        "plan": None if result.plan is None else {
            "stages": len(result.plan.stages), "microbatches": result.plan.microbatches,
            "replica_factor": result.plan.replica_factor, "objective": result.plan.objective,
            "visits": result.stats.visits, "dp_calls": result.stats.dp_calls},
        "clocks": clk.summary(),
    }
    if world == 1 and not a.no_cpu_baseline:
        sampler = RefSampler(nb, a.D, calls, a.cpu_sample_sec, 1)
        rate = sampler.rate()
        # the reference's stock path (pruning on, its default) on the same call:
        # its own pruned visits/s, and the time-to-solution equivalent in the
        # metric's unit via this workload's exact unpruned/pruned ratio (the
        # pruned count per call is the reference's, reproduced bit-exactly)
        stock = RefSampler(nb, a.D, calls, a.cpu_sample_sec / 2, 1, unpruned=False).rate()
        pruned_total = int(np.asarray(last["stats_visits"]).sum())
        ratio = unpruned / pruned_total if pruned_total else None
        line["cpu_baseline"] = {
            "value": rate, "unit": "visits/s", "cores": 1, "kind": "reference",
            "sample": f"reference pipecut.form_stage_dp (baseline/_ref, unmodified) on one call "
                      f"{sampler.calls[0]} of the workload with pruning off, stopped after "
                      f"~{a.cpu_sample_sec:.0f} s by its own visit-budget check; single thread",
            "stock_path": {
                "pruned_visits_per_sec": stock, "unpruned_per_pruned": ratio,
                "equivalent_visits_per_sec": stock * ratio if ratio else None,
                "note": "reference default options (pruning on), same call, "
                        f"~{a.cpu_sample_sec / 2:.0f} s; equivalent = pruned rate x the "
                        "workload's unpruned/pruned visit ratio. Bounded samples start at "
                        "level 1, where a cell costs O(1) but counts up to b*d visits, so "
                        "sampled CPU rates favour the reference"}}
    if not a.no_latency and world == 1:
        line["latency_ms"] = config_latencies(ctx)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def config_latencies(ctx):
    """Reference-semantics partition search on C1-C4 through the public API:
    partition_blocks + form_stage (median of 5 warm runs + 1 cold), beside the
    headline; the reference's own times for the same calls are in
    tests/golden/configs.json (ref_seconds, measured in the build container)."""
    from paper_2103_16063_b200 import form_stage, partition_blocks
    from paper_2103_16063_b200 import flatten as _flat
    from paper_2103_16063_b200.workloads import config_partition
    out = {}
    for name in ("C1", "C2", "C3", "C4"):
        part, model, k, batch, cl = config_partition(name)
        tb, ts = [], []
        for i in range(6):
            _flat._ATOM_CACHE.clear()
            ctx.problem_owner = None
            ctx.lib.pc_reset_cache(ctx.h)
            gc.collect()          # the CPU-baseline sampler leaves large garbage behind
            t0 = time.perf_counter()
            bs = partition_blocks(part, model, k)
            t1 = time.perf_counter()
            res = form_stage(cl.num_nodes, cl.devices_per_node, batch, bs)
            t2 = time.perf_counter()
            tb.append((t1 - t0) * 1e3)
            ts.append((t2 - t1) * 1e3)
        med = lambda v: sorted(v[1:])[len(v[1:]) // 2]
        out[name] = {"partition_blocks_ms": med(tb), "form_stage_ms": med(ts),
                     "total_ms": med([a + b for a, b in zip(tb, ts)]),
                     "cold_total_ms": tb[0] + ts[0],
                     "visits": res.stats.visits, "dp_calls": res.stats.dp_calls,
                     "objective": None if res.plan is None else res.plan.objective}
    return out


if __name__ == "__main__":
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)
