"""Benchmark: DP cells/s of RaNNC's partition search (form_stage) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1, NCCL)

Workload (config.workload): BASELINE.json configs[4], the C5 DP scaling
sweep -- an enlarged-BERT layer chain (one BERT-1024 layer per block, +-10%
seeded FLOP jitter), nb = 4096 blocks on D = 256 devices (32 nodes x 8),
batch 8*D, every (n, S, MB) call of form_stage evaluated (full enumeration,
456 calls), the plan chosen by the reference's first-feasible-level rule.
The headline is the largest point whose warm-up + timed steps at the
driver's --steps 20 --warmup 5 stay well inside its step limit (~5 s a step);
the line's `sweep` key holds all 16 points once, 4096 x 1024 (~48 s a step)
included.  A step is one complete search.  DP cells/s = the
reference's unpruned SearchStats.visits unit / step time.
Multi-GPU: the calls are sharded (LPT) over the ranks, one NCCL all-gather
of fixed-size records per step: strong scaling.

Every timed step is one call of the public API, form_stage_sharded(), from
the host BlockSet: host flattening, host->device upload, span/cut tables, the
DP, backtrack, simulate, exchange and the result objects.
  e2e   = unpruned visits / wall time of that call (max over ranks)
  value = unpruned visits / its device-resident part (CUDA events on the
          library stream from after the upload to the result; max over ranks)
A 512 MiB L2 flush precedes every step.  At N = 1 the line adds the 16-point
sweep, the C1-C4 latencies with a phase breakdown and the reference's own
C1-C4 times from this run, and a single-core reference sample.

--impl reference: the unmodified reference (baseline/_ref) on all host cores
through its own form_stage_dp (baseline/ref_arm.py; no repo code loaded).
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DEFAULT_NB = 4096
DEFAULT_D = 256
JITTER_SEED = 0
SWEEP_NB = (64, 256, 1024, 4096)
SWEEP_D = (8, 64, 256, 1024)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--nb", type=int, default=DEFAULT_NB)
    ap.add_argument("--D", type=int, default=DEFAULT_D)
    ap.add_argument("--ref-budget", type=int, default=3 * 10 ** 6,
                    help="visits per reference worker per step (deterministic prefix)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-latency", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    return ap.parse_args()


def call_list(nb, D):
    sys.path.insert(0, os.path.join(ROOT, "baseline"))
    from ref_arm import enumerate_calls, unpruned      # no repo package: shared by both arms
    calls = enumerate_calls(max(1, D // 8), min(8, D), 8 * D, nb)
    return calls, sum(unpruned(nb, c) for c in calls)


def workload_config(nb, D):
    calls, unpruned = call_list(nb, D)
    nodes, dpn = max(1, D // 8), min(8, D)
    return {
        "workload": f"C5 enlarged-BERT layer chain: nb={nb} blocks, D={D} devices "
                    f"({nodes}x{dpn}), batch {8 * D}, full (n,S,MB) enumeration of form_stage",
        "nb": nb, "devices": D, "batch": 8 * D, "calls": len(calls),
        "unpruned_visits_per_step": unpruned, "jitter_seed": JITTER_SEED,
        "parallelism": "calls sharded over GPUs (LPT), one NCCL all-gather",
        "l2": "span/cut tables rebuilt each step; 512 MiB L2 flush before every step",
    }


# --------------------------------------------------------------------------- clocks
class Clocks:
    def __init__(self, index):
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}_{index}.csv")
        self.index = index

    QUERY = ["--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
             "--format=csv,noheader,nounits"]

    def __enter__(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", *self.QUERY, "-lms", "200"],
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
            if os.path.getsize(self.path) == 0:
                # a region shorter than the sampling period: one sample at its end
                try:
                    with open(self.path, "w") as fh:
                        subprocess.run(["nvidia-smi", f"--id={self.index}", *self.QUERY],
                                       stdout=fh, stderr=subprocess.DEVNULL, timeout=30)
                except Exception:
                    pass

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


# --------------------------------------------------------------------------- reference arm
def run_reference_arm(a):
    """The unmodified reference on all host cores (rank 0 only; baseline/ref_arm.py)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "baseline"))
    import ref_arm
    cores = os.cpu_count() or 1
    pool = ref_arm.make_pool(a.nb, a.D, cores, JITTER_SEED)
    vals, last = [], None
    for i in range(a.warmup + a.steps):
        last = ref_arm.sample(a.nb, a.D, cores, a.ref_budget, JITTER_SEED, pool)
        if i >= a.warmup:
            vals.append(last["value"])
    pool.close()
    pool.join()
    value = sorted(vals)[len(vals) // 2]
    sample = (f"{cores} processes x one call of the workload each (calls spread over the "
              f"enumeration), the reference's pipecut.form_stage_dp with pruning off, stopped "
              f"by its own visit-budget check after exactly {a.ref_budget} visits (a "
              f"deterministic prefix: the same work every step); value = total visits / "
              f"slowest worker, median over steps. Prefixes lie in level 1 where a cell "
              f"costs O(1) but counts up to b*d visits: favours the reference")
    line = {
        "impl": "reference", "metric": "dp_cells_per_sec", "value": value,
        "unit": "visits/s", "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": last["seconds"] * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(a.nb, a.D),
        "cpu_baseline": {"value": value, "unit": "visits/s", "cores": cores,
                         "kind": "reference", "sample": sample, "calls": last["calls"],
                         "per_step": vals},
        "e2e": {"value": value, "unit": "visits/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def ref_subprocess(*args, timeout=900):
    """Run baseline/ref_arm.py in a fresh interpreter (no repo code loaded)."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "baseline", "ref_arm.py"), *args],
                         capture_output=True, text=True, timeout=timeout)
    if out.returncode != 0:
        return {"error": out.stderr.strip().splitlines()[-1:] or ["failed"]}
    return json.loads(out.stdout.strip().splitlines()[-1])


# --------------------------------------------------------------------------- GPU arm
class Arm:
    """One process per GPU: the library context, the L2 flush buffer and the
    max-over-ranks helpers."""

    def __init__(self):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(self.local)
        if self.world > 1:
            os.environ.setdefault("NCCL_DEBUG", "WARN")   # stdout carries only the JSON line
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
        self.dev = torch.device("cuda", self.local)
        from paper_2103_16063_b200 import _lib
        self.ctx = _lib.context(self.local)
        self.flush_buf = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=self.dev)

    def barrier(self):
        self.torch.cuda.synchronize()
        if self.world > 1:
            self.dist.barrier()

    def max_over_ranks(self, xs):
        if self.world == 1:
            return list(xs)
        t = self.torch.tensor(list(xs), dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return t.cpu().tolist()

    def fresh(self):
        """Forget the bound problem and the span tables: the next call flattens,
        uploads and rebuilds everything."""
        self.ctx.problem_owner = None
        self.ctx.check(self.ctx.lib.pc_reset_cache(self.ctx.h), "reset")
        self.flush_buf.zero_()

    def step(self, nodes, dpn, BS, bs, **kw):
        """One public-API search; returns (result, timings, e2e_ms, resident_ms),
        times max over ranks."""
        from paper_2103_16063_b200.search import form_stage_sharded
        self.fresh()
        self.barrier()
        tim = {}
        t0 = time.perf_counter()
        res = form_stage_sharded(nodes, dpn, BS, bs, timings=tim, **kw)
        self.torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        e2e_ms, res_ms = self.max_over_ranks([wall, tim.get("resident_ms", wall)])
        return res, tim, e2e_ms, res_ms


PHASES = ("flatten_ms", "upload_ms", "weights_ms", "span_ms", "dp_ms", "post_ms",
          "run_calls_ms", "pack_ms", "exchange_ms", "decide_ms")


def _dp_sha():
    import hashlib
    src = os.path.join(ROOT, "paper_2103_16063_b200", "csrc", "dp.cu")
    return hashlib.sha256(open(src, "rb").read()).hexdigest()[:16]


def roofline(nb, D, world, calls_local, tims, dadd_peak, mix_peak, steps, sm_count, sm_mhz):
    """Dominant kernel k_dp_level.  It is issue-bound on integer / control
    bookkeeping (ncu: no HBM or fp64-pipe roof comes close), so the roof is the
    warp-instruction issue rate: 4 schedulers x SMs x 1 instruction per clock
    at the measured SM clock; achieved = the kernel's warp instructions per
    step (ncu count of this workload, profiles/dp_level_profile.json, tied to
    the dp.cu source by hash) over its live per-step time (CUDA events).  The
    SURVEY 8(d) algorithmic fp64 basis is kept beside it; with exact pruning
    (dominance, objective bound) the kernel skips most of that work, so that
    ratio exceeds 1 and is not a roofline fraction."""
    from paper_2103_16063_b200.workloads import unpruned_visits
    pairs = sum(t["pairs"] for t in tims)
    cands = sum(t["candidates"] for t in tims)
    dp_ms = sum(t["dp_ms"] for t in tims)
    launches = sum(t["dp_launches"] for t in tims)
    f_bar = cands / pairs if pairs else 0.0
    ops = unpruned_visits(nb, calls_local) * steps * (2.0 + 4.0 * f_bar)
    algo = ops / (dp_ms / 1e3) / 1e9 if dp_ms > 0 else 0.0
    ops_exec = 2.0 * pairs + 4.0 * cands
    exec_rate = ops_exec / (dp_ms / 1e3) / 1e9 if dp_ms > 0 else 0.0
    issue_peak = 4.0 * sm_count * sm_mhz * 1e6 / 1e9
    out = {"bound": "issue", "achieved": None, "peak": issue_peak, "unit": "Ginst/s",
           "frac": None, "traffic": None, "kernel": "k_dp_level",
           "avg_launch_ms": dp_ms / max(1, launches), "launches_per_step": launches / max(1, steps),
           "dp_ms_per_step": dp_ms / steps,
           "basis": "k_dp_level warp instructions per step (ncu smsp__inst_executed.sum of this "
                    "workload, profiles/dp_level_profile.json) / its live per-step time; peak = "
                    f"4 x {sm_count} SMs x 1 warp-inst/clk at {sm_mhz:.0f} MHz",
           "fp64_algorithmic": {
               "achieved": algo, "unit": "Gop/s", "dadd_peak": dadd_peak, "mix_peak": mix_peak,
               "ratio_to_dadd_peak": algo / dadd_peak if dadd_peak else None,
               "ops_per_step": ops / steps, "f_bar": f_bar,
               "basis": "SURVEY 8(d): (2 + 4*F_bar) fp64 ops per unpruned visit of this rank's "
                        "calls over its k_dp_level time; > 1 means the exact pruning skips that "
                        "much of the algorithmic work (not a roofline fraction)",
               "executed": {"achieved": exec_rate, "frac_of_dadd_peak":
                            exec_rate / dadd_peak if dadd_peak else None,
                            "ops_per_step": ops_exec / steps}},
           "peak_source": "SM count from the device, clock = median SM clock sampled under load"}
    prof = os.path.join(ROOT, "profiles", "dp_level_profile.json")
    try:
        p = json.load(open(prof))
    except Exception:
        p = None
    if p and p.get("workload") == {"nb": nb, "D": D, "n_gpus": world} and \
            p.get("dp_cu_sha") == _dp_sha() and dp_ms > 0:
        inst = p["warp_inst_per_step"]
        out["achieved"] = inst / (dp_ms / steps / 1e3) / 1e9
        out["frac"] = out["achieved"] / issue_peak
        out["traffic"] = p.get("dram_bytes_per_launch")
        out["ncu"] = {k: p.get(k) for k in ("warp_inst_per_step", "fp64_pipe_inst_per_step",
                                             "active_threads_per_warp", "dram_bytes_per_step",
                                             "launches", "source")}
    else:
        out["note"] = ("no ncu instruction count for this workload and kernel source "
                       "(profiles/dp_level_profile.json): achieved/frac not computed")
    return out


def run_ours(a):
    arm = Arm()
    import ctypes as C
    from paper_2103_16063_b200.search import enumerate_calls, lpt_shard, shard_weights
    from paper_2103_16063_b200.stages import bind_problem
    from paper_2103_16063_b200.workloads import c5_blockset, unpruned_visits

    ctx, world, rank = arm.ctx, arm.world, arm.rank
    nodes, dpn = max(1, a.D // 8), min(8, a.D)
    BS = 8 * a.D
    bs = c5_blockset(a.nb, a.D, jitter_seed=JITTER_SEED)
    nb = len(bs)
    calls, _ = enumerate_calls(nodes, dpn, BS, nb)
    unpruned = unpruned_visits(nb, calls)
    bind_problem(ctx, bs)
    owner = lpt_shard(nb, calls, world, shard_weights(ctx, calls, BS, nb) if world > 1 else None)
    my_calls = [calls[i] for i in range(len(calls)) if owner[i] == rank]
    smc, ccmaj, ccmin = C.c_int32(), C.c_int32(), C.c_int32()
    ctx.check(ctx.lib.pc_device_info(ctx.h, C.byref(smc), C.byref(ccmaj), C.byref(ccmin)), "info")
    dadd, mix = C.c_double(), C.c_double()
    ctx.check(ctx.lib.pc_measure_dadd_peak(ctx.h, C.byref(dadd)), "peak")
    ctx.check(ctx.lib.pc_measure_fp64_peak(ctx.h, C.byref(mix)), "peak")

    # ---- headline: warm-up, then K timed public-API steps
    result = None
    for _ in range(a.warmup):
        result = arm.step(nodes, dpn, BS, bs)[0]
    e2e, resident, tims = [], [], []
    with Clocks(arm.local) as clk:
        for _ in range(a.steps):
            res, tim, e_ms, r_ms = arm.step(nodes, dpn, BS, bs)
            e2e.append(e_ms)
            resident.append(r_ms)
            tims.append(tim)
            if result is not None:
                assert res.plan == result.plan and res.stats == result.stats
            result = res
    ms_per_step = sum(resident) / len(resident)
    e2e_ms = sum(e2e) / len(e2e)
    phases = {k: sum(t.get(k, 0.0) for t in tims) / len(tims) for k in PHASES}
    clk_sum = clk.summary() or {}
    rl = roofline(nb, a.D, world, my_calls, tims, dadd.value, mix.value, a.steps, smc.value,
                  clk_sum.get("sm_mhz") or 1965.0)
    # schedule (i): widening levels in order, stop at the first
    # feasible one -- the reference's own order, same answer
    lvl = []
    for i in range(6):
        arm.fresh()
        arm.barrier()
        t0 = time.perf_counter()
        from paper_2103_16063_b200.search import form_stage_sharded
        r_l = form_stage_sharded(nodes, dpn, BS, bs, speculative=False)
        arm.torch.cuda.synchronize()
        if i:
            lvl.append(arm.max_over_ranks([(time.perf_counter() - t0) * 1e3])[0])
        assert r_l.plan == result.plan and r_l.stats == result.stats
    plan_bytes = 0 if result.plan is None else 48 * len(result.plan.stages)

    line = None
    if rank == 0:
        line = {
            "metric": "dp_cells_per_sec", "value": unpruned / (ms_per_step / 1e3),
            "unit": "visits/s", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(nb, a.D),
            "e2e": {"value": unpruned / (e2e_ms / 1e3), "unit": "visits/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": int(tims[-1].get("h2d_bytes", 0)),
                    "d2h_bytes_per_step": int(tims[-1].get("d2h_bytes", 0)) + plan_bytes,
                    "note": "same timed steps: wall time of the public form_stage_sharded() "
                            "call from the host BlockSet (flatten, upload, search, result "
                            "objects), max over ranks"},
            "gpu_launches": int(tims[-1].get("kernel_launches", 0)),
            "breakdown_ms": dict(phases, resident=ms_per_step, e2e=e2e_ms,
                                 note="rank 0 means over the timed steps; span/dp/post are "
                                      "device (CUDA events): K1/K2 tables, K3 level kernels, "
                                      "then K7 visits + K4 backtrack + stage records + K5 "
                                      "simulate + D2H; run_calls is their host wall time"),
            "schedules_ms": {"speculative": e2e_ms,
                             "level_by_level": sorted(lvl)[len(lvl) // 2],
                             "note": "public API, answer-equal; level by level stops at the "
                                     "first feasible widening level (the reference's order), "
                                     "the metric counts the full enumeration"},
            "roofline": rl,
            "plan": None if result.plan is None else {
                "stages": len(result.plan.stages), "microbatches": result.plan.microbatches,
                "replica_factor": result.plan.replica_factor,
                "objective": result.plan.objective.hex(), "visits": result.stats.visits,
                "dp_calls": result.stats.dp_calls},
            "clocks": clk.summary(),
        }
    if world == 1:
        if not a.no_sweep:
            line["sweep"] = sweep(arm, dadd.value, (a.nb, a.D), line)
        if not a.no_latency:
            line["latency_ms"] = config_latencies(arm)
        if not a.no_cpu_baseline:
            ref = ref_subprocess("sample", "--nb", str(a.nb), "--D", str(a.D), "--cores", "1",
                                 "--budget", str(a.ref_budget), "--seed", str(JITTER_SEED))
            line["cpu_baseline"] = {
                "value": ref.get("value"), "unit": "visits/s", "cores": 1, "kind": "reference",
                "sample": f"reference pipecut.form_stage_dp (baseline/_ref, unmodified, "
                          f"baseline/ref_arm.py in a fresh interpreter) on one call "
                          f"{ref.get('calls')} of the workload with pruning off, stopped by "
                          f"its own visit-budget check after exactly {a.ref_budget} visits; "
                          f"single thread; level-1 prefix, favours the reference",
                "seconds": ref.get("seconds")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        arm.dist.barrier()
        arm.dist.destroy_process_group()


def sweep(arm, dadd_peak, headline, line):
    """BASELINE configs[4]: every (nb, D) point once at N = 1 through the
    public API (one warm-up -- none at 4096 x 1024 -- and one timed step; the
    headline point reuses the headline's timed steps)."""
    from paper_2103_16063_b200.search import enumerate_calls
    from paper_2103_16063_b200.workloads import c5_blockset, unpruned_visits
    out = []
    for nb in SWEEP_NB:
        for D in SWEEP_D:
            if (nb, D) == headline:
                out.append({"nb": nb, "D": D, "steps": line["steps"], "from": "headline",
                            "visits_per_sec": line["value"], "e2e_visits_per_sec": line["e2e"]["value"],
                            "ms": line["ms_per_step"], "dp_ms": line["breakdown_ms"]["dp_ms"],
                            "roofline_frac": line["roofline"]["frac"],
                            "fp64_algorithmic_ratio":
                                line["roofline"]["fp64_algorithmic"]["ratio_to_dadd_peak"],
                            "clocks": line["clocks"]})
                continue
            nodes, dpn = max(1, D // 8), min(8, D)
            bs = c5_blockset(nb, D, jitter_seed=JITTER_SEED)
            calls, _ = enumerate_calls(nodes, dpn, 8 * D, nb)
            unpruned = unpruned_visits(nb, calls)
            big = unpruned > 10 ** 13        # 4096 x 1024: one untimed pass would add ~50 s
            if not big:
                arm.step(nodes, dpn, 8 * D, bs)
            with Clocks(arm.local) as clk:
                res, tim, e_ms, r_ms = arm.step(nodes, dpn, 8 * D, bs)
            rl = roofline(nb, D, 1, calls, [tim], dadd_peak, 0.0, 1, 148, 1965.0)
            out.append({"nb": nb, "D": D, "steps": 1, "warmup": 0 if big else 1,
                        "calls": len(calls),
                        "unpruned_visits": unpruned,
                        "visits_per_sec": unpruned / (r_ms / 1e3),
                        "e2e_visits_per_sec": unpruned / (e_ms / 1e3), "ms": r_ms,
                        "dp_ms": tim["dp_ms"],
                        "fp64_algorithmic_ratio": rl["fp64_algorithmic"]["ratio_to_dadd_peak"],
                        "f_bar": rl["fp64_algorithmic"]["f_bar"],
                        "objective": None if res.plan is None else res.plan.objective.hex(),
                        "clocks": clk.summary()})
    return out


def config_latencies(arm):
    """Reference-semantics partition search on C1-C4 through the public API:
    partition_blocks + form_stage, median of 10 warm runs + 1 cold, with the
    phase split, beside the reference's own times measured in this run
    (baseline/ref_arm.py configs, one process per config)."""
    from paper_2103_16063_b200 import flatten as _flat
    from paper_2103_16063_b200 import form_stage, partition_blocks
    from paper_2103_16063_b200.workloads import config_partition
    ctx = arm.ctx
    ref = ref_subprocess("configs", timeout=1200)
    out = {}
    for name in ("C1", "C2", "C3", "C4"):
        part, model, k, batch, cl = config_partition(name)
        tb, ts, pb_t, fs_t = [], [], [], []
        for i in range(11):
            _flat._ATOM_CACHE.clear()
            ctx.problem_owner = None
            ctx.lib.pc_reset_cache(ctx.h)
            gc.collect()
            t_pb, t_fs = {}, {}
            t0 = time.perf_counter()
            bs = partition_blocks(part, model, k, timings=t_pb)
            t1 = time.perf_counter()
            res = form_stage(cl.num_nodes, cl.devices_per_node, batch, bs, last_stats=t_fs)
            t2 = time.perf_counter()
            tb.append((t1 - t0) * 1e3)
            ts.append((t2 - t1) * 1e3)
            pb_t.append(t_pb)
            fs_t.append(t_fs)
        med = lambda v: sorted(v[1:])[len(v[1:]) // 2]
        mean = lambda ds, k: sum(d.get(k, 0.0) for d in ds[1:]) / len(ds[1:])
        r = ref.get(name, {}) if isinstance(ref, dict) else {}
        entry = {"partition_blocks_ms": med(tb), "form_stage_ms": med(ts),
                 "total_ms": med([x + y for x, y in zip(tb, ts)]),
                 "cold_total_ms": tb[0] + ts[0],
                 "phases_ms": {
                     "partition_blocks": {k: mean(pb_t, k) for k in
                                          ("flatten_ms", "library_ms", "build_ms")},
                     "form_stage": {k: mean(fs_t, k) for k in
                                    ("flatten_ms", "upload_ms", "library_ms", "span_ms",
                                     "device_ms", "post_ms")}},
                 "visits": res.stats.visits, "dp_calls": res.stats.dp_calls,
                 "objective": None if res.plan is None else res.plan.objective.hex()}
        if r:
            entry["ref_ms"] = {k: r[k] for k in ("partition_blocks_ms", "form_stage_ms",
                                                 "total_ms")}
            entry["ref_same_answer"] = (r["objective"] == entry["objective"]
                                        and r["visits"] == entry["visits"]
                                        and r["dp_calls"] == entry["dp_calls"])
            entry["speedup"] = r["total_ms"] / entry["total_ms"]
        elif isinstance(ref, dict) and "error" in ref:
            entry["ref_ms"] = {"error": ref["error"]}
        out[name] = entry
    out["note"] = ("phases: partition_blocks = host atom flattening / library (device "
                   "coarsening + refinement + block profiles) / reference objects; form_stage "
                   "= flatten / upload / pc_form_stage wall (span, device = DP levels, post = "
                   "visits + backtrack + records + simulate, all CUDA events); ref_ms: the "
                   "unmodified reference in this run, one process per config")
    return out


if __name__ == "__main__":
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)
