"""The reference arm: the unmodified reference (`pipecut` installed in
baseline/_ref) timed on the host cores, through its own public API.

Nothing here imports the repo's package (paper_2103_16063_b200) or loads its
native libraries: the workloads are rebuilt from the reference's own
generators and host IR, mirroring paper_2103_16063_b200/workloads.py
(tests/test_ref_arm.py checks both builders give identical BlockSets).

    python baseline/ref_arm.py sample  --nb NB --D D --cores C [--budget V]  -> JSON
    python baseline/ref_arm.py configs                                      -> JSON

`sample`: C worker processes, each running ONE DP call of the workload
(calls spread evenly over the form_stage enumeration, stages.py:389-403)
through `pipecut.form_stage_dp` with pruning off (the metric's unit,
SURVEY.md §8d) and a fixed `visit_budget`: the reference's own per-cell
check (stages.py:214-216) stops it with SearchBudgetExceeded at exactly the
first cell past the budget.  The work is deterministic -- the same prefix of
the same calls on every run, whatever --steps is.  The value is the total
visits over the slowest worker's wall time.

Complete calls are out of reach at these sizes: a level of the reference scans
every previous-level cell for every cell (stages.py:220-222) and profiles each
span by a fold over its tasks (costs.py:120-160), so one nb = 4096 call takes
hours (DESIGN.md §6 has one measured extrapolation).  The budgeted prefix
stays inside level 1, where a cell costs O(1) candidates but counts up to
b*d visits: the sampled rate FAVOURS the reference.

`configs`: C1-C4 partition_blocks + form_stage, each config
in its own process, wall seconds per phase.
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import random
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "_ref")
if REF not in sys.path:
    sys.path.insert(0, REF)

import pipecut as pc  # noqa: E402  (the unmodified reference install)
from pipecut import graph as _g  # noqa: E402

CONFIGS = {
    # name: (generator, args, (nodes, dpn, memory bytes), k, batch) -- SURVEY.md §8d
    "C1": ("bert", (1024, 24, 512, 30522), (1, 8, 2 ** 35), 32, 256),
    "C2": ("bert", (2048, 96, 512, 30522), (4, 8, 32e9), 32, 256),
    "C3": ("resnet", (152, 8), (1, 8, 180e9), 32, 128),
    "C4": ("bert", (4096, 256, 512, 30522), (32, 8, 32e9), 32, 2048),
}


def _val(vid, fixed=0, per_sample=0, param=False):
    return _g.Node(vid, value=_g.ValueInfo(fixed_bytes=fixed, bytes_per_sample=per_sample,
                                           is_param=param))


def chain_graph(nb, hidden=1024, seq=512, jitter_seed=None):
    """C5: one task per BERT-1024 layer, ids t%05d, optional +-10% FLOP jitter."""
    h, s = hidden, seq
    heads = max(1, h // 64)
    flops = 24.0 * s * h * h + 4.0 * s * s * h + 5.0 * s * s * heads + 52.0 * s * h
    rng = random.Random(jitter_seed) if jitter_seed is not None else None
    nodes, edges, prev = [_val("x", per_sample=s * 8)], [], "x"
    for i in range(nb):
        t, v, w = f"t{i:05d}", f"v{i:05d}", f"w{i:05d}"
        f = flops if rng is None else flops * rng.uniform(0.9, 1.1)
        nodes += [_g.Node(t, task=_g.TaskInfo(op="layer", flops_per_sample=f, attrs={})),
                  _val(v, per_sample=s * h * 4),
                  _val(w, fixed=(12 * h * h + 13 * h) * 4, param=True)]
        edges += [(prev, t), (w, t), (t, v)]
        prev = v
    return pc.TaskGraph(nodes, edges, ["x"], [prev])


def chain_blockset(nb, D, jitter_seed=None):
    nodes, dpn = max(1, D // 8), min(8, D)
    cl = pc.ClusterSpec(nodes, dpn, int(32e9), 50e9, 10e9)
    part = pc.build_atomic_subcomponents(chain_graph(nb, jitter_seed=jitter_seed))
    model = pc.CostModel(part.graph, pc.CostModelConfig(), cl)
    return pc.partition_blocks(part, model, k=10 ** 6)


def config_inputs(name):
    kind, args, (nodes, dpn, mem), k, batch = CONFIGS[name]
    g = pc.gen_bert_like(*args) if kind == "bert" else pc.gen_resnet_like(*args)
    cl = pc.ClusterSpec(nodes, dpn, int(mem), 50e9, 10e9)
    part = pc.build_atomic_subcomponents(g)
    model = pc.CostModel(part.graph, pc.CostModelConfig(), cl)
    return part, model, k, batch, cl


def enumerate_calls(num_nodes, dpn, batch_size, nb):
    """form_stage's (S, D, R, MB) calls in its order (stages.py:389-403)."""
    out, n = [], 1
    while n <= num_nodes:
        if num_nodes % n == 0:
            D, R = dpn * n, num_nodes // n
            for S in range(dpn * (n - 1) + 1, D + 1):
                if S > nb:
                    continue
                MB = 1
                while MB * R <= batch_size:
                    out.append((S, D, R, MB))
                    MB *= 2
        n *= 2
    return out


def unpruned(nb, call):
    S, D, _, _ = call
    A, B = nb - S + 1, D - S + 1
    return S * (A * (A + 1) // 2) * (B * (B + 1) // 2)


class _Opts:
    """SearchOptions-compatible: pruning off, a fixed visit budget."""

    def __init__(self, budget):
        self.disable_pruning = True
        self.visit_budget = budget


_BS = None


def _init(nb, D, seed):
    global _BS
    _BS = chain_blockset(nb, D, jitter_seed=seed)


def _run(args):
    """One budgeted call -> (visits, seconds)."""
    call, batch, budget = args
    S, D, R, MB = call
    t0 = time.perf_counter()
    try:
        res = pc.form_stage_dp(_BS, S, D, batch, R, MB, _Opts(budget))
        visits = res.stats.visits
    except pc.SearchBudgetExceeded as exc:
        visits = exc.visits
    return visits, time.perf_counter() - t0


def sample_calls(calls, k):
    step = max(1, len(calls) // k)
    return [calls[(i * step + step // 2) % len(calls)] for i in range(k)]


def sample(nb, D, cores, budget, seed=0, pool=None):
    """One deterministic sample step (see module docstring)."""
    calls = enumerate_calls(max(1, D // 8), min(8, D), 8 * D, nb)
    picks = sample_calls(calls, cores)
    work = [(c, 8 * D, budget) for c in picks]
    if pool is None:
        if _BS is None or len(_BS) != nb:
            _init(nb, D, seed)
        res = [_run(w) for w in work]
    else:
        res = pool.map(_run, work)
    visits = sum(v for v, _ in res)
    slowest = max(t for _, t in res)
    return {"value": visits / slowest, "visits": visits, "seconds": slowest,
            "calls": [list(c) for c in picks], "budget_per_call": budget}


def make_pool(nb, D, cores, seed=0):
    return mp.get_context("fork").Pool(cores, initializer=_init, initargs=(nb, D, seed))


def _config_job(name):
    part, model, k, batch, cl = config_inputs(name)
    t0 = time.perf_counter()
    bs = pc.partition_blocks(part, model, k)
    t1 = time.perf_counter()
    res = pc.form_stage(cl.num_nodes, cl.devices_per_node, batch, bs)
    t2 = time.perf_counter()
    return name, {"partition_blocks_ms": (t1 - t0) * 1e3, "form_stage_ms": (t2 - t1) * 1e3,
                  "total_ms": (t2 - t0) * 1e3, "visits": res.stats.visits,
                  "dp_calls": res.stats.dp_calls,
                  "objective": None if res.plan is None else res.plan.objective.hex()}


def configs():
    with mp.get_context("fork").Pool(len(CONFIGS)) as pool:
        return dict(pool.map(_config_job, list(CONFIGS)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["sample", "configs"])
    ap.add_argument("--nb", type=int, default=4096)
    ap.add_argument("--D", type=int, default=1024)
    ap.add_argument("--cores", type=int, default=1)
    ap.add_argument("--budget", type=int, default=3 * 10 ** 6)
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    if a.what == "configs":
        print(json.dumps(configs()))
    else:
        print(json.dumps(sample(a.nb, a.D, a.cores, a.budget, a.seed)))


if __name__ == "__main__":
    main()
