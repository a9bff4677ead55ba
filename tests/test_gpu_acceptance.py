"""The reference's acceptance gate (pkg/tests/test_acceptance.py, criteria
1-8 and its frozen constants) restated on the device path: every search,
enumeration, coarsening, validation and simulation below runs through the
drop-ins of paper_2103_16063_b200.  Where the reference's own result is cheap
to get (baseline/_ref, unmodified) it is compared exactly too."""

import csv
import importlib
import json
import math
import os
import random
import time

import pytest

import cases
from paper_2103_16063_b200 import (brute_force_partition, form_stage, form_stage_dp, install,
                                   partition_blocks)
from paper_2103_16063_b200._host import pipecut as pc
from paper_2103_16063_b200.simulate import simulate, validate_plan
from plans import result_doc

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")

SEARCH_SEED, SEARCH_COUNT, SEARCH_TIME_LIMIT_SEC = 777, 120, 60.0   # test_acceptance.py:33-36
STRICT_PRUNING_FRACTION = 0.90
FORMULA_REL_TOL = 1e-9
SCALE_GRAPH = (1024, 96, 512, 30522)                                  # :47-54
SCALE_CLUSTER = dict(num_nodes=2, devices_per_node=2, device_memory_bytes=2 ** 35,
                     bw_intra=50e9, bw_inter=10e9)
SCALE_BATCH, SCALE_K, SCALE_BUDGET_FACTOR = 64, 32, 10
BALANCE_GRAPH, BALANCE_K = (1024, 16, 512, 30522), 8                  # :56-62
BALANCE_MAX_OVER_MEAN, NAIVE_MAX_OVER_MEAN = 1.50, 1.66
SWEEP_LAYERS = (24, 48, 96, 192)                                      # :64-68


@pytest.fixture(scope="module")
def searches():
    rng = random.Random(SEARCH_SEED)
    out = []
    t0 = time.monotonic()
    for _ in range(SEARCH_COUNT):
        bs, S, D, BS, R, MB = cases.search_instance(rng)
        out.append((bs, S, D, BS, R, MB, form_stage_dp(bs, S, D, BS, R, MB)))
    return out, time.monotonic() - t0


def test_criterion_1_search_equals_enumeration(gpu, searches):
    runs, elapsed = searches
    t0 = time.monotonic()
    bad = []
    for i, (bs, S, D, BS, R, MB, res) in enumerate(runs):
        ref = brute_force_partition(bs, S, D, BS, R, MB).plan
        got = None if res.plan is None else res.plan.objective
        if got != (None if ref is None else ref.objective):
            bad.append(i)
    assert not bad and elapsed + time.monotonic() - t0 < SEARCH_TIME_LIMIT_SEC
    assert sum(r.plan is not None for *_, r in runs) > 30


def test_criterion_2_pruning_only_skips_work(gpu, searches):
    runs, _ = searches
    strict = 0
    for bs, S, D, BS, R, MB, res in runs:
        off = form_stage_dp(bs, S, D, BS, R, MB, pc.SearchOptions(disable_pruning=True))
        assert off.plan == res.plan
        assert res.stats.visits <= off.stats.visits
        strict += res.stats.visits < off.stats.visits
    assert strict >= math.ceil(STRICT_PRUNING_FRACTION * SEARCH_COUNT)


def test_criterion_4_fill_drain_identity(gpu):
    worst = 0.0
    for S in (1, 2, 3, 4):
        for MB in (1, 2, 4, 8):
            bs = cases.one_block_per_task(cases.chain([1.0] * S), dpn=S)
            plan = form_stage_dp(bs, S, S, MB * 8, 1, MB).plan
            sched = simulate(plan, bs)
            tf, tb = plan.stages[0].t_fwd, plan.stages[0].t_bwd
            want = (MB + S - 1) * (tf + tb)
            worst = max(worst, abs(sched.iteration_time_sec - want) / want)
    assert worst <= FORMULA_REL_TOL


def test_criterion_5_block_search_scale(gpu):
    g = pc.gen_bert_like(*SCALE_GRAPH)
    cl = pc.ClusterSpec(**SCALE_CLUSTER)
    part = pc.build_atomic_subcomponents(g)
    model = pc.CostModel(part.graph, pc.CostModelConfig(), cl)
    blocks = partition_blocks(part, model, SCALE_K)
    res = form_stage(cl.num_nodes, cl.devices_per_node, SCALE_BATCH, blocks)
    assert res.plan is not None
    # the reference's own coarsening and search on the same inputs
    ref_blocks = pc.partition_blocks(part, model, SCALE_K)
    assert blocks.block_atoms == ref_blocks.block_atoms and blocks.costs == ref_blocks.costs
    assert result_doc(res) == result_doc(pc.form_stage(cl.num_nodes, cl.devices_per_node,
                                                       SCALE_BATCH, ref_blocks))
    budget = SCALE_BUDGET_FACTOR * res.stats.visits
    atom_blocks = partition_blocks(part, model, len(part.atoms))
    assert len(atom_blocks) == len(part.atoms)
    with pytest.raises(pc.SearchBudgetExceeded) as err:
        form_stage(cl.num_nodes, cl.devices_per_node, SCALE_BATCH, atom_blocks,
                   options=pc.SearchOptions(visit_budget=budget))
    assert err.value.visits > budget
    with pytest.raises(pc.SearchBudgetExceeded) as ref_err:
        pc.form_stage(cl.num_nodes, cl.devices_per_node, SCALE_BATCH,
                      pc.partition_blocks(part, model, len(part.atoms)),
                      options=pc.SearchOptions(visit_budget=budget))
    assert err.value.visits == ref_err.value.visits


def _layer_of_atoms(part):
    """Model layer of each atom ("L<n>." task ids), embedding/head folded into
    the first/last layer (test_acceptance.py:246-268)."""
    tags = []
    for atom in part.atoms:
        tag = next((int(nid.split(".")[0][1:]) for nid in sorted(atom.node_ids)
                    if part.graph.nodes[nid].is_task and nid.startswith("L") and "." in nid),
                   None)
        tags.append(tag)
    layers = sorted({t for t in tags if t is not None})
    groups = {layer: [] for layer in layers}
    for i, t in enumerate(tags):
        groups[t if t is not None else (layers[0] if i < len(tags) / 2 else layers[-1])].append(i)
    return [groups[layer] for layer in layers]


def test_criterion_6_balance_beats_equal_layers(gpu):
    g = pc.gen_bert_like(*BALANCE_GRAPH)
    cl = pc.ClusterSpec(num_nodes=1, devices_per_node=BALANCE_K, device_memory_bytes=2 ** 35,
                        bw_intra=50e9, bw_inter=10e9)
    part = pc.build_atomic_subcomponents(g)
    model = pc.CostModel(part.graph, pc.CostModelConfig(), cl)
    comp = [r.t_fwd_sec + r.t_bwd_sec
            for r in (model.profile(a, 1, checkpointing=False) for a in part.atoms)]
    mean = sum(comp) / BALANCE_K
    blocks = partition_blocks(part, model, BALANCE_K)
    ratio = max(c.t_fwd_sec + c.t_bwd_sec for c in blocks.costs) / mean
    groups = _layer_of_atoms(part)
    per = len(groups) // BALANCE_K
    naive = [sum(comp[groups[i * per][0]:(groups[(i + 1) * per][0] if i < BALANCE_K - 1
                                            else len(comp))]) for i in range(BALANCE_K)]
    assert ratio <= BALANCE_MAX_OVER_MEAN and max(naive) / mean >= NAIVE_MAX_OVER_MEAN


def _convex(atoms, succ):
    """No path leaves the set and comes back (blocks.py:45-70)."""
    inside = set(atoms)
    stack = [b for a in atoms for b in succ[a] if b not in inside]
    seen = set(stack)
    while stack:
        x = stack.pop()
        for y in succ[x]:
            if y in inside:
                return False
            if y not in seen:
                seen.add(y)
                stack.append(y)
    return True


def test_criterion_7_structural_invariants(gpu, searches):
    runs, _ = searches
    plans = [(r.plan, bs) for bs, *_, r in runs if r.plan is not None]
    assert all(validate_plan(p, bs) == [] for p, bs in plans)
    for bs in {id(bs): bs for bs, *_ in runs}.values():
        succ = [[] for _ in bs.partition.atoms]
        for a, b in bs.partition.dependencies():
            succ[a].append(b)
        budget = bs.model.cluster.device_memory_bytes
        for atoms, cost in zip(bs.block_atoms, bs.costs):
            assert _convex(atoms, succ) and cost.mem_bytes <= budget
    for p, bs in plans[:40]:
        sched = simulate(p, bs)
        lanes = {}
        for e in sched.events:
            lanes.setdefault(e.device, []).append(e)
        for evs in lanes.values():
            evs.sort(key=lambda e: (e.start_sec, e.end_sec))
            assert all(b.start_sec >= a.end_sec - 1e-12 for a, b in zip(evs, evs[1:]))
            assert sum(e.phase == "fwd" for e in evs) == p.microbatches
            assert sum(e.phase == "bwd" for e in evs) == p.microbatches


def test_criterion_8_data_parallel_fails_first(gpu, tmp_path, capsys):
    """The reference CLI's sweep on the device path (install()), equal to the
    reference's own sweep.csv (golden/sweep_c8.csv) and meeting the gate."""
    cluster = dict(num_nodes=2, devices_per_node=2, device_memory_bytes=32 * 10 ** 9,
                   bw_intra=50e9, bw_inter=10e9, link_latency_sec=0.0)
    (tmp_path / "cluster.json").write_text(json.dumps(cluster))
    cli = importlib.import_module(pc.__name__ + ".cli")
    restore = install()
    try:
        rc = cli.main(["sweep", "--cluster", str(tmp_path / "cluster.json"), "--hidden", "2048",
                       "--layers", ",".join(map(str, SWEEP_LAYERS)), "--batch-size", "32",
                       "--out", str(tmp_path)])
    finally:
        restore()
    assert rc == 0
    text = (tmp_path / "sweep.csv").read_text()
    with open(os.path.join(GOLD, "sweep_c8.csv")) as fh:
        assert text == fh.read()
    rows = list(csv.DictReader(text.splitlines()))
    dp_fail = min(int(r["layers"]) for r in rows if r["data_parallel"] == "INFEASIBLE")
    part_fail = min(int(r["layers"]) for r in rows if r["status"] == "INFEASIBLE")
    rescued = [int(r["layers"]) for r in rows
               if r["status"] == "ok" and r["data_parallel"] == "INFEASIBLE"]
    both = [int(r["layers"]) for r in rows if r["status"] == "ok" and r["data_parallel"] == "ok"]
    assert dp_fail < part_fail and rescued and all(n < dp_fail for n in both)
