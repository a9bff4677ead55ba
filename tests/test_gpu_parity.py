"""GPU parity: the CUDA path (through the C-ABI) against the reference's
golden fixtures and the oracle.  Bit-exact plans, objectives and visits."""

import json
import os
import random

import numpy as np
import pytest

import cases
from oracle.oracle import OracleProblem, PC_OK
from paper_2103_16063_b200 import abi, form_stage, form_stage_dp, form_stage_sharded
from paper_2103_16063_b200._host import pipecut as pc
from paper_2103_16063_b200.stages import bind_problem
from plans import result_doc

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


def _rebuild(rec):
    rng = random.Random(rec["seed"])
    gen = cases.stages_random_instance if rec["family"] == "stages" else cases.search_instance
    for _ in range(rec["index"] + 1):
        inst = gen(rng)
    return inst


def test_profile_spans_match_oracle(gpu):
    import ctypes as C
    rng = random.Random(3)
    graphs = [cases.stages_random_instance(rng)[0] for _ in range(6)]
    g = pc.gen_bert_like(64, 3, 16, 100)
    part = pc.build_atomic_subcomponents(g)
    graphs.append(pc.partition_blocks(part, pc.CostModel(part.graph, pc.CostModelConfig(),
                                                         pc.ClusterSpec(2, 2, 2 ** 40, 5e10, 1e10)), 12))
    graphs.append(cases.c5_blockset(40, 16, jitter_seed=3))
    for bs in graphs:
        flat = bind_problem(gpu, bs)
        op = OracleProblem(flat)
        nb = len(bs)
        q = [(lo, hi, m, ck) for lo in range(nb) for hi in range(lo + 1, nb + 1)
             for m in (1, 5) for ck in (0, 1)]
        lo = np.array([x[0] for x in q], np.int32)
        hi = np.array([x[1] for x in q], np.int32)
        m = np.array([x[2] for x in q], np.int64)
        ck = np.array([x[3] for x in q], np.int32)
        tf, tb, mem = np.zeros(len(q)), np.zeros(len(q)), np.zeros(len(q), np.int64)
        rc = gpu.lib.pc_profile_spans(gpu.h, len(q), lo.ctypes.data, hi.ctypes.data,
                                      m.ctypes.data, ck.ctypes.data, tf.ctypes.data,
                                      tb.ctypes.data, mem.ctypes.data)
        assert rc == 0, gpu.error()
        for i, (a, b, mm, c) in enumerate(q):
            assert (float(tf[i]), float(tb[i]), int(mem[i])) == op.span(a, b, mm, c)


def test_form_stage_dp_golden_random_families(gpu):
    recs = _load("random_dp.json")
    for rec in recs:
        bs, S, D, BS, R, MB = _rebuild(rec)
        for key, prune in (("pruned", True), ("unpruned", False)):
            res = form_stage_dp(bs, S, D, BS, R, MB, pc.SearchOptions(disable_pruning=not prune))
            assert result_doc(res) == rec[key], (rec["family"], rec["seed"], rec["index"], key)


def test_known_optima_and_accounting(gpu):
    bs = cases.one_block_per_task(cases.chain([1.0, 1.0]))
    plan = form_stage_dp(bs, 2, 2, 1, 1, 1).plan
    assert plan.objective == 3.0
    assert [st.blocks for st in plan.stages] == [(0, 1), (1, 2)]
    assert [st.replicas for st in plan.stages] == [1, 1]
    bs = cases.one_block_per_task(cases.chain([3.0, 1.0, 1.0, 1.0], params=[0, 0, 0, 128]))
    plan = form_stage_dp(bs, 1, 1, 2, 1, 1).plan
    assert plan.objective == 36.0 and plan.stages[0].t_fwd == 12.0 and plan.stages[0].mem == 512
    bs = cases.one_block_per_task(cases.chain([1.0, 1.0], sizes=[1000, 1000]), mem=5000)
    res = form_stage_dp(bs, 1, 1, 8, 1, 1)
    assert res.plan is None and res.stats.dp_calls == 1
    g = cases.chain([1.0] * 4, sizes=[1000] * 4)
    bs = cases.one_block_per_task(g, mem=6000, ckpt=True)
    assert form_stage_dp(bs, 1, 2, 4, 1, 1).plan is None
    assert form_stage_dp(bs, 2, 2, 4, 1, 4).plan is not None
    bs = cases.one_block_per_task(cases.chain([1.0, 1.0]))
    assert form_stage_dp(bs, 1, 2, 1, 1, 1).plan is None
    assert form_stage_dp(bs, 1, 2, 4, 1, 1, pc.SearchOptions(disable_pruning=True)).stats.visits == 9
    with pytest.raises(pc.InvalidArgs):
        form_stage_dp(bs, 3, 4, 4, 1, 1)
    with pytest.raises(pc.InvalidArgs):
        form_stage_dp(bs, 1, 0, 4, 1, 1)


def test_budget_semantics_match_reference(gpu):
    """SearchBudgetExceeded at the first crossing cell, same visits value."""
    bs = cases.one_block_per_task(cases.chain([1.0] * 6))
    for budget in (0, 3, 10, 57, 200):
        try:
            pc.form_stage_dp(bs, 2, 4, 8, 1, 1, pc.SearchOptions(visit_budget=budget))
            want = None
        except pc.SearchBudgetExceeded as e:
            want = e.visits
        try:
            form_stage_dp(bs, 2, 4, 8, 1, 1, pc.SearchOptions(visit_budget=budget))
            got = None
        except pc.SearchBudgetExceeded as e:
            got = e.visits
            assert e.budget == budget
        assert got == want, budget
    bs = cases.one_block_per_task(cases.chain([1.0] * 4), nodes=1, dpn=2)
    for budget in (2, 20, 45, 80):
        def run(fn):
            try:
                r = fn(1, 2, 8, bs, pc.SearchOptions(visit_budget=budget))
                return ("ok", r.stats.visits)
            except pc.SearchBudgetExceeded as e:
                return ("budget", e.visits)
        want = run(pc.form_stage)
        assert run(form_stage) == want, budget
        for spec in (True, False):         # both sharded schedules
            assert run(lambda *a, **k: form_stage_sharded(*a, speculative=spec, **k)) == want
    # a multi-level search (2 nodes: widening levels n = 1, 2) with budgets that
    # cross in either level
    bs = cases.one_block_per_task(cases.chain([1.0, 2.0, 1.5, 1.0, 3.0]), nodes=2, dpn=2)
    for budget in (5, 40, 120, 400, 2000, None):
        def run2(fn):
            try:
                r = fn(2, 2, 8, bs, pc.SearchOptions(visit_budget=budget))
                return ("ok", r.stats.visits, r.stats.dp_calls,
                        None if r.plan is None else r.plan.objective)
            except pc.SearchBudgetExceeded as e:
                return ("budget", e.visits)
        want = run2(pc.form_stage)
        for spec in (True, False):
            assert run2(lambda *a, **k: form_stage_sharded(*a, speculative=spec, **k)) == want


def test_form_stage_small_cases(gpu):
    """test_stages.py TestFormStage shapes against the reference live."""
    cases_ = [
        (cases.one_block_per_task(cases.chain([1.0, 1.0]), nodes=1, dpn=1), (1, 1, 4)),
        (cases.one_block_per_task(cases.chain([1.0, 1.0], params=[64, 64]), nodes=2, dpn=1), (2, 1, 8)),
        (cases.one_block_per_task(cases.chain([1.0] * 4, params=[1000] * 4), mem=12000, nodes=2, dpn=1), (2, 1, 4)),
        (cases.one_block_per_task(cases.chain([1.0] * 4, params=[1000] * 4), mem=4500, nodes=2, dpn=1), (2, 1, 4)),
        (cases.one_block_per_task(cases.chain([2.0, 1.0, 1.0, 2.0], sizes=[64] * 4, params=[128] * 4),
                                  nodes=2, dpn=2, bw=(1e6, 5e5)), (2, 2, 16)),
    ]
    for bs, (n, dpn, BS) in cases_:
        want = result_doc(pc.form_stage(n, dpn, BS, bs))
        for spec in (True, False):
            assert result_doc(form_stage(n, dpn, BS, bs, speculative=spec)) == want


def test_form_stage_golden_chains(gpu):
    gold = _load("chains.json")
    for key, doc in gold.items():
        nb, D, seed = key.split("_")
        nb, D = int(nb[2:]), int(D[1:])
        seed = None if seed == "seedNone" else int(seed[4:])
        bs = cases.c5_blockset(nb, D, jitter_seed=seed)
        res = form_stage(max(1, D // 8), min(8, D), 8 * D, bs, pc.SearchOptions(disable_pruning=True))
        assert result_doc(res) == doc, key


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_form_stage_golden_configs(gpu, name):
    gold = _load("configs.json")[name]
    part, model, k, batch, cl = cases.config_partition(name)
    bs = pc.partition_blocks(part, model, k)
    assert [list(g) for g in bs.block_atoms] == gold["block_atoms"]
    res = form_stage(cl.num_nodes, cl.devices_per_node, batch, bs)
    assert result_doc(res) == gold["form_stage"]


def test_full_enumeration_per_call_matches_oracle(gpu):
    """C2 with every widening level (SURVEY §8d 'full enumeration'): each of the
    192 DP calls equals the oracle's _run_dp restatement."""
    import ctypes as C
    part, model, k, batch, cl = cases.config_partition("C2")
    bs = pc.partition_blocks(part, model, k)
    flat = bind_problem(gpu, bs)
    op = OracleProblem(flat)
    calls = []
    n = 1
    while n <= cl.num_nodes:
        if cl.num_nodes % n == 0:
            D, R = cl.devices_per_node * n, cl.num_nodes // n
            for S in range(cl.devices_per_node * (n - 1) + 1, D + 1):
                if S > len(bs):
                    continue
                MB = 1
                while MB * R <= batch:
                    calls.append((S, D, R, MB))
                    MB *= 2
        n *= 2
    arr = (abi.PcCall * len(calls))(*[abi.PcCall(*c) for c in calls])
    res = (abi.PcCallResult * len(calls))()
    bufs = [abi.PlanBuffers(c[0]) for c in calls]
    plans = (abi.PcPlan * len(calls))(*[b.s for b in bufs])
    st = abi.PcStats()
    rc = gpu.lib.pc_run_calls(gpu.h, len(calls), arr, batch, 0, 1, res, plans, C.byref(st))
    assert rc == 0, gpu.error()
    for i, (S, D, R, MB) in enumerate(calls):
        orc, stages, obj, visits = op.form_stage_dp(S, D, batch, R, MB)
        assert res[i].visits == visits
        assert bool(res[i].feasible) == (orc == PC_OK)
        if orc == PC_OK:
            assert res[i].objective == obj
            p = plans[i]
            got = [(bufs[i].lo[k], bufs[i].hi[k], bufs[i].devices[k], bufs[i].t_fwd[k],
                    bufs[i].t_bwd[k], bufs[i].mem[k]) for k in range(p.n_stages)]
            assert got == stages
            want_it = op.simulate(stages, batch, R, MB)
            assert res[i].iteration_time == want_it
