"""CPU: pin the oracle (oracle/pipecut_oracle.c) and the flattener against the
reference -- live (baseline/_ref or /root/reference) and the committed golden
fixtures generated from the reference by tests/golden/make_golden.py."""

import json
import os
import random

import pytest

import cases
from oracle.oracle import OracleProblem, PC_OK
from paper_2103_16063_b200._host import pipecut as pc
from paper_2103_16063_b200.flatten import flatten_blockset

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _oracle_plan_doc(rc, stages, obj, S, D, BS, R, MB):
    if rc != PC_OK:
        return None
    return {"stages": [[lo, hi, dev, dev * R, tf.hex(), tb.hex(), mem]
                       for (lo, hi, dev, tf, tb, mem) in stages],
            "microbatches": MB, "replica_factor": R, "objective": obj.hex(),
            "batch_size": BS, "devices_total": D}


def _rebuild(rec):
    rng = random.Random(rec["seed"])
    gen = cases.stages_random_instance if rec["family"] == "stages" else cases.search_instance
    for _ in range(rec["index"] + 1):
        inst = gen(rng)
    return inst


def _golden_random():
    with open(os.path.join(GOLD, "random_dp.json")) as fh:
        return json.load(fh)


def test_span_profile_matches_reference_random_graphs():
    """A.1 restatement: every span x m x ckpt equals CostModel.profile."""
    rng = random.Random(2024)
    checked = 0
    for _ in range(12):
        bs, *_ = cases.stages_random_instance(rng)
        op = OracleProblem(flatten_blockset(bs))
        nb = len(bs)
        for lo in range(nb):
            for hi in range(lo + 1, nb + 1):
                for m in (1, 3, 7):
                    for ck in (False, True):
                        r = bs.model.profile(bs.span(lo, hi), m, checkpointing=ck)
                        assert op.span(lo, hi, m, ck) == (r.t_fwd_sec, r.t_bwd_sec, r.mem_bytes)
                        checked += 1
    assert checked > 500


@pytest.mark.parametrize("kind", ["bert", "resnet"])
def test_span_profile_matches_reference_model_graphs(kind):
    g = pc.gen_bert_like(64, 3, 16, 100) if kind == "bert" else pc.gen_resnet_like(50, 1)
    cl = pc.ClusterSpec(2, 2, 2 ** 40, 50e9, 10e9)
    part = pc.build_atomic_subcomponents(g)
    model = pc.CostModel(part.graph, pc.CostModelConfig(), cl)
    bs = pc.partition_blocks(part, model, 12)
    fp = flatten_blockset(bs)
    op = OracleProblem(fp)
    for lo in range(len(bs)):
        for hi in range(lo + 1, len(bs) + 1):
            for m in (1, 4):
                for ck in (False, True):
                    r = model.profile(bs.span(lo, hi), m, checkpointing=ck)
                    assert op.span(lo, hi, m, ck) == (r.t_fwd_sec, r.t_bwd_sec, r.mem_bytes)


@pytest.mark.parametrize("beta", [3.0, 1.5, 0.7, 4.0])
def test_span_profile_matches_reference_backward_ratio(beta):
    """beta * x per task folded without FMA (costs.py:138-140; test_costs.py
    uses beta = 3): the oracle's t_bwd equals CostModel.profile's bit for bit."""
    g = pc.gen_bert_like(64, 3, 16, 100)
    cl = pc.ClusterSpec(2, 2, 2 ** 40, 50e9, 10e9)
    part = pc.build_atomic_subcomponents(g)
    model = pc.CostModel(part.graph, pc.CostModelConfig(bwd_fwd_ratio=beta), cl)
    bs = pc.partition_blocks(part, model, 12)
    op = OracleProblem(flatten_blockset(bs))
    for lo in range(len(bs)):
        for hi in range(lo + 1, len(bs) + 1):
            for m in (1, 5):
                r = model.profile(bs.span(lo, hi), m, checkpointing=True)
                assert op.span(lo, hi, m, True) == (r.t_fwd_sec, r.t_bwd_sec, r.mem_bytes)


def test_cut_time_matches_reference():
    rng = random.Random(11)
    for _ in range(10):
        bs, *_ = cases.stages_random_instance(rng)
        op = OracleProblem(flatten_blockset(bs))
        prof = pc.stages._Profiler(bs)
        for cut in range(len(bs) + 1):
            for m in (1, 2, 9):
                for cum in range(1, 7):
                    assert op.cut_time(cut, m, cum) == prof.cut_time(cut, m, cum)


def test_oracle_dp_matches_golden_random_families():
    """The reference's own DP test families (test_stages.py:158-241,
    test_acceptance.py:92-176): plans, objectives and visits, pruned and not."""
    recs = _golden_random()
    assert len(recs) == 275
    for rec in recs:
        bs, S, D, BS, R, MB = _rebuild(rec)
        assert [S, D, BS, R, MB] == rec["args"]
        op = OracleProblem(flatten_blockset(bs))
        for key, prune in (("pruned", True), ("unpruned", False)):
            rc, stages, obj, visits = op.form_stage_dp(S, D, BS, R, MB, disable_pruning=not prune)
            assert _oracle_plan_doc(rc, stages, obj, S, D, BS, R, MB) == rec[key]["plan"], rec
            assert visits == rec[key]["visits"]


def test_oracle_known_optima():
    """Known answers of test_stages.py:57-106."""
    def run(flops, S, D, BS, R, MB, **kw):
        bs = cases.one_block_per_task(cases.chain(flops, kw.pop("sizes", None),
                                                  kw.pop("params", None)), **kw)
        return OracleProblem(flatten_blockset(bs)).form_stage_dp(S, D, BS, R, MB)

    rc, st, obj, _ = run([1.0, 1.0], 2, 2, 1, 1, 1)
    assert obj == 3.0 and [(s[0], s[1]) for s in st] == [(0, 1), (1, 2)]
    rc, st, obj, _ = run([3.0, 1.0, 1.0, 1.0], 2, 2, 1, 1, 1)
    assert obj == 9.0 and [(s[0], s[1]) for s in st] == [(0, 1), (1, 4)]
    rc, st, obj, _ = run([3.0, 1.0, 1.0, 1.0], 1, 1, 2, 1, 1, params=[0, 0, 0, 128])
    assert obj == 36.0 and st[0][3] == 12.0 and st[0][5] == 512
    rc, st, obj, _ = run([1.0, 1.0], 2, 2, 1, 1, 1, sizes=[1000, 0], dpn=2, bw=(1000.0, 1000.0))
    assert obj == 5.0
    rc, st, obj, _ = run([1.0, 1.0], 1, 1, 8, 1, 1, sizes=[1000, 1000], mem=5000)
    assert rc != PC_OK
    bs = cases.one_block_per_task(cases.chain([1.0, 1.0]))
    rc, _, _, visits = OracleProblem(flatten_blockset(bs)).form_stage_dp(
        1, 2, 4, 1, 1, disable_pruning=True)
    assert visits == 9                                   # test_stages.py:137-142


def test_oracle_form_stage_matches_golden_chains():
    with open(os.path.join(GOLD, "chains.json")) as fh:
        gold = json.load(fh)
    for key, doc in gold.items():
        nb, D, seed = key.split("_")
        nb, D = int(nb[2:]), int(D[1:])
        seed = None if seed == "seedNone" else int(seed[4:])
        bs = cases.c5_blockset(nb, D, jitter_seed=seed)
        op = OracleProblem(flatten_blockset(bs))
        rc, plan, visits, calls = op.form_stage(max(1, D // 8), min(8, D), 8 * D,
                                                disable_pruning=True)
        want = doc["plan"]
        assert rc == PC_OK
        assert plan["objective"].hex() == want["objective"]
        assert [[s[0], s[1], s[2]] for s in plan["stages"]] == [s[:3] for s in want["stages"]]
        assert plan["MB"] == want["microbatches"] and plan["R"] == want["replica_factor"]
        assert visits == doc["visits"] and calls == doc["dp_calls"]


def test_oracle_span_row_path_matches_per_span_and_reference():
    """The oracle's memo-row fold (monotone graphs: chains and the reference's
    random DP families are monotone) equals its per-span fold and
    CostModel.profile bit for bit, at every span, share and ckpt."""
    rng = random.Random(31)
    cases_ = [cases.c5_blockset(40, 16, jitter_seed=3)]
    for _ in range(6):
        cases_.append(cases.stages_random_instance(rng)[0])
    checked = 0
    for bs in cases_:
        fp = flatten_blockset(bs)
        if not fp.monotone:
            continue
        op = OracleProblem(fp)
        nb = len(bs)
        for lo in range(nb):
            for hi in range(lo + 1, nb + 1):
                for m in (1, 5, 64):
                    for ck in (False, True):
                        got = op.span_row(lo, hi, m, ck)
                        assert got == op.span(lo, hi, m, ck)
                        if (lo * 7 + hi) % 5 == 0:
                            r = bs.model.profile(bs.span(lo, hi), m, checkpointing=ck)
                            assert got == (r.t_fwd_sec, r.t_bwd_sec, r.mem_bytes)
                        checked += 1
    assert checked > 5000
