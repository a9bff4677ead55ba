"""Negative task times: the reference accepts negative
flops_per_sample (graph.py:45-48, never checked) and negative measured
cost-table times (costs.py:57-80 parses any float), so span times need not be
monotone and their sign is data.  The device marks infeasible spans with NaN
in that case (common.cuh: span_mark) instead of the sign bit, and turns the
DP's prefix skip off.  Checked live against the unmodified reference
(baseline/_ref): form_stage_dp pruned/unpruned, form_stage and
brute_force_partition, plans bit-exact."""

import random

import pytest

import cases
from plans import result_doc
from paper_2103_16063_b200 import brute_force_partition, form_stage, form_stage_dp
from paper_2103_16063_b200._host import pipecut as pc

pytestmark = pytest.mark.gpu


def _neg_instance(rng):
    """test_stages.py-style chain whose FLOPs may be negative, tight budgets."""
    n = rng.randint(3, 9)
    flops = [round(rng.uniform(-2.0, 4.0), 3) for _ in range(n)]
    sizes = [rng.choice([0, 64, 256, 1024]) for _ in range(n)]
    params = [rng.choice([0, 0, 512, 2048]) for _ in range(n)]
    S = rng.randint(1, min(4, n))
    D = rng.randint(S, 6)
    R = rng.choice([1, 2])
    MB = rng.choice([1, 2, 4])
    BS = R * MB * D * rng.randint(1, 3)
    state = sum(p * 4 for p in params)
    acts = sum(sizes) * (BS // (MB * R)) + 64
    budget = rng.choice([2 ** 40, max(int((state + acts) * rng.uniform(0.3, 0.9)), 64)])
    nodes, dpn = rng.choice([(1, 6), (2, 3)])
    g = cases.chain(flops, sizes, params, x_bytes=16)
    while True:
        try:
            bs = cases.one_block_per_task(g, mem=budget, nodes=nodes, dpn=dpn, bw=(1e3, 5e2),
                                          latency=rng.choice([0.0, 0.01]),
                                          ckpt=rng.random() < 0.5)
            return bs, S, D, BS, R, MB, (nodes, dpn)
        except pc.InfeasibleAtom:
            budget *= 4


def _both(fn_ours, fn_ref):
    def run(fn):
        try:
            return result_doc(fn()), None
        except Exception as e:  # noqa: BLE001
            return None, (type(e).__name__, str(e))
    return run(fn_ours), run(fn_ref)


def test_negative_flops_match_reference(gpu):
    rng = random.Random(909)
    n_inf = n_neg = 0
    for _ in range(60):
        bs, S, D, BS, R, MB, (nodes, dpn) = _neg_instance(rng)
        n_neg += any(c.t_fwd_sec < 0 for c in bs.costs)
        for prune in (True, False):
            opts = pc.SearchOptions(disable_pruning=not prune)
            a, b = _both(lambda: form_stage_dp(bs, S, D, BS, R, MB, opts),
                         lambda: pc.form_stage_dp(bs, S, D, BS, R, MB, opts))
            assert a == b
            n_inf += a[0] is not None and a[0]["plan"] is None
        a, b = _both(lambda: form_stage(nodes, dpn, BS, bs),
                     lambda: pc.form_stage(nodes, dpn, BS, bs))
        assert a == b
        if len(bs) <= 12 and D <= 8:
            a, b = _both(lambda: brute_force_partition(bs, S, D, BS, R, MB),
                         lambda: pc.brute_force_partition(bs, S, D, BS, R, MB))
            assert a == b
    assert n_neg > 20 and n_inf > 0


def _neg_cost_table_instance(rng):
    n = rng.randint(3, 9)
    g = cases.typed_chain(rng, n)
    S = rng.randint(1, min(4, n))
    nodes, dpn = rng.choice([(1, 4), (2, 2)])
    D = rng.randint(S, nodes * dpn)
    R = rng.choice([1, 2])
    MB = rng.choice([1, 2, 4])
    BS = R * MB * D * rng.randint(1, 3)
    table = {}
    for op, attrs in cases.TYPED_OPS:
        info = pc.graph.TaskInfo(op=op, flops_per_sample=0.0, attrs=dict(attrs))
        for m in range(1, BS + 1):
            if rng.random() < 0.4:
                continue
            tb = None if rng.random() < 0.5 else round(rng.uniform(-3.0, 8.0), 4)
            act = None if rng.random() < 0.5 else rng.choice([0, 300, 4096])
            table[pc.costs.op_signature(info, m)] = pc.CostTableEntry(
                microbatch=m, t_fwd=round(rng.uniform(-3.0, 6.0), 4), t_bwd=tb, act_bytes=act)
    budget = rng.choice([2 ** 40, rng.randint(4096, 65536)])
    cl = pc.ClusterSpec(num_nodes=nodes, devices_per_node=dpn, device_memory_bytes=budget,
                        bw_intra=1e3, bw_inter=5e2, link_latency_sec=rng.choice([0.0, 0.01]))
    part = pc.build_atomic_subcomponents(g)
    cfg = pc.CostModelConfig(device_flops_per_sec=1.0, checkpointing=rng.random() < 0.5,
                             cost_table=table)
    model = pc.CostModel(part.graph, cfg, cl)
    try:
        bs = pc.partition_blocks(part, model, 10 ** 6)
    except pc.InfeasibleAtom:
        return None
    return bs, S, D, BS, R, MB, (nodes, dpn)


def test_negative_cost_table_times_match_reference(gpu):
    rng = random.Random(4711)
    done = 0
    while done < 40:
        inst = _neg_cost_table_instance(rng)
        if inst is None:
            continue
        bs, S, D, BS, R, MB, (nodes, dpn) = inst
        for prune in (True, False):
            opts = pc.SearchOptions(disable_pruning=not prune)
            a, b = _both(lambda: form_stage_dp(bs, S, D, BS, R, MB, opts),
                         lambda: pc.form_stage_dp(bs, S, D, BS, R, MB, opts))
            assert a == b
        a, b = _both(lambda: form_stage(nodes, dpn, BS, bs),
                     lambda: pc.form_stage(nodes, dpn, BS, bs))
        assert a == b
        done += 1


def test_nan_flops_rejected(gpu):
    g = cases.chain([1.0, float("nan"), 2.0])
    bs = cases.one_block_per_task(g)
    with pytest.raises(ValueError, match="NaN"):
        form_stage_dp(bs, 2, 2, 4, 1, 1)
