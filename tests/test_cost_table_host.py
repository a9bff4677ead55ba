"""Host side of measured cost tables (CPU): the dense override arrays the
device profiles read hold exactly the reference's table lookups
(costs.py:130-137), and the shares a search resolves cover every microbatch
size its span profiles are taken at (stages.py:201-206)."""

import math
import random

import numpy as np

import cases
from paper_2103_16063_b200._host import pipecut as pc
from paper_2103_16063_b200.flatten import flatten_atoms, flatten_blockset, resolve_overrides
from paper_2103_16063_b200.search import enumerate_calls
from paper_2103_16063_b200.stages import call_shares


def test_resolve_overrides_matches_reference_lookup():
    rng = random.Random(4242)
    checked = 0
    for _ in range(30):
        part, model, k, (nodes, dpn, S, D, BS, R, MB) = cases.cost_table_instance(rng)
        bs = pc.partition_blocks(part, pc.CostModel(part.graph, pc.CostModelConfig(
            device_flops_per_sec=1.0, cost_table=model.config.cost_table), pc.ClusterSpec(
            1, 1, 2 ** 40, 1.0, 1.0)), k)
        flat = flatten_blockset(bs)
        assert flat.has_cost_table
        shares = sorted({1, 2, 3, BS, BS + 1})
        ms, has, tf, tb, act = resolve_overrides(flat.cost_config, flat.task_nodes, shares)
        assert list(ms) == shares
        table = model.config.cost_table
        for i, m in enumerate(shares):
            for t, task in enumerate(flat.task_nodes):
                e = table.get(pc.costs.op_signature(task, m))
                assert bool(has[i, t]) == (e is not None)
                if e is None:
                    continue
                assert tf[i, t] == e.t_fwd
                assert (math.isnan(tb[i, t]) if e.t_bwd is None else tb[i, t] == e.t_bwd)
                assert act[i, t] == (-1 if e.act_bytes is None else e.act_bytes)
                checked += 1
        fa = flatten_atoms(part, model)
        ms1, has1, tf1, _, _ = resolve_overrides(model.config, fa_tasks(part), [1])
        assert np.array_equal(fa.ov_has, has1[0]) and np.array_equal(fa.ov_tf, tf1[0])
    assert checked > 100


def fa_tasks(part):
    g = part.graph
    return [g.nodes[nid].task for nid in sorted(g.nodes) if g.nodes[nid].task is not None]


def test_no_table_means_no_overrides():
    bs = cases.one_block_per_task(cases.chain([1.0, 2.0]))
    assert not flatten_blockset(bs).has_cost_table


def test_call_shares_cover_form_stage():
    for nodes, dpn, BS in ((1, 4, 16), (2, 2, 24), (4, 8, 512), (3, 2, 7)):
        calls, _ = enumerate_calls(nodes, dpn, BS, 64)
        want = set()
        for S, D, R, MB in calls:
            for dev in range(1, D - S + 2):
                if BS // (MB * R * dev) >= 1:
                    want.add(BS // (MB * R * dev))
        assert call_shares(calls, BS) == want
