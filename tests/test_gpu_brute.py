"""GPU parity of brute_force_partition (stages.py:304-369): the device
enumeration against the reference's own brute force (goldens), its guard and
argument errors, and -- past the reference's guard -- against the DP, which is
exact, and the closed-form pair count."""

import json
import math
import os
import random

import pytest

import cases
from paper_2103_16063_b200 import brute_force_partition, form_stage_dp, partition_blocks
from paper_2103_16063_b200._host import pipecut as pc
from plans import result_doc

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


def test_brute_force_golden_random_families(gpu):
    recs = _load("random_dp.json")
    streams = {}
    n_plans = 0
    for rec in recs:
        key = (rec["family"], rec["seed"])
        if key not in streams:
            streams[key] = random.Random(rec["seed"])
        gen = cases.stages_random_instance if rec["family"] == "stages" else cases.search_instance
        bs, S, D, BS, R, MB = gen(streams[key])
        got = result_doc(brute_force_partition(bs, S, D, BS, R, MB))
        assert got == rec["brute"], (rec["family"], rec["seed"], rec["index"])
        n_plans += got["plan"] is not None
    assert n_plans > 150


def test_brute_force_golden_cost_tables(gpu):
    rng = random.Random(4242)
    n = 0
    for rec in _load("cost_tables.json"):
        part, model, k, (nodes, dpn, S, D, BS, R, MB) = cases.cost_table_instance(rng)
        if "brute" not in rec:
            continue
        bs = partition_blocks(part, model, k)
        assert result_doc(brute_force_partition(bs, S, D, BS, R, MB)) == rec["brute"], rec["index"]
        n += 1
    assert n > 40


def test_brute_force_guards_and_args(gpu):
    # test_stages.py:127-133 and 120-125
    bs = cases.one_block_per_task(cases.chain([1.0] * 13))
    with pytest.raises(pc.stages.TooLarge):
        brute_force_partition(bs, 2, 4, 8, 1, 1)
    small = cases.one_block_per_task(cases.chain([1.0, 1.0]))
    with pytest.raises(pc.stages.TooLarge):
        brute_force_partition(small, 2, 9, 32, 1, 1)
    for args in [(0, 2, 4, 1, 1), (1, 0, 4, 1, 1), (1, 2, 0, 1, 1), (1, 2, 4, 0, 1),
                 (1, 2, 4, 1, 0), (3, 2, 4, 1, 1), (3, 4, 4, 1, 1)]:
        with pytest.raises(pc.InvalidArgs):
            brute_force_partition(small, *args)


@pytest.mark.parametrize("nb,D,S,seed", [(24, 16, 4, 0), (32, 12, 5, 1), (20, 24, 3, 2),
                                         (40, 8, 6, 3)])
def test_brute_force_past_the_guard_equals_dp(gpu, nb, D, S, seed):
    bs = cases.c5_blockset(nb, D, jitter_seed=seed)
    for R, MB in ((1, 1), (1, 4), (2, 2)):
        BS = 8 * D
        bf = brute_force_partition(bs, S, D, BS, R, MB, guard=False)
        dp = form_stage_dp(bs, S, D, BS, R, MB, pc.SearchOptions(disable_pruning=True))
        assert bf.stats.visits == math.comb(nb - 1, S - 1) * math.comb(D - 1, S - 1)
        assert bf.stats.dp_calls == 0
        assert (bf.plan is None) == (dp.plan is None)
        if bf.plan is not None:
            assert bf.plan.objective == dp.plan.objective
            # the brute-force plan is a valid assignment whose own stage costs
            # give back its objective (stages.py:333-349)
            assert sum(st.devices for st in bf.plan.stages) == D
            assert bf.plan.stages[0].blocks[0] == 0 and bf.plan.stages[-1].blocks[1] == nb
