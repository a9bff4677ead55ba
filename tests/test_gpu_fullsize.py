"""Parity at the bench's full size (C5 chain, nb = 1024 blocks, D = 256
devices, batch 2048): calls of that enumeration the C oracle
finishes quickly (S = 1; S = 256, one device per stage, ~35 s in the oracle's
restatement of the reference's scan over all previous cells) are compared
exactly -- plan, objective bits, visits -- and the whole 456-call search must
give the same result single-GPU, speculative or level by level, and through
the sharded path."""

import pytest

import cases
from oracle.oracle import OracleProblem, PC_OK
from paper_2103_16063_b200 import form_stage, form_stage_dp, form_stage_sharded
from paper_2103_16063_b200._host import pipecut as pc
from paper_2103_16063_b200.flatten import flatten_blockset
from plans import result_doc

pytestmark = pytest.mark.gpu

NB, D, BS = 1024, 256, 2048


@pytest.fixture(scope="module")
def workload():
    bs = cases.c5_blockset(NB, D, jitter_seed=0)
    return bs, OracleProblem(flatten_blockset(bs))


@pytest.mark.parametrize("S,R,MB,modes", [(1, 32, 1, (True, False)), (1, 32, 64, (True, False)),
                                          (1, 16, 8, (True, False)), (256, 1, 1, (True,))])
def test_full_size_calls_match_oracle(gpu, workload, S, R, MB, modes):
    bs, op = workload
    Dc = D // R                  # the call's devices: dpn * n with R = N / n (stages.py:389-395)
    for prune in modes:
        res = form_stage_dp(bs, S, Dc, BS, R, MB, pc.SearchOptions(disable_pruning=not prune))
        rc, stages, obj, visits = op.form_stage_dp(S, Dc, BS, R, MB, disable_pruning=not prune)
        assert res.stats.visits == visits
        if rc == PC_OK:
            got = [(s.blocks[0], s.blocks[1], s.devices, s.t_fwd, s.t_bwd, s.mem)
                   for s in res.plan.stages]
            assert got == stages and res.plan.objective == obj
        else:
            assert res.plan is None


def test_full_size_search_consistent(gpu, workload):
    bs, _ = workload
    a = result_doc(form_stage(32, 8, BS, bs))                        # first level, then the rest
    b = result_doc(form_stage(32, 8, BS, bs, speculative=False))     # level by level
    assert result_doc(form_stage(32, 8, BS, bs, speculative=True)) == a   # all at once
    c = result_doc(form_stage_sharded(32, 8, BS, bs))
    d = result_doc(form_stage_sharded(32, 8, BS, bs, speculative=False))
    assert a == b == c == d
    assert a["plan"] is not None and a["dp_calls"] == 56
