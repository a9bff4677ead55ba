"""Edge cases of the stage search on the device, checked against the C oracle
(pinned to the reference in test_oracle.py): a single block, zero-share
calls, budgets nothing fits, one device per stage, very wide device ranges,
and capacity limits that must raise rather than truncate."""

import pytest

import cases
from oracle.oracle import OracleProblem, PC_OK
from paper_2103_16063_b200 import brute_force_partition, form_stage, form_stage_dp
from paper_2103_16063_b200._host import pipecut as pc
from paper_2103_16063_b200._lib import DeviceError
from paper_2103_16063_b200.flatten import flatten_blockset

pytestmark = pytest.mark.gpu


def _dp_matches_oracle(bs, S, D, BS, R, MB):
    op = OracleProblem(flatten_blockset(bs))
    for prune in (True, False):
        res = form_stage_dp(bs, S, D, BS, R, MB, pc.SearchOptions(disable_pruning=not prune))
        rc, stages, obj, visits = op.form_stage_dp(S, D, BS, R, MB, disable_pruning=not prune)
        assert res.stats.visits == visits, (S, D, BS, R, MB, prune)
        if rc == PC_OK:
            got = [(s.blocks[0], s.blocks[1], s.devices, s.t_fwd, s.t_bwd, s.mem)
                   for s in res.plan.stages]
            assert got == stages and res.plan.objective == obj
        else:
            assert res.plan is None


def test_single_block(gpu):
    bs = cases.one_block_per_task(cases.chain([2.0], params=[512]), dpn=4)
    assert len(bs) == 1
    for D in (1, 2, 4):
        for R, MB in ((1, 1), (2, 1), (1, 8)):
            _dp_matches_oracle(bs, 1, D, 16, R, MB)
    res = form_stage(1, 4, 16, bs)
    rc, want, visits, calls = OracleProblem(flatten_blockset(bs)).form_stage(1, 4, 16)
    assert res.plan.objective == want["objective"] and res.stats.visits == visits
    assert brute_force_partition(bs, 1, 4, 16, 1, 1).plan.objective == \
        form_stage_dp(bs, 1, 4, 16, 1, 1).plan.objective


def test_zero_share_calls(gpu):
    # MB * R * dev > batch: every (or every wide) stage gets m == 0 (stages.py:224-228)
    bs = cases.one_block_per_task(cases.chain([1.0, 2.0, 1.5, 1.0], sizes=[64] * 4), dpn=6)
    for S, D, BS, R, MB in ((2, 6, 4, 1, 4), (2, 6, 4, 2, 2), (1, 6, 2, 1, 4), (3, 6, 6, 1, 2),
                            (2, 6, 1, 1, 1), (4, 6, 8, 2, 1)):
        _dp_matches_oracle(bs, S, D, BS, R, MB)


def test_budget_nothing_fits(gpu):
    g = cases.chain([1.0, 1.0, 1.0], sizes=[4096] * 3, params=[1 << 20] * 3)
    for mem in (1 << 22, 5 << 20, 9 << 20):
        try:
            bs = cases.one_block_per_task(g, mem=mem, dpn=4, ckpt=True)
        except pc.InfeasibleAtom:
            continue
        for S in (1, 2, 3):
            _dp_matches_oracle(bs, S, 4, 64, 1, 2)
            _dp_matches_oracle(bs, S, 4, 64, 2, 8)


def test_one_device_per_stage_and_wide_ranges(gpu):
    bs = cases.c5_blockset(12, 8, jitter_seed=4)
    for S in (1, 6, 8):
        _dp_matches_oracle(bs, S, S, 8 * S, 1, 1)           # D == S: one device each
    wide = cases.c5_blockset(6, 512, jitter_seed=5)
    for S, D in ((2, 300), (3, 512), (6, 512)):
        _dp_matches_oracle(wide, S, D, 8 * D, 1, 4)


def test_capacity_limits_raise(gpu):
    bs = cases.c5_blockset(4, 8)
    with pytest.raises(DeviceError):
        form_stage_dp(bs, 2, 4096, 8 * 4096, 1, 1)           # D beyond the packed key range


def test_concurrent_callers(gpu):
    """Threads sharing the process's context get the sequential results (the
    drop-ins serialise on the library lock; SURVEY.md §8b threading)."""
    import random
    import threading

    from plans import result_doc

    rng = random.Random(11)
    inst = [cases.stages_random_instance(rng) for _ in range(8)]
    want = [result_doc(form_stage_dp(*x)) for x in inst]
    got = [None] * len(inst)

    def work(i):
        for _ in range(3):
            got[i] = result_doc(form_stage_dp(*inst[i]))

    ts = [threading.Thread(target=work, args=(i,)) for i in range(len(inst))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert got == want


@pytest.mark.parametrize("beta", [3.0, 1.5, 0.7, 4.0])
def test_backward_ratio_not_two(gpu, beta):
    """t_bwd = beta * t_fwd per task (costs.py:138-140): with beta not a power of
    two the span tables store t_bwd (no derivation), and the -fmad=false folds
    must still match the oracle bit for bit (test_costs.py uses beta = 3)."""
    import random

    rng = random.Random(int(beta * 10))
    for _ in range(6):
        n = rng.randint(3, 8)
        g = cases.chain([round(rng.uniform(0.5, 4.0), 3) for _ in range(n)],
                        sizes=[rng.choice([0, 64, 256]) for _ in range(n)],
                        params=[rng.choice([0, 512]) for _ in range(n)])
        cl = pc.ClusterSpec(num_nodes=2, devices_per_node=3, device_memory_bytes=2 ** 40,
                            bw_intra=1e3, bw_inter=5e2, link_latency_sec=0.01)
        part = pc.build_atomic_subcomponents(g)
        cfg = pc.CostModelConfig(device_flops_per_sec=1.0, bwd_fwd_ratio=beta,
                                 checkpointing=rng.random() < 0.5)
        bs = pc.partition_blocks(part, pc.CostModel(part.graph, cfg, cl), k=10 ** 6)
        S = rng.randint(1, min(3, n))
        _dp_matches_oracle(bs, S, 6, 24, 1, 2)
        res = form_stage(2, 3, 24, bs)
        rc, want, visits, calls = OracleProblem(flatten_blockset(bs)).form_stage(2, 3, 24)
        assert res.stats.visits == visits and res.stats.dp_calls == calls
        assert (res.plan is None) == (want is None)
        if want is not None:
            assert res.plan.objective == want["objective"]
