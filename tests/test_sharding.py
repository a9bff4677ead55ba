"""CPU: the multi-GPU host logic of form_stage_sharded -- enumeration order,
LPT sharding, record packing, the all-gather exchange (gloo, world_size 2 and 4)
and the reference's selection / budget rule -- against the reference."""

import os
import random
import socket

import numpy as np
import pytest

import cases
from paper_2103_16063_b200._host import pipecut as pc
from paper_2103_16063_b200.search import (_pack, decide, enumerate_calls, exchange, lpt_shard,
                                          select)


def _ref_enumeration(num_nodes, dpn, BS, nb):
    # restates the loop nest of stages.py:389-403 independently
    out = []
    n = 1
    while n <= num_nodes:
        if num_nodes % n == 0:
            D = dpn * n
            R = num_nodes // n
            for S in range(dpn * (n - 1) + 1, D + 1):
                if S <= nb:
                    MB = 1
                    while MB * R <= BS:
                        out.append((S, D, R, MB))
                        MB *= 2
        n *= 2
    return out


@pytest.mark.parametrize("args", [(1, 8, 256, 32), (4, 8, 256, 32), (32, 8, 2048, 32),
                                  (3, 2, 17, 5), (6, 3, 64, 40), (1, 1, 4, 2)])
def test_enumeration_matches_reference_order(args):
    calls, levels = enumerate_calls(*args)
    assert calls == _ref_enumeration(*args)
    assert levels == sorted(levels)


def test_lpt_shard_is_deterministic_and_balanced():
    calls, _ = enumerate_calls(32, 8, 2048, 1024)
    from paper_2103_16063_b200.search import call_weight
    for world in (1, 2, 3, 4, 8):
        a = lpt_shard(1024, calls, world)
        assert a == lpt_shard(1024, calls, world)
        loads = [0] * world
        for c, r in zip(calls, a):
            loads[r] += call_weight(1024, c)
        assert max(loads) <= 1.05 * (sum(loads) / world) + max(call_weight(1024, c) for c in calls)


class _FakeRes:
    def __init__(self, feasible, objective, iteration, visits):
        self.feasible = feasible
        self.objective = objective
        self.iteration_time = iteration
        self.visits = visits

    def __getitem__(self, field):      # run_calls' results are a structured array
        return getattr(self, field)


class _FakeBuf:
    def __init__(self, S, rng):
        self.lo = np.arange(S, dtype=np.int32)
        self.hi = np.arange(1, S + 1, dtype=np.int32)
        self.devices = np.ones(S, np.int32) * rng.randint(1, 3)
        self.t_fwd = np.array([rng.random() for _ in range(S)])
        self.t_bwd = np.array([rng.random() for _ in range(S)])
        self.mem = np.array([rng.randint(1, 2 ** 40) for _ in range(S)], np.int64)


class _FakeBatch:
    def __init__(self, results, bufs):
        self.results = results
        self.bufs = bufs


def _fake_records(calls, seed):
    rng = random.Random(seed)
    recs = []
    for c in calls:
        feas = rng.random() < 0.4
        # ties on iteration time are deliberate: the rank key must break them
        it = rng.choice([1.0, 2.0, 2.0, 3.0]) if feas else float("nan")
        obj = rng.choice([0.5, 0.5, 0.25]) if feas else float("nan")
        recs.append((_FakeRes(int(feas), obj, it, rng.randint(0, 1000)), _FakeBuf(c[0], rng)))
    return recs


def _select_reference_way(calls, levels, recs, budget):
    """The reference's rule written out: level by level, (it, obj, MB) min,
    first wins, budget on the running visits."""
    running = 0
    counted = 0
    for lv in sorted(set(levels)):
        cand = []
        for i, (c, l) in enumerate(zip(calls, levels)):
            if l != lv:
                continue
            counted += 1
            if budget is not None and running + recs[i][0].visits > budget:
                return ("budget", i)
            running += recs[i][0].visits
            if recs[i][0].feasible:
                cand.append(i)
        if cand:
            best = min(cand, key=lambda i: (recs[i][0].iteration_time, recs[i][0].objective,
                                            calls[i][3]))
            return ("plan", best, running, counted)
    return ("plan", None, running, counted)


@pytest.mark.parametrize("seed", range(6))
def test_single_rank_pack_and_decide(seed):
    calls, levels = enumerate_calls(4, 2, 16, 6)
    recs = _fake_records(calls, seed)
    batch = _FakeBatch([r for r, _ in recs], [b for _, b in recs])
    owner = [0] * len(calls)
    rec, plan_w = _pack(6, calls, levels, owner, 0, batch, list(range(len(calls))),
                        max(levels) + 1, max(c[0] for c in calls))
    for budget in (None, 500, 3000):
        want = _select_reference_way(calls, levels, recs, budget)
        got = decide(rec.reshape(1, -1), calls, levels, owner, plan_w, budget, 16)
        if want[0] == "budget":
            assert got[0] == "budget" and got[1] == want[1]
            continue
        res = got[1]
        assert res.stats.visits == want[2] and res.stats.dp_calls == want[3]
        if want[1] is None:
            assert res.plan is None
        else:
            S, D, R, MB = calls[want[1]]
            assert res.plan.microbatches == MB and len(res.plan.stages) == S
            assert res.plan.objective == recs[want[1]][0].objective
            buf = recs[want[1]][1]
            assert [st.t_fwd for st in res.plan.stages] == list(buf.t_fwd)
            assert [st.mem for st in res.plan.stages] == list(buf.mem)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, seed, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        calls, levels = enumerate_calls(4, 2, 16, 6)
        recs = _fake_records(calls, seed)
        owner = lpt_shard(6, calls, world)
        local = [i for i in range(len(calls)) if owner[i] == rank]
        batch = _FakeBatch([recs[i][0] for i in local], [recs[i][1] for i in local])
        rec, plan_w = _pack(6, calls, levels, owner, rank, batch, local, max(levels) + 1,
                            max(c[0] for c in calls))
        allrec = exchange(rec, None, None)
        out = decide(allrec, calls, levels, owner, plan_w, None, 16)
        res = out[1]
        q.put((rank, None if res.plan is None else res.plan.to_json(), res.stats.visits,
               res.stats.dp_calls))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("seed,world", [(0, 2), (3, 2), (5, 4)])
def test_gloo_exchange_matches_single_rank(seed, world):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    calls, levels = enumerate_calls(4, 2, 16, 6)
    recs = _fake_records(calls, seed)
    want = _select_reference_way(calls, levels, recs, None)
    for rank, plan, visits, dp_calls in outs:
        assert visits == want[2] and dp_calls == want[3]
        if want[1] is None:
            assert plan is None
        else:
            assert plan["microbatches"] == calls[want[1]][3]
            assert plan["objective"] == recs[want[1]][0].objective
    assert all(o[1:] == outs[0][1:] for o in outs)


def test_select_matches_reference_form_stage_semantics_live():
    """select() over the reference's own per-call results gives the reference
    form_stage answer (stats included)."""
    bs = cases.one_block_per_task(cases.chain([2.0, 1.0, 1.0, 2.0], sizes=[64] * 4,
                                              params=[128] * 4), nodes=2, dpn=2, bw=(1e6, 5e5))
    calls, levels = enumerate_calls(2, 2, 16, len(bs))
    visits, feas, keys, plans = [], [], [], []
    for i, (S, D, R, MB) in enumerate(calls):
        r = pc.form_stage_dp(bs, S, D, 16, R, MB)
        visits.append(r.stats.visits)
        feas.append(r.plan is not None)
        it = pc.simulate(r.plan, bs).iteration_time_sec if r.plan else 0.0
        keys.append((it, r.plan.objective if r.plan else 0.0, MB, i))
        plans.append(r.plan)
    best, counted, running, cross, _ = select(levels, visits, feas, keys, None)
    ref = pc.form_stage(2, 2, 16, bs)
    assert plans[best] == ref.plan
    assert running == ref.stats.visits and counted == ref.stats.dp_calls


def _level_worker(rank, world, port, seed, heavy, q):
    """Schedule (i) on gloo with run_calls faked: light levels run on every
    rank without an exchange, heavy ones are sharded (search.REPLICATE_BELOW)."""
    import torch.distributed as dist

    from paper_2103_16063_b200 import search
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        calls, levels = enumerate_calls(4, 2, 16, 6)
        recs = _fake_records(calls, seed)
        index = {c: i for i, c in enumerate(calls)}
        exchanges = []

        def fake_run_calls(ctx, sub, bs, prune, want):
            idx = [index[c] for c in sub]
            return _FakeBatch([recs[i][0] for i in idx], [recs[i][1] for i in idx])

        real_exchange = search.exchange

        def counting_exchange(rec, group, dev):
            exchanges.append(1)
            return real_exchange(rec, group, None)

        search.run_calls = fake_run_calls
        search.exchange = counting_exchange
        # heavy levels above the replication threshold, the rest below it
        search.call_weight = lambda nb, c: (int(search.REPLICATE_BELOW)
                                            if levels[calls.index(c)] in heavy else 1)
        w = [1] * len(calls)
        res = search._sharded_by_level(None, calls, levels, max(levels) + 1,
                                       max(c[0] for c in calls), 6, w, world, rank, None, None,
                                       pc.SearchOptions(), 16)
        q.put((rank, None if res.plan is None else res.plan.to_json(), res.stats.visits,
               res.stats.dp_calls, len(exchanges)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("seed,world,heavy", [(0, 2, ()), (3, 2, (1,)), (5, 4, (0, 2)),
                                              (4, 2, (0, 1, 2))])
def test_gloo_level_by_level_replicates_light_levels(seed, world, heavy):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_level_worker, args=(r, world, port, seed, heavy, q))
             for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    calls, levels = enumerate_calls(4, 2, 16, 6)
    recs = _fake_records(calls, seed)
    want = _select_reference_way(calls, levels, recs, None)
    for rank, plan, visits, dp_calls, n_ex in outs:
        assert visits == want[2] and dp_calls == want[3]
        if want[1] is None:
            assert plan is None
        else:
            assert plan["microbatches"] == calls[want[1]][3]
            assert plan["objective"] == recs[want[1]][0].objective
        # one exchange per sharded level evaluated, none for the light ones
        evaluated = sorted({levels[i] for i in range(len(calls))})[:len(set(levels))]
        assert n_ex <= sum(1 for lv in evaluated if lv in heavy)
    assert all(o[1:] == outs[0][1:] for o in outs)
