"""The DP's objective bound (csrc/dp.cu) changes no result:
plans, objectives, iteration times and the reference's pruned visit counts
are the same with the bound on, off, and deliberately too tight (every call
then leaves its final cell empty and is re-run unbounded).  The bound is a
pure work saver; these tests compare the device against itself AND against
the oracle-pinned C5 goldens, and check that the bound actually engaged."""

import ctypes as C
import json
import os

import pytest

import cases
from paper_2103_16063_b200 import _lib, form_stage
from paper_2103_16063_b200.search import enumerate_calls, run_calls
from paper_2103_16063_b200.stages import bind_problem
from plans import result_doc

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _bound_info(ctx):
    b, r, f = C.c_int64(), C.c_int64(), C.c_int64()
    ctx.check(ctx.lib.pc_bound_info(ctx.h, C.byref(b), C.byref(r), C.byref(f)), "pc_bound_info")
    return b.value, r.value


def _records(batch, BS):
    out = []
    for j in range(len(batch.calls)):
        r = batch.results[j]
        p = batch.plan(j, BS)
        out.append((int(r["visits"]), bool(r["feasible"]),
                    None if p is None else (p.objective.hex(), float(r["iteration_time"]).hex(),
                                            tuple((s.blocks, s.devices, s.t_fwd.hex(),
                                                   s.t_bwd.hex(), s.mem) for s in p.stages))))
    return out


@pytest.fixture
def env(monkeypatch):
    def set_(**kw):
        for k, v in kw.items():
            if v is None:
                monkeypatch.delenv(k, raising=False)
            else:
                monkeypatch.setenv(k, str(v))
    return set_


@pytest.mark.parametrize("nb,D,seed", [(256, 64, 1), (512, 64, 2), (1024, 64, 0)])
def test_bound_on_off_too_tight_agree(gpu, env, nb, D, seed):
    bs = cases.c5_blockset(nb, D, jitter_seed=seed)
    ctx = _lib.context()
    bind_problem(ctx, bs)
    calls, _ = enumerate_calls(max(1, D // 8), min(8, D), 8 * D, nb)
    env(PIPECUT_B200_BOUND_MIN_VISITS=0, PIPECUT_B200_NO_BOUND=1)
    ref = _records(run_calls(ctx, calls, 8 * D, False, True), 8 * D)
    assert _bound_info(ctx) == (0, 0)
    env(PIPECUT_B200_NO_BOUND=None)
    got = _records(run_calls(ctx, calls, 8 * D, False, True), 8 * D)
    bounded, reruns = _bound_info(ctx)
    assert got == ref and bounded > 0 and reruns == 0
    env(PIPECUT_B200_BOUND_SCALE=0.97)                 # every bound below its optimum
    tight = _records(run_calls(ctx, calls, 8 * D, False, True), 8 * D)
    bounded, reruns = _bound_info(ctx)
    assert tight == ref and reruns > 0
    env(PIPECUT_B200_BOUND_SCALE=-1)         # U < 0: reachability only, as for calls
    reach_only = _records(run_calls(ctx, calls, 8 * D, False, True), 8 * D)  # without a greedy plan
    bounded, reruns = _bound_info(ctx)
    assert reach_only == ref and reruns > 0
    env(PIPECUT_B200_BOUND_SCALE=None, PIPECUT_B200_BOUND_WAVES=1)   # partner-plan bounds
    waves = _records(run_calls(ctx, calls, 8 * D, False, True), 8 * D)
    assert waves == ref and _bound_info(ctx)[0] > 0


def test_too_tight_bound_matches_goldens(gpu, env):
    """The re-run path against the oracle: nb = 256 first-level goldens."""
    with open(os.path.join(GOLD, "c5_first_level.json")) as fh:
        first = json.load(fh)
    env(PIPECUT_B200_BOUND_MIN_VISITS=0, PIPECUT_B200_BOUND_SCALE=0.99)
    n = 0
    for key, doc in sorted(first.items()):
        if doc["nb"] != 256:
            continue
        bs = cases.c5_blockset(doc["nb"], doc["D"], jitter_seed=doc["seed"])
        res = form_stage(doc["nodes"], doc["dpn"], doc["batch"], bs)
        a = doc["answer"]
        assert res.stats.visits == doc["visits"] and res.stats.dp_calls == doc["dp_calls"]
        assert res.plan.objective.hex() == a["objective"]
        assert [s.devices for s in res.plan.stages] == a["devices"]
        n += 1
    assert n >= 5


def test_bound_off_for_cost_tables_and_negative_times(gpu, env):
    """No bound where its lower bounds do not hold (cost tables, negative
    times): those searches report zero bounded calls."""
    import random
    import test_gpu_negative_times as neg
    env(PIPECUT_B200_BOUND_MIN_VISITS=0)
    rng = random.Random(5)
    bs, S, D, BS, R, MB, (nodes, dpn) = neg._neg_instance(rng)
    while all(c.t_fwd_sec >= 0 for c in bs.costs):
        bs, S, D, BS, R, MB, (nodes, dpn) = neg._neg_instance(rng)
    from paper_2103_16063_b200 import form_stage_dp
    form_stage_dp(bs, S, D, BS, R, MB)
    assert _bound_info(_lib.context())[0] == 0
    rng = random.Random(6)
    inst = None
    while inst is None:
        inst = neg._neg_cost_table_instance(rng)
    bs, S, D, BS, R, MB, _ = inst
    form_stage_dp(bs, S, D, BS, R, MB)
    assert _bound_info(_lib.context())[0] == 0


def test_bound_engages_on_the_search_path(gpu, env):
    """form_stage at C5 scale runs bounded (default size floor) and equals the
    unbounded search."""
    bs = cases.c5_blockset(1024, 256, jitter_seed=0)
    a = result_doc(form_stage(32, 8, 2048, bs, speculative=True))
    assert _bound_info(_lib.context())[0] > 0
    env(PIPECUT_B200_NO_BOUND=1)
    b = result_doc(form_stage(32, 8, 2048, bs, speculative=True))
    assert a == b


def test_deep_batch_list_kernel_matches_goldens(gpu, env):
    """Batches of many levels take the 10-CTA instantiation of the list
    kernel (DP_DEEP_LEVELS); forced on every bounded batch it gives the
    oracle-pinned first-level answers."""
    with open(os.path.join(GOLD, "c5_first_level.json")) as fh:
        first = json.load(fh)
    env(PIPECUT_B200_BOUND_MIN_VISITS=0, PIPECUT_B200_DEEP_LEVELS=1)
    n = 0
    for key, doc in sorted(first.items()):
        if doc["nb"] != 1024 or doc["seed"] > 1:
            continue
        bs = cases.c5_blockset(doc["nb"], doc["D"], jitter_seed=doc["seed"])
        res = form_stage(doc["nodes"], doc["dpn"], doc["batch"], bs)
        a = doc["answer"]
        assert res.stats.visits == doc["visits"] and res.stats.dp_calls == doc["dp_calls"]
        assert res.plan.objective.hex() == a["objective"]
        assert [s.devices for s in res.plan.stages] == a["devices"]
        n += 1
    assert n >= 4
