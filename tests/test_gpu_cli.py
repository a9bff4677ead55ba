"""The reference's own CLI (pkg/src/pipecut/cli.py) on the device path:
paper_2103_16063_b200.install() rebinds partition_blocks, form_stage(_dp),
brute_force_partition, validate_plan and simulate, then `pipecut partition
--oracle-check`, `simulate --gantt`, `sweep` and a cost-table partition must
write exactly the files and stdout the unmodified reference wrote
(tests/golden/cli.json, golden/make_cli_golden.py); and the drop-in
simulate/validate_plan must equal the reference on plans of the test
families."""

import dataclasses
import importlib
import json
import os
import random

import pytest

import cases
from golden.make_cli_golden import COMMANDS, OUTPUTS, setup
from paper_2103_16063_b200 import form_stage_dp, install
from paper_2103_16063_b200._host import pipecut as pc
from paper_2103_16063_b200.simulate import InvalidPlan, simulate, validate_plan

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_reference_cli_on_device(gpu, tmp_path, monkeypatch, capsys):
    with open(os.path.join(GOLD, "cli.json")) as fh:
        gold = json.load(fh)
    cli = importlib.import_module(pc.__name__ + ".cli")
    setup(str(tmp_path))
    monkeypatch.chdir(tmp_path)
    restore = install()
    try:
        assert cli.simulate is simulate and cli.validate_plan is validate_plan
        for (name, argv), want in zip(COMMANDS, gold["commands"]):
            capsys.readouterr()
            rc = cli.main(argv)
            out = capsys.readouterr().out
            assert (rc, out) == (want["rc"], want["stdout"]), name
    finally:
        restore()
    for f in OUTPUTS:
        with open(tmp_path / f) as fh:
            assert fh.read() == gold["files"][f], f


def _ref_simulate():
    return importlib.import_module(pc.__name__ + ".simulate").simulate


def test_simulate_equals_reference(gpu):
    """Events, iteration time, bubble and throughput bit for bit on the DP
    plans of the reference's random families (stages.py plans)."""
    ref_sim = _ref_simulate()
    rng = random.Random(1234)
    n = 0
    for _ in range(60):
        bs, S, D, BS, R, MB = cases.stages_random_instance(rng)
        plan = form_stage_dp(bs, S, D, BS, R, MB).plan
        if plan is None:
            continue
        assert validate_plan(plan, bs) == []
        got, want = simulate(plan, bs), ref_sim(plan, bs)
        assert got == want
        n += 1
    assert n > 15
    # C5 chain plans with many stages, replicas and microbatches
    for nb, D, MB in ((48, 16, 8), (64, 32, 16)):
        bs = cases.c5_blockset(nb, D, jitter_seed=2)
        for S in (1, 4, 11):
            plan = form_stage_dp(bs, S, D, 8 * D, 1, MB).plan
            if plan is not None:
                assert simulate(plan, bs) == ref_sim(plan, bs)


def test_validate_plan_flags_like_reference(gpu):
    ref_validate = importlib.import_module(pc.__name__ + ".stages").validate_plan
    rng = random.Random(99)
    checked = 0
    for _ in range(40):
        bs, S, D, BS, R, MB = cases.stages_random_instance(rng)
        plan = form_stage_dp(bs, S, D, BS, R, MB).plan
        if plan is None:
            continue
        st0 = plan.stages[0]
        bad = [
            dataclasses.replace(plan, objective=plan.objective * 2),
            dataclasses.replace(plan, microbatches=plan.batch_size * 4),
            dataclasses.replace(plan, stages=(dataclasses.replace(st0, mem=st0.mem + 1),)
                                + plan.stages[1:]),
            dataclasses.replace(plan, stages=(dataclasses.replace(st0, t_fwd=st0.t_fwd * 1.5),)
                                + plan.stages[1:]),
            dataclasses.replace(plan, devices_total=plan.devices_total + 1),
            dataclasses.replace(plan, stages=plan.stages[:-1]),
            dataclasses.replace(plan, stages=()),
            dataclasses.replace(plan, replica_factor=0),
        ]
        for p in bad:
            got = [dataclasses.astuple(v) for v in validate_plan(p, bs)]
            want = [dataclasses.astuple(v) for v in ref_validate(p, bs)]
            assert got == want
            if want:
                with pytest.raises(InvalidPlan):
                    simulate(p, bs)
            checked += 1
    assert checked > 100
