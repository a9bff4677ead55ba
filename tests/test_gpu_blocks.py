"""GPU parity of partition_blocks (blocks.py:361-397): exact block_atoms,
block profiles and Subcomponents against the reference's known answers, the
C1-C4 golden fixtures and seeded random layered graphs."""

import json
import os
import random

import pytest

import cases
from paper_2103_16063_b200 import partition_blocks
from paper_2103_16063_b200._host import pipecut as pc

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _same(a, b):
    assert a.block_atoms == b.block_atoms
    assert a.costs == b.costs
    assert a.blocks == b.blocks
    assert a._cut_fixed == b._cut_fixed and a._cut_per_sample == b._cut_per_sample


def test_known_answers(gpu):
    # test_blocks.py:139-225
    p, m = cases.blocks_inputs(cases.weighted_chain([1e9, 1e9, 10e9, 1e9]))
    assert partition_blocks(p, m, 2).block_atoms == ((0, 1), (2, 3))
    assert partition_blocks(p, m, 3).block_atoms == ((0, 1), (2,), (3,))
    p, m = cases.blocks_inputs(cases.weighted_chain([1e9] * 16))
    bs = partition_blocks(p, m, 4)
    assert all(len(g) == 4 for g in bs.block_atoms)
    p, m = cases.blocks_inputs(cases.weighted_chain([1e9, 1e9, 10e9, 1e9], sizes=[1.0, 100.0, 1.0, 1.0]))
    assert partition_blocks(p, m, 2).block_atoms == ((0,), (1, 2, 3))
    p, m = cases.blocks_inputs(cases.param_chain([1e9] * 4, param_bytes=150), mem=1000)
    with pytest.raises(pc.CompactionStuck) as exc:
        partition_blocks(p, m, 2)
    assert exc.value.n_groups == 4 and exc.value.target == 2
    p, m = cases.blocks_inputs(cases.weighted_chain([1e9] * 3, sizes=[64.0, 5000.0, 64.0]), mem=2000)
    with pytest.raises(pc.InfeasibleAtom) as exc:
        partition_blocks(p, m, 2)
    ref = None
    try:
        pc.partition_blocks(p, m, 2)
    except pc.InfeasibleAtom as e:
        ref = e
    assert (exc.value.atom_id, exc.value.mem_bytes, exc.value.budget_bytes) == \
        (ref.atom_id, ref.mem_bytes, ref.budget_bytes)
    with pytest.raises(ValueError):
        partition_blocks(p, m, 0)
    # parallel branches folded by compaction (test_blocks.py:199-225)
    n = [cases._val("x1", per_sample=4.0), cases._task("ta", 1e9), cases._val("va", per_sample=4.0),
         cases._val("x2", per_sample=4.0), cases._task("tb", 1e9), cases._val("vb", per_sample=4.0)]
    e = [("x1", "ta"), ("ta", "va"), ("x2", "tb"), ("tb", "vb")]
    g = pc.TaskGraph(n, e, ["x1", "x2"], ["va", "vb"])
    p, m = cases.blocks_inputs(g)
    assert partition_blocks(p, m, 1).block_atoms == ((0, 1),)
    n2 = n + [cases._val("wa", fixed=160, param=True), cases._val("wb", fixed=160, param=True)]
    g2 = pc.TaskGraph(n2, e + [("wa", "ta"), ("wb", "tb")], ["x1", "x2"], ["va", "vb"])
    p, m = cases.blocks_inputs(g2, mem=1000)
    with pytest.raises(pc.CompactionStuck):
        partition_blocks(p, m, 1)


@pytest.mark.parametrize("seed", [17, 5, 6, 31, 3])
def test_random_layered_graphs_match_reference(gpu, seed):
    rng = random.Random(seed)
    for _ in range(25):
        g = cases.layered_graph(rng)
        k = rng.choice([1, 2, 3, 5, 8])
        p, m = cases.blocks_inputs(g)
        try:
            want = pc.partition_blocks(p, m, k)
        except pc.CompactionStuck as e:
            with pytest.raises(pc.CompactionStuck) as got:
                partition_blocks(p, m, k)
            assert got.value.n_groups == e.n_groups
            continue
        _same(partition_blocks(p, m, k), want)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_configs_match_golden(gpu, name):
    with open(os.path.join(GOLD, "configs.json")) as fh:
        gold = json.load(fh)[name]
    part, model, k, batch, cl = cases.config_partition(name)
    bs = partition_blocks(part, model, k)
    assert [list(g) for g in bs.block_atoms] == gold["block_atoms"]
    assert [[c.t_fwd_sec.hex(), c.t_bwd_sec.hex(), c.mem_bytes] for c in bs.costs] == gold["costs"]


def test_bert_smoke_and_atom_level(gpu):
    g = pc.gen_bert_like(128, 6, 32, 200)
    cl = pc.ClusterSpec(2, 2, 2 ** 40, 50e9, 10e9)
    p = pc.build_atomic_subcomponents(g)
    m = pc.CostModel(p.graph, pc.CostModelConfig(), cl)
    for k in (8, 3, len(p.atoms), 10 ** 6):
        _same(partition_blocks(p, m, k), pc.partition_blocks(p, m, k))


@pytest.mark.parametrize("seed,width,k", [(1, 150, 2), (2, 90, 3), (3, 40, 1)])
def test_fan_graphs_many_levels(gpu, seed, width, k):
    """Few merges per coarsening pass: up to 76 levels, so a refinement move
    rewrites dozens of coarser levels (k_refine's per-level splice)."""
    g = cases.fan_graph(random.Random(seed), width)
    p, m = cases.blocks_inputs(g)
    _same(partition_blocks(p, m, k), pc.partition_blocks(p, m, k))


@pytest.mark.parametrize("cluster", ["1", "2", "16"])
def test_refinement_cluster_sizes(gpu, monkeypatch, cluster):
    """k_refine spreads a window over a thread-block cluster; a smaller
    cluster (one CTA: all sequencing inside one SM) gives the same blocks."""
    monkeypatch.setenv("PIPECUT_B200_REFINE_CLUSTER", cluster)
    with open(os.path.join(GOLD, "configs.json")) as fh:
        gold = json.load(fh)["C1"]
    part, model, k, batch, cl = cases.config_partition("C1")
    assert [list(g) for g in partition_blocks(part, model, k).block_atoms] == gold["block_atoms"]
    rng = random.Random(23)
    for _ in range(10):
        g = cases.layered_graph(rng)
        p, m = cases.blocks_inputs(g)
        try:
            want = pc.partition_blocks(p, m, 3)
        except pc.CompactionStuck:
            continue
        _same(partition_blocks(p, m, 3), want)
    g = cases.fan_graph(random.Random(2), 90)
    p, m = cases.blocks_inputs(g)
    _same(partition_blocks(p, m, 3), pc.partition_blocks(p, m, 3))
