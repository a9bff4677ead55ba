"""The C++ flatteners (csrc/flatten_native.cpp) against the Python
restatements (flatten.py) on CPU: identical arrays on the C1-C4 partitions, the
reference test families, cost-table instances and random layered graphs; inputs
outside the native common case (non-integral byte counts) fall back to the
Python path and raise its error."""

import random

import numpy as np
import pytest

import cases
from paper_2103_16063_b200 import flatten as F
from paper_2103_16063_b200._host import pipecut as pc
from paper_2103_16063_b200.workloads import config_partition

pytestmark = pytest.mark.skipif(F._flatten_native is None, reason="native flattener not built")

_SKIP = ("task_nodes", "cost_config", "keepalive")


def _same(a, b):
    assert a.__dict__.keys() == b.__dict__.keys()
    for k, x in a.__dict__.items():
        if k in _SKIP:
            continue
        y = b.__dict__[k]
        if isinstance(x, np.ndarray) or isinstance(y, np.ndarray):
            assert x is not None and y is not None, k
            assert x.dtype == y.dtype and x.shape == y.shape, k
            assert np.array_equal(x, y, equal_nan=x.dtype.kind == "f"), k
        else:
            assert x == y, k


def _partitions():
    for name in ("C1", "C3"):
        part, model, k, _, _ = config_partition(name)
        yield part, model, k
    rng = random.Random(4242)
    for _ in range(12):
        part, model, k, _ = cases.cost_table_instance(rng)
        yield part, model, k
    rng = random.Random(9)
    for _ in range(12):
        p, m = cases.blocks_inputs(cases.layered_graph(rng))
        yield p, m, 6


def test_native_flatten_atoms_matches_python():
    for part, model, _ in _partitions():
        _same(F._flatten_atoms(part, model), F._flatten_atoms_py(part, model))


def test_native_flatten_blockset_matches_python():
    n = 0
    for part, model, k in _partitions():
        try:
            bs = pc.partition_blocks(part, model, k)
        except (pc.InfeasibleAtom, pc.CompactionStuck):
            continue
        _same(F.flatten_blockset(bs), F._flatten_blockset_py(bs))
        n += 1
    rng = random.Random(1234)
    for _ in range(10):
        bs = cases.stages_random_instance(rng)[0]
        _same(F.flatten_blockset(bs), F._flatten_blockset_py(bs))
        n += 1
    assert n > 20


def test_integral_float_sizes_take_the_native_path():
    g = cases.chain([1.0, 2.0, 3.0], sizes=[64.0, 128.0, 32.0], params=[256, 0, 512])
    part = pc.build_atomic_subcomponents(g)
    model = pc.CostModel(part.graph, pc.CostModelConfig(), pc.ClusterSpec(1, 2, 2 ** 40, 1e9, 1e9))
    F._flatten_native.flatten_atoms(part, model)                  # no fallback
    _same(F._flatten_atoms(part, model), F._flatten_atoms_py(part, model))


def test_non_integral_size_falls_back_and_raises():
    g = cases.chain([1.0, 2.0], sizes=[4.5, 8.0])
    part = pc.build_atomic_subcomponents(g)
    model = pc.CostModel(part.graph, pc.CostModelConfig(), pc.ClusterSpec(1, 2, 2 ** 40, 1e9, 1e9))
    with pytest.raises(Exception):
        F._flatten_native.flatten_atoms(part, model)
    with pytest.raises(F.UnsupportedGraph):
        F._flatten_atoms(part, model)
