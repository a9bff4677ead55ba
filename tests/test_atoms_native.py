"""The C++ atomic decomposition (csrc/atoms_native.cpp)
against the reference's build_atomic_subcomponents (pkg/src/pipecut/atoms.py:
164-222) on CPU: the same AtomicPartition -- expanded TaskGraph (node order,
edge tuple, adjacency), atoms, clone map and lookup tables -- on the
generators, the reference test families, random graphs with shared constant
support, and the same exception (type and message) on graphs it rejects."""

import random

import pytest

import cases
from paper_2103_16063_b200 import atoms as A
from paper_2103_16063_b200._host import pipecut as pc

# the unmodified reference function (the checker); install() may rebind the name later
_reference = pc.atoms.build_atomic_subcomponents

_val, _task, TaskGraph = cases._val, cases._task, cases.TaskGraph


def _same(p, q):
    assert p.graph == q.graph
    assert list(p.graph.nodes) == list(q.graph.nodes)
    assert p.graph.edges == q.graph.edges
    assert p.graph._succ == q.graph._succ and p.graph._pred == q.graph._pred
    assert p.graph.inputs == q.graph.inputs and p.graph.outputs == q.graph.outputs
    assert p.atoms == q.atoms
    assert list(p.clone_origins.items()) == list(q.clone_origins.items())
    assert p._task_atom == q._task_atom and p._value_owner == q._value_owner
    assert list(p._consumer_atoms.items()) == list(q._consumer_atoms.items())
    assert p.to_json() == q.to_json() and p.dependencies() == q.dependencies()
    if p.atoms:
        idx = list(range(0, len(p.atoms), 2))
        assert p.merged(idx, "M") == q.merged(idx, "M")


def _outcome(fn, g):
    try:
        return fn(g), None
    except Exception as e:  # noqa: BLE001  (the comparison is the point)
        return None, (type(e), str(e))


def _check(g):
    got, gerr = _outcome(A.build_atomic_subcomponents, g)
    want, werr = _outcome(_reference, g)
    assert gerr == werr
    if werr is None:
        _same(got, want)
    return werr is None


def shared_constants(rng, n_tasks=None):
    """Random graph with constant support (params -> constant transforms)
    shared by several non-constant tasks, so atoms get clones."""
    n_tasks = n_tasks or rng.randint(2, 12)
    nodes, edges = [_val("x", per_sample=16)], []
    live, consts = ["x"], []
    for c in range(rng.randint(1, 4)):
        w = f"p{c}"
        nodes.append(_val(w, fixed=64, param=True))
        consts.append(w)
        for d in range(rng.randint(0, 2)):                 # constant transform chain
            t, v = f"p{c}.t{d}", f"p{c}.v{d}"
            nodes += [_task(t, 1.0, "transpose"), _val(v, fixed=64)]
            edges += [(consts[-1], t), (t, v)]
            if rng.random() < 0.3 and len(consts) > 1:
                edges.append((rng.choice(consts[:-1]), t))
            consts.append(v)
    used = set()
    for i in range(n_tasks):
        t, v = f"m{i:02d}", f"y{i:02d}"
        nodes += [_task(t, float(rng.randint(1, 50))), _val(v, per_sample=rng.randint(0, 8) * 4)]
        for src in rng.sample(live, rng.randint(1, min(2, len(live)))):
            edges.append((src, t))
        for src in rng.sample(consts, rng.randint(0, min(2, len(consts)))):
            edges.append((src, t))
            used.add(src)
        edges.append((t, v))
        live.append(v)
    for c in consts:                                        # every constant feeds some atom
        if not any(src == c for src, _ in edges):
            edges.append((c, f"m{rng.randrange(n_tasks):02d}"))
    edges = sorted(set(edges))
    outs = [live[-1]] + ([live[1]] if rng.random() < 0.3 else [])
    inputs = ["x"]
    if rng.random() < 0.3:                                  # a dead model input -> atom 0
        nodes.append(_val("z_dead", per_sample=4))
        inputs.append("z_dead")
    return TaskGraph(nodes, edges, inputs, outs)


def test_generators():
    for g in (pc.gen_bert_like(64, 2, 16, 100), pc.gen_bert_like(128, 6, 32, 500),
              pc.gen_resnet_like(50), pc.gen_resnet_like(101, 2)):
        assert _check(g)
    g = pc.gen_bert_like(64, 2, 16, 100)                      # the native path itself, no fallback
    _same(A._atoms_native.build_atomic_subcomponents(
        g, pc.graph.Node, pc.TaskGraph, pc.atoms.Subcomponent, pc.atoms.AtomicPartition,
        pc.graph.CycleError, pc.atoms.NoNonConstantTask, pc.atoms.DanglingOutput),
        _reference(g))


def test_reference_families():
    for flops in ([1.0], [1.0, 2.0, 3.0]):
        assert _check(cases.chain(flops, params=[64] * len(flops)))
    rng = random.Random(3)
    for _ in range(40):
        assert _check(cases.layered_graph(rng))


def test_shared_constant_support_is_cloned_identically():
    rng = random.Random(17)
    n_cloned = 0
    for _ in range(150):
        g = shared_constants(rng)
        if _check(g):
            n_cloned += bool(A.build_atomic_subcomponents(g).clone_origins)
    assert n_cloned > 40


def test_shared_transpose():
    # the reference test's shape (pkg/tests/test_atoms.py:24-33)
    nodes = [_val("x", per_sample=16), _val("w", fixed=64, param=True), _task("tr"),
             _val("wt", fixed=64), _task("m1", 10.0), _val("y1", per_sample=16),
             _task("m2", 10.0), _val("y2", per_sample=16)]
    edges = [("w", "tr"), ("tr", "wt"), ("x", "m1"), ("wt", "m1"), ("m1", "y1"),
             ("y1", "m2"), ("wt", "m2"), ("m2", "y2")]
    g = TaskGraph(nodes, edges, ["x"], ["y2"])
    assert _check(g)
    assert sorted(A.build_atomic_subcomponents(g).clone_origins) == [
        "tr::c0", "tr::c1", "w::c0", "w::c1", "wt::c0", "wt::c1"]


def test_rejected_graphs_raise_the_reference_errors():
    x, y = _val("x", per_sample=4), _val("y", per_sample=4)
    bad = [
        # no task depends on an input
        TaskGraph([x, _val("w", fixed=4, param=True), _task("t"), y], [("w", "t"), ("t", "y")],
                  ["x"], ["y"]),
        # output produced by a constant task
        TaskGraph([x, _val("w", fixed=4, param=True), _task("c"), _val("k"), _task("t"), y],
                  [("w", "c"), ("c", "k"), ("x", "t"), ("t", "y")], ["x"], ["y", "k"]),
        # output that nothing produces and is not an input
        TaskGraph([x, _task("t"), y, _val("o")], [("x", "t"), ("t", "y")], ["x"], ["y", "o"]),
        # a constant task and a source value feeding no atom
        TaskGraph([x, _val("w", fixed=4, param=True), _task("c"), _val("k"), _task("t"), y,
                   _val("u", fixed=4)],
                  [("w", "c"), ("c", "k"), ("x", "t"), ("t", "y")], ["x"], ["y"]),
        # clone id collides with an existing node
        TaskGraph([x, _val("w", fixed=4, param=True), _val("w::c0", fixed=4), _task("a"),
                   _val("ya"), _task("b"), y],
                  [("x", "a"), ("w", "a"), ("a", "ya"), ("ya", "b"), ("w", "b"), ("b", "y"),
                   ("w::c0", "b")], ["x"], ["y"]),
        # a cycle
        TaskGraph([x, _task("a"), _val("va"), _task("b"), y],
                  [("x", "a"), ("a", "va"), ("va", "b"), ("b", "y"), ("y", "a")], ["x"], ["y"]),
    ]
    # two dangling constant tasks whose topological order differs from id order
    # (the reference reports the first in topological order)
    bad.append(TaskGraph([x, _val("w", fixed=4, param=True), _task("z1"), _val("k1"),
                          _task("a2"), _val("k2"), _task("t"), y],
                         [("w", "z1"), ("z1", "k1"), ("k1", "a2"), ("a2", "k2"), ("x", "t"),
                          ("t", "y")], ["x"], ["y"]))
    # two dangling outputs: the first in sorted id order
    bad.append(TaskGraph([x, _task("t"), y, _val("o2"), _val("o1")], [("x", "t"), ("t", "y")],
                         ["x"], ["y", "o2", "o1"]))
    # a long cycle: the message lists the first 8 stuck ids
    ring = [f"r{i:02d}" for i in range(12)]
    nodes = [x, y, _task("t")]
    edges = [("x", "t"), ("t", "y")]
    for i, r in enumerate(ring):
        nodes += [_task(r), _val(r + "v")]
        edges += [(r, r + "v"), (r + "v", ring[(i + 1) % len(ring)])]
    bad.append(TaskGraph(nodes, edges, ["x"], ["y"]))
    kinds = set()
    for g in bad:
        assert not _check(g)
        kinds.add(_outcome(_reference, g)[1][0].__name__)
    assert kinds == {"NoNonConstantTask", "DanglingOutput", "ValueError", "CycleError"}


def test_missing_native_module_is_a_hard_error(monkeypatch):
    monkeypatch.setattr(A, "_atoms_native", None)
    with pytest.raises(A.NativeUnavailable):
        A.build_atomic_subcomponents(pc.gen_bert_like(64, 2, 16, 100))


def test_input_as_output_and_dead_inputs():
    nodes = [_val("x", per_sample=4), _val("z", per_sample=4), _task("t"), _val("y")]
    g = TaskGraph(nodes, [("x", "t"), ("t", "y")], ["x", "z"], ["y", "x"])
    assert _check(g)
    assert "z" in A.build_atomic_subcomponents(g).atoms[0].node_ids


def test_install_rebinds_the_cli_name():
    import pipecut.cli

    import paper_2103_16063_b200 as pb
    restore = pb.install()
    try:
        assert pipecut.cli.build_atomic_subcomponents is pb.build_atomic_subcomponents
    finally:
        restore()
    assert pipecut.cli.build_atomic_subcomponents is _reference
