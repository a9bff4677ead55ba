"""Atomic decomposition drop-in: `build_atomic_subcomponents`
(reference pkg/src/pipecut/atoms.py:164-222) in C++ (csrc/atoms_native.cpp),
SURVEY.md §8f rank 4.  It returns the reference's own AtomicPartition, with
the same (possibly clone-expanded) TaskGraph, atoms and clone map.

Graphs the reference rejects (NoNonConstantTask, DanglingOutput, clone-id
collisions, cycles) go to the reference function, so the caller sees its
exact exception.  Without the native module (not built) the reference
function runs; this is host-side graph preparation, not the GPU path.
"""

from ._host import pipecut as _pc

try:
    from . import _atoms_native
except ImportError:  # pragma: no cover - built by `make` / __graft_entry__.build()
    _atoms_native = None

from pipecut import atoms as _ref_atoms  # noqa: E402  (the reference module, via _host)
from pipecut import graph as _ref_graph  # noqa: E402

_reference = _ref_atoms.build_atomic_subcomponents


def build_atomic_subcomponents(g: "_pc.TaskGraph") -> "_pc.AtomicPartition":
    """atoms.py:164-222, natively; same result and exceptions as the reference."""
    if _atoms_native is not None and type(g) is _ref_graph.TaskGraph:
        try:
            return _atoms_native.build_atomic_subcomponents(
                g, _ref_graph.Node, _ref_graph.TaskGraph, _ref_atoms.Subcomponent,
                _ref_atoms.AtomicPartition)
        except _atoms_native.Fallback:
            pass
    return _reference(g)
