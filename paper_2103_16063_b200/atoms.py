"""Atomic decomposition drop-in: `build_atomic_subcomponents`
(reference pkg/src/pipecut/atoms.py:164-222) in C++ (csrc/atoms_native.cpp),
SURVEY.md §8f rank 4.  It returns the reference's own AtomicPartition, with
the same (possibly clone-expanded) TaskGraph, atoms and clone map, and raises
the reference's own exceptions with its messages on graphs it rejects
(CycleError, NoNonConstantTask, DanglingOutput, the clone-id ValueError).

There is no fallback to the reference function: without the native module
(built by `make` / __graft_entry__.build()) the call raises NativeUnavailable.
"""

from ._host import pipecut as _pc

try:
    from . import _atoms_native
except ImportError:  # pragma: no cover - built by `make` / __graft_entry__.build()
    _atoms_native = None

from pipecut import atoms as _ref_atoms  # noqa: E402  (the reference module, via _host)
from pipecut import graph as _ref_graph  # noqa: E402


class NativeUnavailable(RuntimeError):
    """The C++ atomic decomposition (_atoms_native) is not built."""


def build_atomic_subcomponents(g: "_pc.TaskGraph") -> "_pc.AtomicPartition":
    """atoms.py:164-222, natively; same result and exceptions as the reference."""
    if _atoms_native is None:
        raise NativeUnavailable("paper_2103_16063_b200._atoms_native is not built "
                                "(run __graft_entry__.build())")
    if not isinstance(g, _ref_graph.TaskGraph):
        raise TypeError(f"build_atomic_subcomponents expects a pipecut TaskGraph, got "
                        f"{type(g).__name__}")
    return _atoms_native.build_atomic_subcomponents(
        g, _ref_graph.Node, _ref_graph.TaskGraph, _ref_atoms.Subcomponent,
        _ref_atoms.AtomicPartition, _ref_graph.CycleError, _ref_atoms.NoNonConstantTask,
        _ref_atoms.DanglingOutput)
