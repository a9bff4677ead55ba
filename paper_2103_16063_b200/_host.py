"""Locate the reference host package (`pipecut`).

The drop-in keeps the reference's graph IR, atom rules, cost-model config and
result dataclasses as its host API: callers hand us a
`pipecut.BlockSet` / `pipecut.AtomicPartition` and get `pipecut.SearchResult`
/ `pipecut.BlockSet` back.  This module only finds that package; it never runs
any of the reference's search or profiling code.

Search order: an already-importable `pipecut`, then the unmodified install in
`<repo>/baseline/_ref` (pip --target of /root/reference/pkg).
"""

from __future__ import annotations

import os
import sys

_REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_CANDIDATES = (
    os.path.join(_REPO, "baseline", "_ref"),
)


def ensure_pipecut():
    try:
        import pipecut  # noqa: F401
        return sys.modules["pipecut"]
    except ImportError:
        pass
    for path in _CANDIDATES:
        if os.path.isdir(os.path.join(path, "pipecut")):
            if path not in sys.path:
                sys.path.insert(0, path)
            import pipecut  # noqa: F401
            return sys.modules["pipecut"]
    raise ImportError(
        "the reference host package `pipecut` is not importable; install it "
        "with `python -m pip install --no-index --no-build-isolation "
        "--target baseline/_ref <copy of /root/reference/pkg>` (DESIGN.md)")


pipecut = ensure_pipecut()
