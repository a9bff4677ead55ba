"""B200-native partition-search hot path of RaNNC (arxiv 2103.16063).

Drop-in replacements for the reference package `pipecut`'s hot path:

    partition_blocks (pkg/src/pipecut/blocks.py:361-397)
    form_stage_dp    (pkg/src/pipecut/stages.py:282-291)
    form_stage       (pkg/src/pipecut/stages.py:372-413)
    form_stage_sharded  -- form_stage over the GPUs of a torch.distributed group
    build_atomic_subcomponents (pkg/src/pipecut/atoms.py:164-222) -- host C++

They take and return the reference's own host objects (BlockSet,
SearchOptions, SearchResult, Plan) and run the span-cost tables, the Pareto
stage DP, the visit accounting, the backtrack and the simulated-iteration-time
ranking on an sm_100a GPU.  `install()` rebinds the reference's names so its
CLI and library users pick the GPU path up unchanged.
"""

from ._host import pipecut as _pc  # noqa: F401  (host API package)
from .atoms import build_atomic_subcomponents
from .blocks import partition_blocks
from .search import form_stage_sharded
from .stages import brute_force_partition, form_stage, form_stage_dp

__all__ = ["brute_force_partition", "build_atomic_subcomponents", "form_stage", "form_stage_dp", "form_stage_sharded", "install", "partition_blocks"]


def install():
    """Point the reference's modules at the GPU entry points:
    partition_blocks, form_stage_dp, form_stage, brute_force_partition,
    validate_plan, simulate and build_atomic_subcomponents in pipecut,
    pipecut.atoms, pipecut.blocks, pipecut.stages, pipecut.simulate and
    pipecut.cli (the CLI binds the names at import, cli.py:17-41).  Returns a function that restores the reference's own."""
    import sys

    import pipecut
    import pipecut.atoms
    import pipecut.blocks
    import pipecut.cli
    import pipecut.simulate  # noqa: F401  (the package attribute is the function)
    import pipecut.stages

    from .simulate import simulate, validate_plan

    swaps = (("form_stage", form_stage), ("form_stage_dp", form_stage_dp),
             ("partition_blocks", partition_blocks),
             ("brute_force_partition", brute_force_partition),
             ("validate_plan", validate_plan), ("simulate", simulate),
             ("build_atomic_subcomponents", build_atomic_subcomponents))
    saved = []
    mods = [sys.modules["pipecut" + x] for x in ("", ".atoms", ".stages", ".blocks", ".simulate",
                                                ".cli")]
    for mod in mods:
        for name, fn in swaps:
            if hasattr(mod, name):
                saved.append((mod, name, getattr(mod, name)))
                setattr(mod, name, fn)

    def restore():
        for mod, name, fn in reversed(saved):
            setattr(mod, name, fn)

    return restore
