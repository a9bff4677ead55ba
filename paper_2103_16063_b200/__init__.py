"""B200-native partition-search hot path of RaNNC (arxiv 2103.16063).

Drop-in replacements for the reference package `pipecut`'s hot path:

    form_stage_dp   (pkg/src/pipecut/stages.py:282-291)
    form_stage      (pkg/src/pipecut/stages.py:372-413)

They take and return the reference's own host objects (BlockSet,
SearchOptions, SearchResult, Plan) and run the span-cost tables, the Pareto
stage DP, the visit accounting, the backtrack and the simulated-iteration-time
ranking on an sm_100a GPU.  `install()` rebinds the reference's names so its
CLI and library users pick the GPU path up unchanged.
"""

from ._host import pipecut as _pc  # noqa: F401  (host API package)
from .stages import form_stage, form_stage_dp

__all__ = ["form_stage", "form_stage_dp", "install"]


def install():
    """Point the reference's modules at the GPU entry points."""
    import pipecut
    import pipecut.cli
    import pipecut.stages

    for mod in (pipecut, pipecut.stages, pipecut.cli):
        if hasattr(mod, "form_stage"):
            mod.form_stage = form_stage
        if hasattr(mod, "form_stage_dp"):
            mod.form_stage_dp = form_stage_dp
