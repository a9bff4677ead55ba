"""Plan (de)serialisation for golden fixtures: floats as float.hex()."""

from __future__ import annotations


def plan_doc(plan):
    if plan is None:
        return None
    return {
        "stages": [[s.blocks[0], s.blocks[1], s.devices, s.replicas, s.t_fwd.hex(),
                    s.t_bwd.hex(), s.mem] for s in plan.stages],
        "microbatches": plan.microbatches,
        "replica_factor": plan.replica_factor,
        "objective": plan.objective.hex(),
        "batch_size": plan.batch_size,
        "devices_total": plan.devices_total,
    }


def result_doc(res):
    return {"plan": plan_doc(res.plan), "visits": res.stats.visits,
            "dp_calls": res.stats.dp_calls}
