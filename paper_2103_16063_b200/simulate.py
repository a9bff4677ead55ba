"""Drop-in `validate_plan` / `simulate` backed by the device.

Same signatures, results and exceptions as the reference
(pkg/src/pipecut/stages.py:416-492, pkg/src/pipecut/simulate.py:79-179): the
reference's `Violation`, `InvalidPlan`, `Event` and `Schedule` come back.  The
fresh stage records, comm-charged times and objective of `validate_plan`
(`pc_check_plan`) and the whole event timeline, busy time, bubble fraction and
throughput of `simulate` (`pc_simulate`, csrc/sim.cu: k_schedule) are computed
on the GPU; the host only applies the structural checks, compares, and builds
the result objects.
"""

from __future__ import annotations

import ctypes as C
import importlib
import math

import numpy as np

from . import _lib, abi
from ._host import pipecut as _pc
from .stages import bind_overrides, bind_problem

# the package re-exports the function `simulate`, which hides the submodule
_sim = importlib.import_module(_pc.__name__ + ".simulate")
Violation = _pc.graph.Violation
InvalidPlan = _sim.InvalidPlan
Event = _sim.Event
Schedule = _sim.Schedule
PHASES = _sim.PHASES
throughput = _sim.throughput


def _plan_buffers(plan) -> abi.PlanBuffers:
    S = len(plan.stages)
    buf = abi.PlanBuffers(max(S, 1))
    for i, st in enumerate(plan.stages):
        buf.lo[i], buf.hi[i] = st.blocks
        buf.devices[i] = st.devices
        buf.t_fwd[i] = st.t_fwd
        buf.t_bwd[i] = st.t_bwd
        buf.mem[i] = st.mem
    s = buf.s
    s.n_stages = S
    s.S = S
    s.D = plan.devices_total
    s.R = plan.replica_factor
    s.MB = plan.microbatches
    return buf


def _structure(plan, nb):
    """Boundary / device / replica checks (stages.py:418-450)."""
    S = len(plan.stages)
    if S == 0:
        return [Violation("empty-plan", (), "plan has no stages")]
    if plan.microbatches < 1 or plan.replica_factor < 1 or plan.batch_size < 1:
        return [Violation("counts", (), "microbatches, replica factor and "
                                        "batch size must be at least 1")]
    out = []
    end = 0
    for i, st in enumerate(plan.stages):
        lo, hi = st.blocks
        if lo != end or hi <= lo:
            out.append(Violation("boundary", (f"stage {i}",),
                                 f"stage {i} covers [{lo}, {hi}) but the "
                                 f"previous stage ended at {end}"))
        end = hi
        if st.devices < 1:
            out.append(Violation("devices", (f"stage {i}",), f"stage {i} has {st.devices} devices"))
        if st.replicas != st.devices * plan.replica_factor:
            out.append(Violation("replicas", (f"stage {i}",),
                                 f"stage {i} replicas {st.replicas} != devices "
                                 f"x replica factor"))
    if end != nb:
        out.append(Violation("boundary", ("stage last",), f"stages end at block {end}, not {nb}"))
    used = sum(st.devices for st in plan.stages)
    if used != plan.devices_total:
        out.append(Violation("devices", (), f"stage devices sum to {used}, "
                                            f"plan says {plan.devices_total}"))
    return out


def _close(a, b):
    return math.isclose(a, b, rel_tol=1e-9, abs_tol=1e-15)


@_lib.serialized
def validate_plan(plan, blocks):
    """Recheck a plan from scratch; empty list iff it is sound (GPU records)."""
    out = _structure(plan, len(blocks))
    if out:
        return out
    S = len(plan.stages)
    denom = plan.microbatches * plan.replica_factor
    shares = [plan.batch_size // (denom * st.devices) for st in plan.stages]
    ctx = _lib.context()
    flat = bind_problem(ctx, blocks)
    bind_overrides(ctx, flat, {m for m in shares if m >= 1})
    buf = _plan_buffers(plan)
    rtf, rtb, ctf, ctb = (np.zeros(S) for _ in range(4))
    rmem = np.zeros(S, np.int64)
    obj = C.c_double()
    ctx.check(ctx.lib.pc_check_plan(ctx.h, C.byref(buf.s), plan.batch_size, rtf.ctypes.data,
                                    rtb.ctypes.data, rmem.ctypes.data, ctf.ctypes.data,
                                    ctb.ctypes.data, C.byref(obj)), "validate_plan")
    budget = blocks.model.cluster.device_memory_bytes
    for i, st in enumerate(plan.stages):
        if shares[i] == 0:
            out.append(Violation("microbatch", (f"stage {i}",),
                                 f"stage {i} gets zero samples per device"))
            continue
        mem = int(rmem[i])
        if mem > budget:
            out.append(Violation("memory", (f"stage {i}",),
                                 f"stage {i} needs {mem} bytes, device holds {budget}"))
        if mem != st.mem or not (_close(float(rtf[i]), st.t_fwd) and _close(float(rtb[i]), st.t_bwd)):
            out.append(Violation("profile", (f"stage {i}",),
                                 f"stage {i} stored profile does not match a fresh one"))
    if not out and any(m >= 1 for m in shares):
        v = obj.value
        if not _close(v, plan.objective):
            out.append(Violation("objective", (),
                                 f"recomputed objective {v} != stored {plan.objective}"))
    return out


@_lib.serialized
def simulate(plan, blocks):
    """Event-level replay of one iteration of the plan (GPU), as the
    reference's Schedule."""
    violations = validate_plan(plan, blocks)
    if violations:
        raise InvalidPlan(violations)
    ctx = _lib.context()
    bind_problem(ctx, blocks)
    S, MB = len(plan.stages), plan.microbatches
    cap = S * (5 * MB + 1)
    buf = _plan_buffers(plan)
    off = np.zeros(S + 1, np.int32)
    ev_mb = np.zeros(cap, np.int32)
    ev_ph = np.zeros(cap, np.int8)
    ev_st = np.zeros(cap)
    ev_en = np.zeros(cap)
    summary = np.zeros(5)
    ctx.check(ctx.lib.pc_simulate(ctx.h, C.byref(buf.s), plan.batch_size, cap, off.ctypes.data,
                                  ev_mb.ctypes.data, ev_ph.ctypes.data, ev_st.ctypes.data,
                                  ev_en.ctypes.data, summary.ctypes.data), "simulate")
    mbs, phs = ev_mb.tolist(), ev_ph.tolist()
    sts, ens = ev_st.tolist(), ev_en.tolist()
    events = []
    cum = 0
    for s, st in enumerate(plan.stages):
        lane = [(mbs[q], PHASES[phs[q]], sts[q], ens[q]) for q in range(off[s], off[s + 1])]
        for dev in range(cum, cum + st.devices):
            events.extend(Event(device=dev, stage=s, microbatch=mb, phase=ph, start_sec=a,
                                end_sec=b) for mb, ph, a, b in lane)
        cum += st.devices
    return Schedule(events=tuple(events), iteration_time_sec=float(summary[0]),
                    bubble_fraction=float(summary[2]), n_devices=cum,
                    samples_per_sec=float(summary[3]))
