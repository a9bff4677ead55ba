"""ctypes binding of libpipecut_b200.so (the C-ABI of include/pipecut_b200.h).

There is deliberately no CPU fallback: if the library or a B200 is missing,
every entry point raises ``DeviceUnavailable``.
"""

from __future__ import annotations

import ctypes as C
import functools
import threading
import os
import threading

from . import abi
from .abi import PcCall, PcCallResult, PcPlan, PcProblem, PcStats

_HERE = os.path.dirname(os.path.abspath(__file__))
# PIPECUT_B200_LIB: an alternative build of the same library (A/B timing)
LIB_PATH = os.environ.get("PIPECUT_B200_LIB") or os.path.join(_HERE, "libpipecut_b200.so")


class DeviceUnavailable(RuntimeError):
    """The CUDA library could not be loaded or no sm_100 device is usable."""


class DeviceError(RuntimeError):
    """A CUDA error or capacity limit inside the library."""


_lib = None
_lock = threading.Lock()


def load():
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise DeviceUnavailable(
                f"{LIB_PATH} is missing; build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        try:
            lib = C.CDLL(LIB_PATH)
        except OSError as exc:
            raise DeviceUnavailable(f"cannot load {LIB_PATH}: {exc}") from exc
        P = C.POINTER
        lib.pc_ctx_create.argtypes = [C.c_int, P(C.c_void_p)]
        lib.pc_ctx_destroy.argtypes = [C.c_void_p]
        lib.pc_ctx_destroy.restype = None
        lib.pc_last_error.argtypes = [C.c_void_p]
        lib.pc_last_error.restype = C.c_char_p
        lib.pc_device_info.argtypes = [C.c_void_p, P(C.c_int32), P(C.c_int32), P(C.c_int32)]
        lib.pc_set_problem.argtypes = [C.c_void_p, P(PcProblem)]
        lib.pc_profile_spans.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_void_p]
        lib.pc_form_stage_dp.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.c_int32,
                                         C.c_int32, C.c_int32, C.c_int64, P(PcPlan), P(PcStats)]
        lib.pc_run_calls.argtypes = [C.c_void_p, C.c_int32, P(PcCall), C.c_int64, C.c_int32,
                                     C.c_int32, P(PcCallResult), P(PcPlan), P(PcStats)]
        lib.pc_last_crossing.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.c_int64,
                                         P(C.c_int64)]
        lib.pc_form_stage.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.c_int32,
                                      C.c_int64, C.c_int32, P(PcPlan), P(PcStats)]
        lib.pc_partition_blocks.argtypes = [C.c_void_p, P(abi.PcAtoms), C.c_int32, P(C.c_int32),
                                            C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_void_p, C.c_void_p]
        lib.pc_set_overrides.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_void_p]
        lib.pc_brute_force.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.c_int32,
                                       C.c_int32, P(PcPlan), P(PcStats)]
        lib.pc_check_plan.argtypes = [C.c_void_p, P(PcPlan), C.c_int64, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_void_p, P(C.c_double)]
        lib.pc_simulate.argtypes = [C.c_void_p, P(PcPlan), C.c_int64, C.c_int32, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        lib.pc_call_weights.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int64, C.c_void_p]
        lib.pc_reset_cache.argtypes = [C.c_void_p]
        lib.pc_timer_start.argtypes = [C.c_void_p]
        lib.pc_timer_stop.argtypes = [C.c_void_p, P(C.c_double)]
        lib.pc_measure_fp64_peak.argtypes = [C.c_void_p, P(C.c_double)]
        lib.pc_measure_dadd_peak.argtypes = [C.c_void_p, P(C.c_double)]
        lib.pc_bound_info.argtypes = [C.c_void_p, P(C.c_int64), P(C.c_int64), P(C.c_int64)]
        for name in ("pc_ctx_create", "pc_device_info", "pc_set_problem", "pc_profile_spans",
                     "pc_form_stage_dp", "pc_run_calls", "pc_last_crossing", "pc_form_stage",
                     "pc_reset_cache", "pc_timer_start", "pc_timer_stop",
                     "pc_measure_fp64_peak", "pc_measure_dadd_peak", "pc_bound_info",
                     "pc_partition_blocks",
                     "pc_set_overrides", "pc_brute_force", "pc_check_plan", "pc_simulate",
                     "pc_call_weights"):
            getattr(lib, name).restype = C.c_int
        _lib = lib
        return lib


EXPORTS = ("pc_ctx_create", "pc_ctx_destroy", "pc_last_error", "pc_device_info",
           "pc_set_problem", "pc_profile_spans", "pc_form_stage_dp", "pc_run_calls",
           "pc_last_crossing", "pc_form_stage", "pc_reset_cache", "pc_timer_start",
           "pc_timer_stop", "pc_measure_fp64_peak", "pc_measure_dadd_peak", "pc_bound_info",
           "pc_partition_blocks",
           "pc_set_overrides", "pc_brute_force", "pc_check_plan", "pc_simulate", "pc_call_weights")


class Context:
    """One library context (device memory, stream, key-table cache) per device."""

    def __init__(self, device: int = 0):
        lib = load()
        h = C.c_void_p()
        rc = lib.pc_ctx_create(device, C.byref(h))
        if rc != abi.PC_OK or not h.value:
            raise DeviceUnavailable(f"no usable sm_100 device {device} for pipecut_b200 (rc={rc})")
        self.lib = lib
        self.h = h
        self.device = device
        self.problem_owner = None   # weakref to the BlockSet currently uploaded
        self.problem_flat = None
        self.problem_shares = frozenset()   # cost-table shares resolved on device

    def error(self) -> str:
        return self.lib.pc_last_error(self.h).decode(errors="replace")

    def check(self, rc: int, what: str):
        if rc in (abi.PC_OK, abi.PC_INFEASIBLE, abi.PC_ERR_BUDGET):
            return rc
        if rc == abi.PC_ERR_INVALID:
            raise ValueError(f"{what}: {self.error()}")
        raise DeviceError(f"{what} failed (rc={rc}): {self.error()}")

    def close(self):
        if self.h:
            self.lib.pc_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_contexts: dict[int, Context] = {}


# The library is not re-entrant and a context (device memory, stream, key
# cache) is shared by every thread of the process: the drop-ins serialise on
# one re-entrant lock (the reference itself is single-threaded).
_call_lock = threading.RLock()


def serialized(fn):
    """Run a drop-in entry point under the process-wide library lock."""
    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        with _call_lock:
            return fn(*args, **kwargs)
    return wrapper


def context(device: int | None = None) -> Context:
    if device is None:
        device = int(os.environ.get("PIPECUT_B200_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    with _call_lock:
        ctx = _contexts.get(device)
        if ctx is None:
            ctx = Context(device)
            _contexts[device] = ctx
        return ctx
