"""ORACLE wrapper — test infrastructure only (see pipecut_oracle.c header).

ctypes binding of oracle/liboracle.so, the plain-C restatement of the
reference's span profile (costs.py:97-160), DP (stages.py:188-279), simulator
(simulate.py:79-165) and form_stage (stages.py:372-413) over the flat arrays
of include/pipecut_b200.h.  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg import this module.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

from paper_2103_16063_b200.abi import (
    PC_ERR_BUDGET,
    PC_OK,
    PcPlan,
    PlanBuffers,
    problem_struct,
)

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB


def load():
    global _lib
    if _lib is None:
        deps = [os.path.join(_HERE, "pipecut_oracle.c"),
                os.path.join(os.path.dirname(_HERE), "include", "pipecut_b200.h")]
        if not os.path.exists(_LIB) or any(os.path.getmtime(_LIB) < os.path.getmtime(d) for d in deps):
            build()
        lib = C.CDLL(_LIB)
        lib.orc_span_record.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int64, C.c_int,
                                        C.POINTER(C.c_double), C.POINTER(C.c_double),
                                        C.POINTER(C.c_int64)]
        lib.orc_span_record.restype = None
        lib.orc_span_record_row.argtypes = lib.orc_span_record.argtypes
        lib.orc_span_record_row.restype = None
        lib.orc_cut_time.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_int64]
        lib.orc_cut_time.restype = C.c_double
        lib.orc_form_stage_dp.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int64, C.c_int,
                                          C.c_int, C.c_int, C.c_int64, C.POINTER(PcPlan),
                                          C.POINTER(C.c_int64)]
        lib.orc_form_stage.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int64, C.c_int,
                                       C.c_int64, C.POINTER(PcPlan), C.POINTER(PcPlan),
                                       C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        lib.orc_simulate.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int]
        lib.orc_simulate.restype = C.c_double
        _lib = lib
    return _lib


class OracleProblem:
    """Keeps the flat arrays alive while the C struct points into them."""

    def __init__(self, flat):
        self.flat = flat
        self.s = problem_struct(flat)
        self.ref = C.byref(self.s)

    def span(self, lo, hi, m, ckpt):
        tf, tb, mem = C.c_double(), C.c_double(), C.c_int64()
        load().orc_span_record(self.ref, lo, hi, m, int(ckpt),
                               C.byref(tf), C.byref(tb), C.byref(mem))
        return tf.value, tb.value, mem.value

    def span_row(self, lo, hi, m, ckpt):
        """The memo-row path (monotone graphs only) of the same record."""
        tf, tb, mem = C.c_double(), C.c_double(), C.c_int64()
        load().orc_span_record_row(self.ref, lo, hi, m, int(ckpt),
                                   C.byref(tf), C.byref(tb), C.byref(mem))
        return tf.value, tb.value, mem.value

    def cut_time(self, cut, m, cum):
        return load().orc_cut_time(self.ref, cut, m, cum)

    def form_stage_dp(self, S, D, BS, R, MB, disable_pruning=False, budget=None):
        """-> (rc, stages, objective, visits); stages = [(lo, hi, dev, tf, tb, mem)]."""
        buf = PlanBuffers(max(S, 1))
        visits = C.c_int64()
        rc = load().orc_form_stage_dp(self.ref, S, D, BS, R, MB, int(disable_pruning),
                                      -1 if budget is None else budget,
                                      C.byref(buf.s), C.byref(visits))
        stages = buf.stages() if rc == PC_OK else None
        return rc, stages, (buf.s.objective if rc == PC_OK else None), visits.value

    def form_stage(self, N, dpn, BS, disable_pruning=False, budget=None):
        """-> (rc, plan_dict|None, visits, dp_calls)."""
        cap = max(self.flat.nb, 1)
        out, scratch = PlanBuffers(cap), PlanBuffers(cap)
        visits, calls = C.c_int64(), C.c_int64()
        rc = load().orc_form_stage(self.ref, N, dpn, BS, int(disable_pruning),
                                   -1 if budget is None else budget,
                                   C.byref(out.s), C.byref(scratch.s),
                                   C.byref(visits), C.byref(calls))
        plan = None
        if rc == PC_OK:
            plan = dict(stages=out.stages(), S=out.s.S, D=out.s.D, R=out.s.R, MB=out.s.MB,
                        objective=out.s.objective, iteration_time=out.s.iteration_time)
        return rc, plan, visits.value, calls.value

    def simulate(self, stages, BS, R, MB):
        import numpy as np
        S = len(stages)
        lo = np.array([s[0] for s in stages], np.int32)
        hi = np.array([s[1] for s in stages], np.int32)
        dev = np.array([s[2] for s in stages], np.int32)
        tf = np.array([s[3] for s in stages], np.float64)
        tb = np.array([s[4] for s in stages], np.float64)
        return load().orc_simulate(self.ref, S, lo.ctypes.data, hi.ctypes.data,
                                   dev.ctypes.data, tf.ctypes.data, tb.ctypes.data,
                                   BS, R, MB)


__all__ = ["OracleProblem", "load", "build", "PC_OK", "PC_ERR_BUDGET"]
