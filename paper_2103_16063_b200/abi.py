"""ctypes mirror of include/pipecut_b200.h (layout only, no library loading)."""

from __future__ import annotations

import ctypes as C

import numpy as np

PC_OK = 0
PC_INFEASIBLE = 1
PC_ERR_INVALID = -1
PC_ERR_BUDGET = -2
PC_ERR_ATOM = -3
PC_ERR_STUCK = -4
PC_ERR_CUDA = -5
PC_ERR_CAPACITY = -6

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)


class PcProblem(C.Structure):
    _fields_ = [
        ("nb", C.c_int32),
        ("n_tasks", C.c_int32),
        ("task_block", _i32p),
        ("task_flops", _f64p),
        ("task_fp_fix", _i64p),
        ("task_fp_ps", _i64p),
        ("task_prod_fix", _i64p),
        ("task_prod_ps", _i64p),
        ("task_dep_off", _i32p),
        ("dep_ob", _i32p),
        ("dep_fix", _i64p),
        ("dep_ps", _i64p),
        ("n_in", C.c_int32),
        ("in_ob", _i32p),
        ("in_cons_off", _i32p),
        ("in_cons", _i32p),
        ("in_fix", _i64p),
        ("in_ps", _i64p),
        ("blk_param", _i64p),
        ("blk_res_fix", _i64p),
        ("blk_res_ps", _i64p),
        ("cut_fixed", _i64p),
        ("cut_ps", _f64p),
        ("flops_per_sec", C.c_double),
        ("bwd_fwd_ratio", C.c_double),
        ("grad_factor", C.c_double),
        ("opt_factor", C.c_double),
        ("checkpointing", C.c_int32),
        ("num_nodes", C.c_int32),
        ("devices_per_node", C.c_int32),
        ("monotone", C.c_int32),
        ("has_cost_table", C.c_int32),
        ("mem_budget", C.c_int64),
        ("bw_intra", C.c_double),
        ("bw_inter", C.c_double),
        ("latency", C.c_double),
    ]


class PcAtoms(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("n_tasks", C.c_int32), ("n_in", C.c_int32), ("n_traffic", C.c_int32),
        ("atom_param", _i64p),
        ("task_atom", _i32p), ("task_flops", _f64p), ("task_fp1", _i64p),
        ("dep_off", _i32p), ("dep_owner", _i32p), ("dep_size", _i64p),
        ("atom_task_off", _i32p), ("atom_tasks", _i32p),
        ("atom_in_off", _i32p), ("atom_in", _i32p),
        ("in_owner", _i32p), ("in_size", _i64p), ("in_atoms_off", _i32p), ("in_atoms", _i32p),
        ("succ_off", _i32p), ("succ", _i32p), ("pred_off", _i32p), ("pred", _i32p),
        ("nbr_off", _i32p), ("nbr", _i32p),
        ("tr_owner", _i32p), ("tr_size", _i64p), ("tr_cons_off", _i32p), ("tr_cons", _i32p),
        ("atom_tr_off", _i32p), ("atom_tr", _i32p),
        ("task_prod1", _i64p),
        ("ov_has", C.POINTER(C.c_uint8)), ("ov_tf", _f64p), ("ov_tb", _f64p), ("ov_act", _i64p),
        ("budget", C.c_int64),
        ("flops_per_sec", C.c_double), ("bwd_fwd_ratio", C.c_double),
        ("grad_factor", C.c_double), ("opt_factor", C.c_double),
    ]


def atoms_struct(fa) -> PcAtoms:
    s = PcAtoms()
    s.n = fa.n
    s.n_tasks = int(fa.task_atom.shape[0])
    s.n_in = int(fa.in_owner.shape[0])
    s.n_traffic = int(fa.tr_owner.shape[0])
    ctypes_of = {np.dtype(np.int32): C.c_int32, np.dtype(np.int64): C.c_int64,
                 np.dtype(np.float64): C.c_double, np.dtype(np.uint8): C.c_uint8}
    for name, _ in PcAtoms._fields_:
        v = getattr(fa, name, None)
        if isinstance(v, np.ndarray):
            setattr(s, name, _ptr(v, ctypes_of[v.dtype]))
    s.budget = fa.budget
    s.flops_per_sec = fa.flops_per_sec
    s.bwd_fwd_ratio = fa.bwd_fwd_ratio
    s.grad_factor = fa.factor_g
    s.opt_factor = fa.factor_o
    return s


class PcCall(C.Structure):
    _fields_ = [("S", C.c_int32), ("D", C.c_int32), ("R", C.c_int32), ("MB", C.c_int32)]


class PcPlan(C.Structure):
    _fields_ = [
        ("cap_stages", C.c_int32),
        ("n_stages", C.c_int32),
        ("lo", _i32p), ("hi", _i32p), ("devices", _i32p),
        ("t_fwd", _f64p), ("t_bwd", _f64p),
        ("mem", _i64p),
        ("S", C.c_int32), ("D", C.c_int32), ("R", C.c_int32), ("MB", C.c_int32),
        ("objective", C.c_double),
        ("iteration_time", C.c_double),
    ]


class PcStats(C.Structure):
    _fields_ = [
        ("visits", C.c_int64),
        ("dp_calls", C.c_int64),
        ("visits_unpruned", C.c_int64),
        ("cells", C.c_int64),
        ("pairs", C.c_int64),
        ("candidates", C.c_int64),
        ("dp_launches", C.c_int64),
        ("kernel_launches", C.c_int64),
        ("device_ms", C.c_double),
        ("span_ms", C.c_double),
        ("post_ms", C.c_double),
    ]


class PcCallResult(C.Structure):
    _fields_ = [
        ("feasible", C.c_int32),
        ("n_stages", C.c_int32),
        ("objective", C.c_double),
        ("iteration_time", C.c_double),
        ("visits", C.c_int64),
        ("visits_unpruned", C.c_int64),
        ("budget_cross", C.c_int64),
    ]


def _ptr(arr, ctype):
    return arr.ctypes.data_as(C.POINTER(ctype))


def problem_struct(fp) -> PcProblem:
    """Build a PcProblem viewing the numpy arrays of a FlatProblem."""
    s = PcProblem()
    s.nb = fp.nb
    s.n_tasks = fp.n_tasks
    s.task_block = _ptr(fp.task_block, C.c_int32)
    s.task_flops = _ptr(fp.task_flops, C.c_double)
    s.task_fp_fix = _ptr(fp.task_fp_fix, C.c_int64)
    s.task_fp_ps = _ptr(fp.task_fp_ps, C.c_int64)
    s.task_prod_fix = _ptr(fp.task_prod_fix, C.c_int64)
    s.task_prod_ps = _ptr(fp.task_prod_ps, C.c_int64)
    s.task_dep_off = _ptr(fp.task_dep_off, C.c_int32)
    s.dep_ob = _ptr(fp.dep_ob, C.c_int32)
    s.dep_fix = _ptr(fp.dep_fix, C.c_int64)
    s.dep_ps = _ptr(fp.dep_ps, C.c_int64)
    s.n_in = int(fp.in_ob.shape[0])
    s.in_ob = _ptr(fp.in_ob, C.c_int32)
    s.in_cons_off = _ptr(fp.in_cons_off, C.c_int32)
    s.in_cons = _ptr(fp.in_cons, C.c_int32)
    s.in_fix = _ptr(fp.in_fix, C.c_int64)
    s.in_ps = _ptr(fp.in_ps, C.c_int64)
    s.blk_param = _ptr(fp.blk_param, C.c_int64)
    s.blk_res_fix = _ptr(fp.blk_res_fix, C.c_int64)
    s.blk_res_ps = _ptr(fp.blk_res_ps, C.c_int64)
    s.cut_fixed = _ptr(fp.cut_fixed, C.c_int64)
    s.cut_ps = _ptr(fp.cut_ps, C.c_double)
    s.flops_per_sec = fp.flops_per_sec
    s.bwd_fwd_ratio = fp.bwd_fwd_ratio
    s.grad_factor = fp.grad_factor
    s.opt_factor = fp.opt_factor
    s.checkpointing = int(fp.checkpointing)
    s.num_nodes = fp.num_nodes
    s.devices_per_node = fp.devices_per_node
    s.monotone = int(fp.monotone)
    s.has_cost_table = int(fp.has_cost_table)
    s.mem_budget = fp.mem_budget
    s.bw_intra = fp.bw_intra
    s.bw_inter = fp.bw_inter
    s.latency = fp.latency
    return s


class PlanBuffers:
    """Caller-owned plan arrays (capacity cap) plus the PcPlan viewing them."""

    def __init__(self, cap: int):
        self.cap = cap
        self.lo = np.zeros(cap, np.int32)
        self.hi = np.zeros(cap, np.int32)
        self.devices = np.zeros(cap, np.int32)
        self.t_fwd = np.zeros(cap, np.float64)
        self.t_bwd = np.zeros(cap, np.float64)
        self.mem = np.zeros(cap, np.int64)
        self.s = PcPlan()
        self.s.cap_stages = cap
        self.s.lo = _ptr(self.lo, C.c_int32)
        self.s.hi = _ptr(self.hi, C.c_int32)
        self.s.devices = _ptr(self.devices, C.c_int32)
        self.s.t_fwd = _ptr(self.t_fwd, C.c_double)
        self.s.t_bwd = _ptr(self.t_bwd, C.c_double)
        self.s.mem = _ptr(self.mem, C.c_int64)

    def stages(self):
        n = self.s.n_stages
        return [(int(self.lo[i]), int(self.hi[i]), int(self.devices[i]),
                 float(self.t_fwd[i]), float(self.t_bwd[i]), int(self.mem[i]))
                for i in range(n)]


def struct_dtype(struct) -> np.dtype:
    """numpy dtype with the exact field offsets of a ctypes Structure
    (pointers as uint64), so arrays of records cross the ABI without a
    Python loop."""
    conv = {C.c_int32: np.int32, C.c_int64: np.int64, C.c_double: np.float64,
            C.c_uint8: np.uint8}
    names, formats, offsets = [], [], []
    for name, ctype in struct._fields_:
        names.append(name)
        formats.append(conv.get(ctype, np.uint64))
        offsets.append(getattr(struct, name).offset)
    return np.dtype({"names": names, "formats": formats, "offsets": offsets,
                     "itemsize": C.sizeof(struct)})


PLAN_DTYPE = struct_dtype(PcPlan)
CALL_RESULT_DTYPE = struct_dtype(PcCallResult)


class PlanView:
    """One call's stages inside a PlanArena (the PlanBuffers field names)."""

    __slots__ = ("lo", "hi", "devices", "t_fwd", "t_bwd", "mem")

    def __init__(self, arena, i):
        a, b = int(arena.off[i]), int(arena.off[i + 1])
        self.lo, self.hi, self.devices = arena.lo[a:b], arena.hi[a:b], arena.devices[a:b]
        self.t_fwd, self.t_bwd, self.mem = arena.t_fwd[a:b], arena.t_bwd[a:b], arena.mem[a:b]


class PlanArena:
    """Plan outputs of a whole batch: one contiguous array per field and a
    PcPlan record per call pointing into it (no per-call Python objects)."""

    def __init__(self, caps):
        caps = np.asarray(caps, np.int64)
        self.n = len(caps)
        self.off = np.zeros(self.n + 1, np.int64)
        np.cumsum(caps, out=self.off[1:])
        tot = max(int(self.off[-1]), 1)
        self.lo = np.zeros(tot, np.int32)
        self.hi = np.zeros(tot, np.int32)
        self.devices = np.zeros(tot, np.int32)
        self.t_fwd = np.zeros(tot, np.float64)
        self.t_bwd = np.zeros(tot, np.float64)
        self.mem = np.zeros(tot, np.int64)
        self.rec = np.zeros(max(self.n, 1), PLAN_DTYPE)
        r, o = self.rec[:self.n], self.off[:-1]
        r["cap_stages"] = caps
        for name in ("lo", "hi", "devices", "t_fwd", "t_bwd", "mem"):
            arr = getattr(self, name)
            r[name] = arr.ctypes.data + arr.itemsize * o

    def ptr(self):
        return self.rec.ctypes.data_as(C.POINTER(PcPlan))

    def __getitem__(self, i):
        return PlanView(self, i)
