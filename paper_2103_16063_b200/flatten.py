"""Flatten a reference `BlockSet` into the plain arrays the C-ABI consumes.

The device never sees Python objects.  This module turns the reference's
host IR (TaskGraph + AtomicPartition + CostModel + BlockSet) into the
`pc_problem` arrays declared in include/pipecut_b200.h, under which the span
profile `CostModel.profile(BlockSet.span(lo, hi), m, ckpt)`
(pkg/src/pipecut/costs.py:97-160, blocks.py:333-343, atoms.py:127-143)
becomes pure integer/fp64 array arithmetic:

* t_fwd / t_bwd: fold over the tasks in sorted node-id order
  (graph.py:90-93, costs.py:120) of ``(f*m)/F`` and ``beta*x``
  (costs.py:137-140); tasks carry their block index.
* input bytes: a value ``v`` that some atom lists in ``input_values`` is in
  the span's input set iff one of those atoms lies in ``[lo, hi)`` and ``v``
  is a model input or its owner block is outside the span (atoms.py:136-138).
  With owner block ``ob(v) <= min(consumer blocks)`` (checked here) that is
  ``ob(v) < lo and cstar(v, lo) < hi``.
* resident bytes: produced bytes of every task plus producer-less,
  non-parameter values owned in the span that are not inputs
  (costs.py:122-128, 142-149) -- additive per block.
* footprint: ``produced_t`` plus non-parameter predecessors that are not span
  inputs (costs.py:150-155); the only span dependence is through
  predecessors owned in a block ``ob``: they count iff ``ob >= lo``.
* parameter bytes: additive per block (costs.py:124-125).
* boundary bytes: ``BlockSet._cut_fixed / _cut_per_sample`` as built by the
  reference itself (blocks.py:308-321).

Every structural assumption above is verified while flattening; a graph that
violates one raises ``UnsupportedGraph`` instead of silently diverging.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

_EXACT = float(2 ** 53)


class UnsupportedGraph(ValueError):
    """The BlockSet uses a construct the flat restatement does not cover."""


def _as_int(x, what: str) -> int:
    if isinstance(x, (int, np.integer)) and not isinstance(x, bool):
        return int(x)
    xf = float(x)
    if not xf.is_integer() or abs(xf) >= _EXACT:
        raise UnsupportedGraph(f"{what} = {x!r} is not an exact integer byte count")
    return int(xf)


@dataclass
class FlatProblem:
    nb: int
    # tasks, sorted node-id order
    task_block: np.ndarray      # int32 [T]
    task_flops: np.ndarray      # float64 [T]
    task_fp_fix: np.ndarray     # int64 [T] produced + span-independent preds (fixed)
    task_fp_ps: np.ndarray      # int64 [T] ... per sample
    task_dep_off: np.ndarray    # int32 [T+1] CSR of span-dependent preds
    dep_ob: np.ndarray          # int32 owner block of the pred value
    dep_fix: np.ndarray         # int64
    dep_ps: np.ndarray          # int64
    # values appearing in some atom's input_values
    in_ob: np.ndarray           # int32 owner block, -1 for model inputs / unowned
    in_cons_off: np.ndarray     # int32 [V+1] CSR of sorted consumer blocks
    in_cons: np.ndarray         # int32
    in_fix: np.ndarray          # int64
    in_ps: np.ndarray           # int64
    # per block additive terms
    blk_param: np.ndarray       # int64 [nb]
    blk_res_fix: np.ndarray     # int64 [nb]
    blk_res_ps: np.ndarray      # int64 [nb]
    # boundary arrays (blocks.py:308-321)
    cut_fixed: np.ndarray       # int64 [nb+1]
    cut_ps: np.ndarray          # float64 [nb+1]
    # CostModelConfig (costs.py:27-40)
    flops_per_sec: float
    bwd_fwd_ratio: float
    grad_factor: float
    opt_factor: float
    checkpointing: bool
    # ClusterSpec (graph.py:176-199)
    num_nodes: int
    devices_per_node: int
    mem_budget: int
    bw_intra: float
    bw_inter: float
    latency: float
    monotone: bool              # task_block non-decreasing along sorted ids
    keepalive: list = field(default_factory=list, repr=False)

    @property
    def n_tasks(self) -> int:
        return int(self.task_block.shape[0])


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _i64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def atom_node_tables(partition):
    """node id -> atom index, and per-atom input sets (atoms.py:259-305)."""
    atom_of = {}
    for idx, atom in enumerate(partition.atoms):
        for nid in atom.node_ids:
            if nid in atom_of:
                raise UnsupportedGraph(f"node {nid!r} belongs to two atoms")
            atom_of[nid] = idx
    return atom_of


def flatten_blockset(bs) -> FlatProblem:
    model = bs.model
    cfg = model.config
    if cfg.cost_table is not None:
        raise UnsupportedGraph("measured cost tables are not supported by the "
                               "device span-cost kernel yet (SURVEY.md §8f)")
    cl = model.cluster
    g = model.graph
    part = bs.partition
    nb = len(bs.block_atoms)
    atom_of = atom_node_tables(part)
    block_of_atom = {}
    for bi, grp in enumerate(bs.block_atoms):
        for a in grp:
            block_of_atom[a] = bi
    n_atoms = len(part.atoms)
    if len(block_of_atom) != n_atoms:
        raise UnsupportedGraph("block_atoms must cover every atom exactly once")

    def blk_of_node(nid):
        a = atom_of.get(nid)
        return -1 if a is None else block_of_atom[a]

    # ---- values that appear in some atom's input_values -----------------
    inputs_of_atom = [frozenset(a.input_values) for a in part.atoms]
    cons: dict[str, set[int]] = {}
    for idx, ins in enumerate(inputs_of_atom):
        for vid in ins:
            cons.setdefault(vid, set()).add(block_of_atom[idx])
    in_ids = sorted(cons)
    in_index = {vid: i for i, vid in enumerate(in_ids)}
    in_ob, in_off, in_cons, in_fix, in_ps = [], [0], [], [], []
    graph_inputs = g.inputs
    for vid in in_ids:
        node = g.nodes[vid]
        if not node.is_value:
            raise UnsupportedGraph(f"atom input {vid!r} is not a value")
        cb = sorted(cons[vid])
        if vid in graph_inputs:
            ob = -1
            own = blk_of_node(vid)
            if own >= 0 and own not in cb:
                raise UnsupportedGraph(f"model input {vid!r} is owned outside its consumers")
        else:
            ob = blk_of_node(vid)
            if ob > cb[0]:
                raise UnsupportedGraph(f"value {vid!r} is consumed before its owner block")
        in_ob.append(ob)
        in_cons.extend(cb)
        in_off.append(len(in_cons))
        in_fix.append(_as_int(node.value.fixed_bytes, f"{vid}.fixed_bytes"))
        in_ps.append(_as_int(node.value.bytes_per_sample, f"{vid}.bytes_per_sample"))

    # ---- per block additive terms and per task footprints -----------------
    blk_param = [0] * nb
    blk_res_fix = [0] * nb
    blk_res_ps = [0] * nb
    task_block, task_flops = [], []
    fp_fix, fp_ps, dep_off, dep_ob, dep_fix, dep_ps = [], [], [0], [], [], []
    for nid, node in g.nodes.items():  # sorted id order (graph.py:90-93)
        b = blk_of_node(nid)
        if b < 0:
            continue
        if node.is_value:
            info = node.value
            if info.is_param:
                blk_param[b] += _as_int(info.fixed_bytes, f"{nid}.fixed_bytes")
            elif g.producer(nid) is None:
                # resident unless it is a span input; a model input owned in
                # the span is an input iff it has a consuming atom at all
                if not (nid in graph_inputs and nid in in_index):
                    blk_res_fix[b] += _as_int(info.fixed_bytes, nid)
                    blk_res_ps[b] += _as_int(info.bytes_per_sample, nid)
            continue
        task = node.task
        a = atom_of[nid]
        pf = pp = 0
        for vid in g.succ(nid):
            info = g.nodes[vid].value
            if info is not None and not info.is_param:
                pf += _as_int(info.fixed_bytes, vid)
                pp += _as_int(info.bytes_per_sample, vid)
        blk_res_fix[b] += pf
        blk_res_ps[b] += pp
        bf, bp = pf, pp
        for vid in g.pred(nid):
            info = g.nodes[vid].value
            if info is None or info.is_param:
                continue
            vf = _as_int(info.fixed_bytes, vid)
            vp = _as_int(info.bytes_per_sample, vid)
            i = in_index.get(vid)
            if i is None:
                bf += vf
                bp += vp
                continue
            ob = in_ob[i]
            if vid not in inputs_of_atom[a]:
                # consumed inside its own atom: never a span input when the
                # task is in the span (owner block == task block)
                if ob != b:
                    raise UnsupportedGraph(f"task {nid!r} reads {vid!r} across atoms "
                                           f"without listing it as an input")
                bf += vf
                bp += vp
                continue
            if ob < 0:
                continue  # model input / unowned: always a span input
            dep_ob.append(ob)
            dep_fix.append(vf)
            dep_ps.append(vp)
        task_block.append(b)
        task_flops.append(float(task.flops_per_sample))
        fp_fix.append(bf)
        fp_ps.append(bp)
        dep_off.append(len(dep_ob))

    tb = _i32(task_block)
    monotone = bool(np.all(tb[1:] >= tb[:-1])) if tb.size else True
    cut_fixed = [_as_int(x, "cut_fixed") for x in bs._cut_fixed]
    cut_ps = [float(x) for x in bs._cut_per_sample]
    return FlatProblem(
        nb=nb,
        task_block=tb, task_flops=_f64(task_flops),
        task_fp_fix=_i64(fp_fix), task_fp_ps=_i64(fp_ps),
        task_dep_off=_i32(dep_off), dep_ob=_i32(dep_ob),
        dep_fix=_i64(dep_fix), dep_ps=_i64(dep_ps),
        in_ob=_i32(in_ob), in_cons_off=_i32(in_off), in_cons=_i32(in_cons),
        in_fix=_i64(in_fix), in_ps=_i64(in_ps),
        blk_param=_i64(blk_param), blk_res_fix=_i64(blk_res_fix),
        blk_res_ps=_i64(blk_res_ps),
        cut_fixed=_i64(cut_fixed), cut_ps=_f64(cut_ps),
        flops_per_sec=float(cfg.device_flops_per_sec),
        bwd_fwd_ratio=float(cfg.bwd_fwd_ratio),
        grad_factor=float(cfg.grad_factor),
        opt_factor=float(cfg.optimizer_state_factor),
        checkpointing=bool(cfg.checkpointing),
        num_nodes=int(cl.num_nodes), devices_per_node=int(cl.devices_per_node),
        mem_budget=_as_int(cl.device_memory_bytes, "device_memory_bytes"),
        bw_intra=float(cl.bw_intra), bw_inter=float(cl.bw_inter),
        latency=float(cl.link_latency_sec),
        monotone=monotone,
    )
