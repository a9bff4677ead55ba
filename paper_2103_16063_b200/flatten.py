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

import itertools
import weakref
from dataclasses import dataclass, field

import numpy as np

_EXACT = float(2 ** 53)


class UnsupportedGraph(ValueError):
    """The BlockSet uses a construct the flat restatement does not cover."""


def _as_int(x, what: str) -> int:
    if type(x) is int:
        return x
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
    task_prod_fix: np.ndarray   # int64 [T] produced bytes alone (cost-table act_bytes replaces it)
    task_prod_ps: np.ndarray    # int64 [T]
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
    has_cost_table: bool = False
    task_nodes: list = field(default_factory=list, repr=False)   # TaskInfo per task
    cost_config: object = field(default=None, repr=False)        # CostConfig (cost table)
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
    """Native traversal for the common case (csrc/flatten_native.cpp), the
    Python restatement below otherwise (it raises UnsupportedGraph)."""
    if _flatten_native is not None:
        try:
            d = _flatten_native.flatten_blocks(bs)
        except Exception:
            d = None
        if d is not None:
            return _problem_from_arrays(d, bs)
    return _flatten_blockset_py(bs)


def _problem_from_arrays(d, bs) -> FlatProblem:
    model = bs.model
    cfg = model.config
    cl = model.cluster
    tb = d["task_block"]
    monotone = bool(np.all(tb[1:] >= tb[:-1])) if tb.size else True
    return FlatProblem(
        nb=len(bs.block_atoms),
        task_block=tb, task_flops=d["task_flops"],
        task_fp_fix=d["task_fp_fix"], task_fp_ps=d["task_fp_ps"],
        task_prod_fix=d["task_prod_fix"], task_prod_ps=d["task_prod_ps"],
        task_dep_off=d["task_dep_off"], dep_ob=d["dep_ob"],
        dep_fix=d["dep_fix"], dep_ps=d["dep_ps"],
        in_ob=d["in_ob"], in_cons_off=d["in_cons_off"], in_cons=d["in_cons"],
        in_fix=d["in_fix"], in_ps=d["in_ps"],
        blk_param=d["blk_param"], blk_res_fix=d["blk_res_fix"], blk_res_ps=d["blk_res_ps"],
        cut_fixed=_i64([_as_int(x, "cut_fixed") for x in bs._cut_fixed]),
        cut_ps=_f64([float(x) for x in bs._cut_per_sample]),
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
        has_cost_table=cfg.cost_table is not None,
        task_nodes=list(d["task_nodes"]),
        cost_config=cfg,
    )


def _flatten_blockset_py(bs) -> FlatProblem:
    model = bs.model
    cfg = model.config
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
    task_block, task_flops, task_nodes = [], [], []
    fp_fix, fp_ps, dep_off, dep_ob, dep_fix, dep_ps = [], [], [0], [], [], []
    prod_fix, prod_ps = [], []
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
        task_nodes.append(task)
        fp_fix.append(bf)
        fp_ps.append(bp)
        prod_fix.append(pf)
        prod_ps.append(pp)
        dep_off.append(len(dep_ob))

    tb = _i32(task_block)
    monotone = bool(np.all(tb[1:] >= tb[:-1])) if tb.size else True
    cut_fixed = [_as_int(x, "cut_fixed") for x in bs._cut_fixed]
    cut_ps = [float(x) for x in bs._cut_per_sample]
    return FlatProblem(
        nb=nb,
        task_block=tb, task_flops=_f64(task_flops),
        task_fp_fix=_i64(fp_fix), task_fp_ps=_i64(fp_ps),
        task_prod_fix=_i64(prod_fix), task_prod_ps=_i64(prod_ps),
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
        has_cost_table=cfg.cost_table is not None,
        task_nodes=task_nodes,
        cost_config=cfg,
    )


# --------------------------------------------------------------------------- atoms
@dataclass
class FlatAtoms:
    """Atom-level arrays for partition_blocks (blocks.py:73-124): memory of an
    arbitrary atom set G at microbatch 1 with checkpointing, convexity and
    cut traffic.

    mem(G) = int(param(G) * factor + (in(G) + maxfp(G)))  (costs.py:157-159)
      in(G):    values listed in some member atom's input_values that are
                model inputs / unowned or owned outside G (atoms.py:136-138),
                each once;
      maxfp(G): max over member tasks of produced + non-param preds that are
                not inputs of G: an anchor's listed input counts iff its owner
                atom is in G, any other pred always counts (costs.py:150-155).
    """
    n: int
    atom_param: np.ndarray      # int64 [n]
    task_atom: np.ndarray       # int32 [T] sorted node-id order
    task_flops: np.ndarray      # float64 [T]
    task_fp1: np.ndarray        # int64 [T] produced + always-counted preds, at m=1
    task_prod1: np.ndarray      # int64 [T] produced bytes alone at m=1
    dep_off: np.ndarray         # int32 [T+1]
    dep_owner: np.ndarray       # int32 owner atom of an anchor input pred
    dep_size: np.ndarray        # int64 size at m=1
    atom_task_off: np.ndarray   # int32 [n+1]
    atom_tasks: np.ndarray      # int32 task indices, ascending
    atom_in_off: np.ndarray     # int32 [n+1]
    atom_in: np.ndarray         # int32 input-value indices
    in_owner: np.ndarray        # int32 [V] owner atom, -1 model input / unowned
    in_size: np.ndarray         # int64 [V] size at m=1
    in_atoms_off: np.ndarray    # int32 [V+1]
    in_atoms: np.ndarray        # int32 atoms listing the value, ascending
    succ_off: np.ndarray        # int32 [n+1] partition.dependencies() (atoms.py:115-125)
    succ: np.ndarray
    pred_off: np.ndarray
    pred: np.ndarray
    nbr_off: np.ndarray         # int32 [n+1] sorted(succ | pred) (blocks.py:87-88)
    nbr: np.ndarray
    tr_owner: np.ndarray        # int32 [E] value traffic entries (blocks.py:96-102)
    tr_size: np.ndarray         # int64 [E]
    tr_cons_off: np.ndarray     # int32 [E+1]
    tr_cons: np.ndarray         # int32 foreign consumer atoms, ascending
    atom_tr_off: np.ndarray     # int32 [n+1] entries touching each atom
    atom_tr: np.ndarray
    budget: int
    flops_per_sec: float
    bwd_fwd_ratio: float
    factor_g: float
    factor_o: float
    ov_has: np.ndarray = None   # uint8 [T] cost-table entry at m=1 (costs.py:130-148)
    ov_tf: np.ndarray = None    # float64 [T]
    ov_tb: np.ndarray = None    # float64 [T], NaN: bwd_fwd_ratio * t_fwd
    ov_act: np.ndarray = None   # int64 [T], -1: keep produced bytes


def _csr(lists):
    lens = np.fromiter((len(l) for l in lists), dtype=np.int64, count=len(lists))
    off = np.zeros(len(lists) + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    flat = np.fromiter(itertools.chain.from_iterable(lists), dtype=np.int64, count=int(off[-1]))
    return _i32(off), _i32(flat)


def _dependencies(partition, n):
    """AtomicPartition.dependencies() (atoms.py:115-125) with numpy:
    (owner atom, consumer atom) of every produced value, unique, sorted."""
    g = partition.graph
    own, con = [], []
    for vid in g.value_ids():
        if g.producer(vid) is None:
            continue
        o = partition.owner_of_value(vid)
        for c in partition.consumer_atoms(vid):
            if c != o:
                own.append(o)
                con.append(c)
    if not own:
        return []
    key = np.unique(np.asarray(own, np.int64) * n + np.asarray(con, np.int64))
    return list(zip((key // n).tolist(), (key % n).tolist()))


_ATOM_CACHE: dict = {}


def flatten_atoms(partition, model) -> FlatAtoms:
    """Cached per (partition, model) object pair (the reference never mutates
    either); entries are validated by weak references, so a recycled id()
    never returns a stale flattening."""
    hit = _ATOM_CACHE.get(id(partition))
    if hit is not None and hit[0]() is partition and hit[1]() is model:
        return hit[2]
    fa = _flatten_atoms(partition, model)
    if len(_ATOM_CACHE) > 64:
        _ATOM_CACHE.clear()
    _ATOM_CACHE[id(partition)] = (weakref.ref(partition), weakref.ref(model), fa)
    return fa


try:                                         # C++ traversal (csrc/flatten_native.cpp)
    from . import _flatten_native
except ImportError:                          # pragma: no cover - built by build()
    _flatten_native = None


def _flatten_atoms(partition, model) -> FlatAtoms:
    """Native flattening for the common case; anything it does not cover
    (non-integer byte counts, structural violations) runs the Python
    restatement below, which raises the reference-facing errors."""
    if _flatten_native is not None:
        try:
            d = _flatten_native.flatten_atoms(partition, model)
        except Exception:
            d = None
        if d is not None:
            return _atoms_from_arrays(d, model)
    return _flatten_atoms_py(partition, model)


def _atoms_from_arrays(d, model) -> FlatAtoms:
    cfg = model.config
    ov = resolve_overrides(cfg, d["tnodes"], [1]) if cfg.cost_table is not None else None
    return FlatAtoms(
        n=int(d["n"]), atom_param=d["atom_param"], task_atom=d["task_atom"],
        task_flops=d["task_flops"], task_fp1=d["task_fp1"], task_prod1=d["task_prod1"],
        ov_has=None if ov is None else ov[1][0], ov_tf=None if ov is None else ov[2][0],
        ov_tb=None if ov is None else ov[3][0], ov_act=None if ov is None else ov[4][0],
        dep_off=d["dep_off"], dep_owner=d["dep_owner"], dep_size=d["dep_size"],
        atom_task_off=d["atom_task_off"], atom_tasks=d["atom_tasks"],
        atom_in_off=d["atom_in_off"], atom_in=d["atom_in"],
        in_owner=d["in_owner"], in_size=d["in_size"], in_atoms_off=d["in_atoms_off"],
        in_atoms=d["in_atoms"], succ_off=d["succ_off"], succ=d["succ"],
        pred_off=d["pred_off"], pred=d["pred"], nbr_off=d["nbr_off"], nbr=d["nbr"],
        tr_owner=d["tr_owner"], tr_size=d["tr_size"], tr_cons_off=d["tr_cons_off"],
        tr_cons=d["tr_cons"], atom_tr_off=d["atom_tr_off"], atom_tr=d["atom_tr"],
        budget=_as_int(model.cluster.device_memory_bytes, "device_memory_bytes"),
        flops_per_sec=float(cfg.device_flops_per_sec), bwd_fwd_ratio=float(cfg.bwd_fwd_ratio),
        factor_g=float(cfg.grad_factor), factor_o=float(cfg.optimizer_state_factor),
    )


def _flatten_atoms_py(partition, model) -> FlatAtoms:
    cfg = model.config
    g = model.graph
    pg = partition.graph
    n = len(partition.atoms)
    atom_of = atom_node_tables(partition)
    atom_get = atom_of.get
    graph_inputs = g.inputs
    nodes = g.nodes
    succ_of, pred_of = g.succ, g.pred
    sizes = {}                                   # value id -> exact bytes at m = 1

    def size1(info, vid):
        sz = sizes.get(vid)
        if sz is None:
            sz = sizes[vid] = _as_int(info.fixed_bytes, vid) + _as_int(info.bytes_per_sample, vid)
        return sz

    inputs_of_atom = [frozenset(a.input_values) for a in partition.atoms]
    listing = {}
    for a, ins in enumerate(inputs_of_atom):
        for v in ins:
            lst = listing.get(v)
            if lst is None:
                listing[v] = [a]
            else:
                lst.append(a)
    in_ids = sorted(listing)
    in_index = {v: i for i, v in enumerate(in_ids)}
    in_owner, in_size, in_atoms = [], [], []
    for v in in_ids:
        node = nodes[v]
        if not node.is_value:
            raise UnsupportedGraph(f"atom input {v!r} is not a value")
        own = atom_get(v)
        in_owner.append(-1 if (v in graph_inputs or own is None) else own)
        in_size.append(size1(node.value, v))
        in_atoms.append(listing[v])              # ascending: atoms visited in order

    atom_param = [0] * n
    task_atom, task_flops, task_fp1, task_prod1, tnodes = [], [], [], [], []
    dep_owner_l, dep_size_l, dep_off = [], [], [0]
    atom_tasks = [[] for _ in range(n)]
    for nid, node in nodes.items():             # sorted id order (graph.py:90-93)
        a = atom_get(nid)
        if a is None:
            continue
        if node.is_value:
            if node.value.is_param:
                atom_param[a] += _as_int(node.value.fixed_bytes, nid)
            continue
        fp = 0
        for vid in succ_of(nid):
            info = nodes[vid].value
            if info is not None and not info.is_param:
                fp += size1(info, vid)
        task_prod1.append(fp)
        tnodes.append(node.task)
        ins = inputs_of_atom[a]
        for vid in pred_of(nid):
            info = nodes[vid].value
            if info is None or info.is_param:
                continue
            if vid in ins:
                own = in_owner[in_index[vid]]
                if own >= 0:
                    dep_owner_l.append(own)
                    dep_size_l.append(size1(info, vid))
                # model input / unowned: always an input of G, never counted
            else:
                if atom_get(vid) != a:
                    raise UnsupportedGraph(f"task {nid!r} reads {vid!r} across atoms "
                                           f"without listing it as an input")
                fp += size1(info, vid)
        dep_off.append(len(dep_owner_l))
        atom_tasks[a].append(len(task_atom))
        task_atom.append(a)
        task_flops.append(float(node.task.flops_per_sample))
        task_fp1.append(fp)

    succ = [[] for _ in range(n)]
    pred = [[] for _ in range(n)]
    for a, b in _dependencies(partition, n):   # sorted unique pairs
        succ[a].append(b)
        pred[b].append(a)
    nbr = [sorted(set(succ[i]).union(pred[i])) for i in range(n)]

    tr_owner, tr_size, tr_cons = [], [], []
    atom_tr = [[] for _ in range(n)]
    consumer_atoms, owner_of = partition.consumer_atoms, partition.owner_of_value
    for vid in pg.value_ids():                   # blocks.py:96-102
        owner = owner_of(vid)
        foreign = sorted(consumer_atoms(vid) - {owner})
        if foreign:
            e = len(tr_owner)
            tr_owner.append(owner)
            tr_size.append(_as_int(pg.value_size(vid, 1), vid))
            tr_cons.append(foreign)
            for x in sorted({owner, *foreign}):
                atom_tr[x].append(e)

    d_off, d_flat = _i32(dep_off), _i32(dep_owner_l)
    ds = dep_size_l
    at_off, at = _csr(atom_tasks)
    ai_off, ai = _csr([[in_index[v] for v in sorted(ins)] for ins in inputs_of_atom])
    ia_off, ia = _csr(in_atoms)
    s_off, s = _csr(succ)
    p_off, p = _csr(pred)
    n_off, nn = _csr(nbr)
    tc_off, tc = _csr(tr_cons)
    atr_off, atr = _csr(atom_tr)
    ov = resolve_overrides(cfg, tnodes, [1]) if cfg.cost_table is not None else None
    return FlatAtoms(
        n=n, atom_param=_i64(atom_param), task_atom=_i32(task_atom),
        task_flops=_f64(task_flops), task_fp1=_i64(task_fp1), task_prod1=_i64(task_prod1),
        ov_has=None if ov is None else ov[1][0], ov_tf=None if ov is None else ov[2][0],
        ov_tb=None if ov is None else ov[3][0], ov_act=None if ov is None else ov[4][0],
        dep_off=d_off, dep_owner=d_flat, dep_size=_i64(ds),
        atom_task_off=at_off, atom_tasks=at, atom_in_off=ai_off, atom_in=ai,
        in_owner=_i32(in_owner), in_size=_i64(in_size), in_atoms_off=ia_off, in_atoms=ia,
        succ_off=s_off, succ=s, pred_off=p_off, pred=p, nbr_off=n_off, nbr=nn,
        tr_owner=_i32(tr_owner), tr_size=_i64(tr_size), tr_cons_off=tc_off, tr_cons=tc,
        atom_tr_off=atr_off, atom_tr=atr,
        budget=_as_int(model.cluster.device_memory_bytes, "device_memory_bytes"),
        flops_per_sec=float(cfg.device_flops_per_sec), bwd_fwd_ratio=float(cfg.bwd_fwd_ratio),
        factor_g=float(cfg.grad_factor), factor_o=float(cfg.optimizer_state_factor),
    )


# --------------------------------------------------------------------------- cost tables
def _sig_prefixes(tasks):
    """op_signature(task, m) = prefix + str(m) (costs.py:51-54), prefix per task."""
    out = []
    for task in tasks:
        attrs = ",".join(f"{k}={task.attrs[k]}" for k in sorted(task.attrs))
        out.append(f"{task.op}|{attrs}|mb=")
    return out


def resolve_overrides(cfg, tasks, m_values):
    """Measured cost-table entries per (m, task) (costs.py:130-148), dense:
    (m array, has[K,T] u8, tf[K,T], tb[K,T] NaN = ratio*tf, act[K,T] -1 = keep)."""
    table = cfg.cost_table
    ms = sorted({int(m) for m in m_values})
    T = len(tasks)
    has = np.zeros((len(ms), T), np.uint8)
    tf = np.zeros((len(ms), T), np.float64)
    tb = np.full((len(ms), T), np.nan, np.float64)
    act = np.full((len(ms), T), -1, np.int64)
    if table:
        pre = _sig_prefixes(tasks)
        for i, m in enumerate(ms):
            suffix = str(m)
            for t, p in enumerate(pre):
                e = table.get(p + suffix)
                if e is None:
                    continue
                has[i, t] = 1
                tf[i, t] = float(e.t_fwd)
                if e.t_bwd is not None:
                    tb[i, t] = float(e.t_bwd)
                if e.act_bytes is not None:
                    act[i, t] = _as_int(e.act_bytes, "act_bytes")
    return _i64(ms), has, tf, tb, act
