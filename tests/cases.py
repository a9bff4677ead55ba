"""Problem families shared by the parity tests, goldens and bench.

The random families replay the reference tests' generators with the same RNG
call order so seeds give the same instances:
  * stages_random_instance   <- pkg/tests/test_stages.py:158-183
  * search_instance          <- pkg/tests/test_acceptance.py:92-122
The configs C1-C5 follow SURVEY.md §8(d) / BASELINE.md §2.
"""

from __future__ import annotations

from paper_2103_16063_b200._host import pipecut as pc

Node, TaskGraph, TaskInfo, ValueInfo = pc.graph.Node, pc.TaskGraph, pc.graph.TaskInfo, pc.graph.ValueInfo


def _val(vid, fixed=0, per_sample=0, param=False):
    return Node(vid, value=ValueInfo(fixed_bytes=fixed, bytes_per_sample=per_sample,
                                     is_param=param))


def _task(tid, flops=0.0, op="op"):
    return Node(tid, task=TaskInfo(op=op, flops_per_sample=flops, attrs={}))


def chain(flops, sizes=None, params=None, x_bytes=0):
    """x -> t00 -> v00 -> t01 ...; optional weight per task (test_stages.py:25-42)."""
    n = len(flops)
    sizes = sizes or [0] * n
    params = params or [0] * n
    nodes, edges, prev = [_val("x", per_sample=x_bytes)], [], "x"
    for i in range(n):
        t, v = f"t{i:02d}", f"v{i:02d}"
        nodes.append(_task(t, flops[i]))
        nodes.append(_val(v, per_sample=sizes[i]))
        edges.append((prev, t))
        edges.append((t, v))
        if params[i]:
            w = f"w{i:02d}"
            nodes.append(_val(w, fixed=params[i], param=True))
            edges.append((w, t))
        prev = v
    return TaskGraph(nodes, edges, ["x"], [prev])


def one_block_per_task(graph, *, mem=2 ** 40, nodes=1, dpn=4, bw=(1e12, 1e12),
                       latency=0.0, ckpt=False, flops_per_sec=1.0):
    """BlockSet with one block per atom (test_stages.py:45-54)."""
    cl = pc.ClusterSpec(num_nodes=nodes, devices_per_node=dpn, device_memory_bytes=mem,
                        bw_intra=bw[0], bw_inter=bw[1], link_latency_sec=latency)
    part = pc.build_atomic_subcomponents(graph)
    cfg = pc.CostModelConfig(device_flops_per_sec=flops_per_sec, checkpointing=ckpt)
    return pc.partition_blocks(part, pc.CostModel(part.graph, cfg, cl), k=10 ** 6)


def stages_random_instance(rng):
    """Same RNG sequence as test_stages.random_instance."""
    n = rng.randint(2, 8)
    flops = [round(rng.uniform(0.5, 4.0), 3) for _ in range(n)]
    sizes = [rng.choice([0, 0, 64, 256, 1024]) for _ in range(n)]
    params = [rng.choice([0, 0, 0, 512, 2048]) for _ in range(n)]
    S = rng.randint(1, min(4, n))
    D = rng.randint(S, 6)
    R = rng.choice([1, 2])
    MB = rng.choice([1, 2, 4])
    BS = R * MB * D * rng.randint(1, 3)
    state = sum(p * 4 for p in params)
    acts = sum(sizes) * (BS // (MB * R)) + 64
    budget = rng.choice([2 ** 40, max(int((state + acts) * rng.uniform(0.4, 1.1)), 64)])
    nodes_cfg = rng.choice([(1, 6), (2, 2), (2, 3)])
    graph = chain(flops, sizes, params, x_bytes=rng.choice([0, 16]))
    while True:
        try:
            bs = one_block_per_task(graph, mem=budget, nodes=nodes_cfg[0], dpn=nodes_cfg[1],
                                    bw=(1e3, 5e2), latency=rng.choice([0.0, 0.01]),
                                    ckpt=rng.random() < 0.5)
            break
        except pc.InfeasibleAtom:
            budget *= 4
    return bs, S, D, BS, R, MB


def search_instance(rng):
    """Same RNG sequence as test_acceptance._search_instance."""
    S = rng.randint(1, 4)
    n = rng.randint(max(6, S + 2), 10)
    nodes, dpn = rng.choice([(1, 6), (2, 3), (3, 2)])
    D = rng.randint(min(S + 1, 6), 6)
    R = rng.choice([1, 2])
    MB = rng.choice([1, 2, 4])
    BS = R * MB * D * rng.randint(2, 4)
    flops = [round(rng.uniform(0.5, 4.0), 3) for _ in range(n)]
    sizes = [rng.choice([64, 128, 256, 512, 1024]) for _ in range(n)]
    params = [rng.choice([0, 256, 1024]) for _ in range(n)]
    g = chain(flops, sizes=sizes, params=params)
    need = 4 * sum(params) + sum(sizes) * (BS // (MB * R))
    budget = max(int(need * rng.uniform(0.25, 0.50)), 256)
    for _ in range(4):
        cl = pc.ClusterSpec(num_nodes=nodes, devices_per_node=dpn, device_memory_bytes=budget,
                            bw_intra=1e3, bw_inter=5e2,
                            link_latency_sec=rng.choice([0.0, 0.01]))
        part = pc.build_atomic_subcomponents(g)
        model = pc.CostModel(part.graph, pc.CostModelConfig(device_flops_per_sec=1.0,
                                                            checkpointing=False), cl)
        try:
            return pc.partition_blocks(part, model, 10 ** 6), S, D, BS, R, MB
        except pc.InfeasibleAtom:
            budget *= 4
    raise RuntimeError("could not build a feasible random instance")


# ---------------------------------------------------------------- configs
from paper_2103_16063_b200.workloads import (  # noqa: E402,F401
    CONFIGS, bert_layer_chain, c5_blockset, config_partition)


def layered_graph(rng, n_layers=None, branch=2):
    """Same RNG sequence as pkg/tests/helpers.py:random_layered_graph."""
    n_layers = n_layers or rng.randint(2, 8)
    nodes, edges, produced = [_val("in", per_sample=rng.randint(1, 64) * 4)], [], ["in"]
    for i in range(n_layers):
        for j in range(rng.randint(1, branch)):
            tid = f"t{i:02d}_{j}"
            vid = f"{tid}.out"
            nodes.append(_task(tid, float(rng.randint(1, 1000))))
            nodes.append(_val(vid, per_sample=rng.randint(0, 64) * 4, fixed=rng.randint(0, 16) * 4))
            k = rng.randint(1, min(2, len(produced)))
            for src in rng.sample(produced, k):
                edges.append((src, tid))
            if rng.random() < 0.5:
                wid = f"{tid}.w"
                nodes.append(_val(wid, fixed=rng.randint(1, 256) * 4, param=True))
                edges.append((wid, tid))
            edges.append((tid, vid))
            produced.append(vid)
    return TaskGraph(nodes, edges, ["in"], [produced[-1]])


def fan_graph(rng, width):
    """x -> hub -> width parallel tasks -> sink: a coarsening pass can merge
    only a few pairs, so the level count grows with the width."""
    nodes = [_val("x", per_sample=4.0), _task("hub", float(rng.randint(1, 1000))),
             _val("h", per_sample=rng.randint(1, 64) * 4.0)]
    edges = [("x", "hub"), ("hub", "h")]
    outs = []
    for i in range(width):
        t, v = f"t{i:03d}", f"v{i:03d}"
        nodes += [_task(t, float(rng.randint(1, 1000))), _val(v, per_sample=rng.randint(1, 64) * 4.0)]
        edges += [("h", t), (t, v)]
        outs.append(v)
    nodes += [_task("sink", float(rng.randint(1, 1000))), _val("y", per_sample=4.0)]
    edges += [(v, "sink") for v in outs] + [("sink", "y")]
    return TaskGraph(nodes, edges, ["x"], ["y"])


def weighted_chain(flops_list, sizes=None):
    """pkg/tests/test_blocks.py:31-42."""
    sizes = sizes or [4.0] * len(flops_list)
    nodes, edges, prev = [_val("x", per_sample=4.0)], [], "x"
    for i, (f, s) in enumerate(zip(flops_list, sizes)):
        t, v = f"t{i:02d}", f"v{i:02d}"
        nodes += [_task(t, f), _val(v, per_sample=s)]
        edges += [(prev, t), (t, v)]
        prev = v
    return TaskGraph(nodes, edges, ["x"], [prev])


def param_chain(flops_list, param_bytes):
    """pkg/tests/test_blocks.py:45-56."""
    nodes, edges, prev = [_val("x", per_sample=4.0)], [], "x"
    for i, f in enumerate(flops_list):
        t, v, w = f"t{i:02d}", f"v{i:02d}", f"w{i:02d}"
        nodes += [_task(t, f), _val(v, per_sample=4.0), _val(w, fixed=param_bytes, param=True)]
        edges += [(prev, t), (w, t), (t, v)]
        prev = v
    return TaskGraph(nodes, edges, ["x"], [prev])


def blocks_inputs(g, mem=2 ** 40, flops=1e9):
    """(partition, model) as pkg/tests/test_blocks.py:23-28 builds them."""
    cl = pc.ClusterSpec(num_nodes=2, devices_per_node=2, device_memory_bytes=mem,
                        bw_intra=50e9, bw_inter=10e9)
    p = pc.build_atomic_subcomponents(g)
    return p, pc.CostModel(p.graph, pc.CostModelConfig(device_flops_per_sec=flops), cl)


# ---------------------------------------------------------------- measured cost tables
TYPED_OPS = (("matmul", {"h": 1024}), ("matmul", {"h": 4096}), ("gelu", {}),
             ("layernorm", {"eps": 1e-05, "h": 1024}))


def typed_chain(rng, n):
    """Chain whose tasks share a few op signatures, so table entries hit
    several tasks at once (op_signature, costs.py:51-54)."""
    nodes, edges, prev = [_val("x", per_sample=rng.choice([0, 16]))], [], "x"
    for i in range(n):
        op, attrs = rng.choice(TYPED_OPS)
        t, v = f"t{i:02d}", f"v{i:02d}"
        nodes.append(Node(t, task=TaskInfo(op=op, flops_per_sample=round(rng.uniform(0.5, 4.0), 3),
                                           attrs=dict(attrs))))
        nodes.append(_val(v, per_sample=rng.choice([0, 64, 256, 1024])))
        edges += [(prev, t), (t, v)]
        p = rng.choice([0, 0, 512, 2048])
        if p:
            w = f"w{i:02d}"
            nodes.append(_val(w, fixed=p, param=True))
            edges.append((w, t))
        prev = v
    return TaskGraph(nodes, edges, ["x"], [prev])


def random_cost_table(rng, sigs, shares):
    """Entries for a random subset of (signature, microbatch); t_bwd and
    act_bytes optional as load_cost_table allows (costs.py:57-80)."""
    table = {}
    for op, attrs in sigs:
        info = TaskInfo(op=op, flops_per_sample=0.0, attrs=dict(attrs))
        for m in shares:
            if rng.random() < 0.5:
                continue
            tb = None if rng.random() < 0.5 else round(rng.uniform(0.0, 8.0), 4)
            act = None if rng.random() < 0.5 else rng.choice([0, 7, 300, 4096, 65536])
            table[pc.costs.op_signature(info, m)] = pc.CostTableEntry(
                microbatch=m, t_fwd=round(rng.uniform(0.0, 6.0), 4), t_bwd=tb, act_bytes=act)
    return table


def cost_table_instance(rng):
    """Typed chain + random measured table; one block per atom (stage DP
    cases) and a coarsened BlockSet (partition_blocks with overrides)."""
    n = rng.randint(3, 10)
    g = typed_chain(rng, n)
    S = rng.randint(1, min(4, n))
    nodes, dpn = rng.choice([(1, 4), (2, 2), (1, 6)])
    D = rng.randint(S, nodes * dpn)
    R = rng.choice([1, 2])
    MB = rng.choice([1, 2, 4])
    BS = R * MB * D * rng.randint(1, 3)
    table = random_cost_table(rng, TYPED_OPS, range(1, BS + 1))
    ckpt = rng.random() < 0.5
    budget = rng.choice([2 ** 40, rng.randint(4096, 65536)])
    k = rng.choice([10 ** 6, rng.randint(1, n)])
    lat = rng.choice([0.0, 0.01])
    cl = pc.ClusterSpec(num_nodes=nodes, devices_per_node=dpn, device_memory_bytes=budget,
                        bw_intra=1e3, bw_inter=5e2, link_latency_sec=lat)
    part = pc.build_atomic_subcomponents(g)
    cfg = pc.CostModelConfig(device_flops_per_sec=1.0, checkpointing=ckpt, cost_table=table)
    return part, pc.CostModel(part.graph, cfg, cl), k, (nodes, dpn, S, D, BS, R, MB)
