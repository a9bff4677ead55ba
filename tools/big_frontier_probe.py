"""Probe for Pareto frontiers above the 64-entry capacity: chains whose op
kinds have anti-correlated measured forward/backward times (cost tables),
searched unpruned on the device; a capacity error would surface as DeviceError."""
import sys, random, ctypes as C
sys.path[:0] = ['.', 'tests']
import numpy as np
import cases
from oracle.oracle import OracleProblem, load
from paper_2103_16063_b200._host import pipecut as pc
from paper_2103_16063_b200.flatten import flatten_blockset

lib = load()
lib.orc_frontier_hist.argtypes = [C.c_void_p]
best = 0
for seed in range(6):
    rng = random.Random(seed)
    n = 40
    # anti-correlated forward/backward per op kind via a measured table at every share
    kinds = [("fa", {"k": i}) for i in range(12)]
    nodes, edges, prev = [cases._val("x", per_sample=16)], [], "x"
    for i in range(n):
        op, attrs = kinds[rng.randrange(len(kinds))]
        t, v = f"t{i:02d}", f"v{i:02d}"
        nodes.append(cases.Node(t, task=cases.TaskInfo(op=op, flops_per_sample=1.0, attrs=dict(attrs))))
        nodes.append(cases._val(v, per_sample=64))
        edges += [(prev, t), (t, v)]
        prev = v
    g = cases.TaskGraph(nodes, edges, ["x"], [prev])
    BS = 64
    table = {}
    for op, attrs in kinds:
        info = cases.TaskInfo(op=op, flops_per_sample=0.0, attrs=dict(attrs))
        a = rng.uniform(0.1, 10.0)
        for m in range(1, BS + 1):
            table[pc.costs.op_signature(info, m)] = pc.CostTableEntry(microbatch=m, t_fwd=a * m, t_bwd=(10.1 - a) * m * rng.uniform(0.5, 2.0))
    cl = pc.ClusterSpec(num_nodes=2, devices_per_node=4, device_memory_bytes=2 ** 40, bw_intra=1e9, bw_inter=5e8)
    part = pc.build_atomic_subcomponents(g)
    cfg = pc.CostModelConfig(device_flops_per_sec=1.0, cost_table=table)
    bs = pc.partition_blocks(part, pc.CostModel(part.graph, cfg, cl), k=10 ** 6)
    print(len(bs), "blocks", flush=True)
    # the C oracle has no overrides: measure with the device later; here just report
    from paper_2103_16063_b200 import form_stage_dp
    from paper_2103_16063_b200._lib import DeviceError
    for S in (2, 4, 6, 8):
        for MB in (1, 4):
            try:
                r = form_stage_dp(bs, S, 8, BS, 1, MB, pc.SearchOptions(disable_pruning=True))
                print(seed, S, MB, "ok", r.plan is not None, flush=True)
            except DeviceError as e:
                print(seed, S, MB, "CAPACITY", str(e)[:80], flush=True)
