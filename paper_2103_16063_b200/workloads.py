"""Synthetic benchmark inputs.

Built with the reference's own generators and host IR (no network, no
checkpoints): enlarged BERT / ResNet task graphs with FLOP-model profiles,
and BERT-layer chains with one block per layer for the C5 scaling sweep.
"""

from __future__ import annotations

import random

from ._host import pipecut as pc

CONFIGS = {
    # name: (generator, args, (nodes, dpn, memory bytes), k, batch)
    "C1": ("bert", (1024, 24, 512, 30522), (1, 8, 2 ** 35), 32, 256),
    "C2": ("bert", (2048, 96, 512, 30522), (4, 8, 32e9), 32, 256),
    "C3": ("resnet", (152, 8), (1, 8, 180e9), 32, 128),
    "C4": ("bert", (4096, 256, 512, 30522), (32, 8, 32e9), 32, 2048),
}


def config_partition(name):
    """(partition, model, k, batch, cluster) of C1-C4."""
    kind, args, (nodes, dpn, mem), k, batch = CONFIGS[name]
    g = pc.gen_bert_like(*args) if kind == "bert" else pc.gen_resnet_like(*args)
    cl = pc.ClusterSpec(nodes, dpn, int(mem), 50e9, 10e9)
    part = pc.build_atomic_subcomponents(g)
    model = pc.CostModel(part.graph, pc.CostModelConfig(), cl)
    return part, model, k, batch, cl


def _val(vid, fixed=0, per_sample=0, param=False):
    return pc.graph.Node(vid, value=pc.graph.ValueInfo(fixed_bytes=fixed,
                                                       bytes_per_sample=per_sample,
                                                       is_param=param))


def bert_layer_chain(nb, hidden=1024, seq=512, jitter_seed=None):
    """C5: one task per BERT-1024 layer (FLOPs, activation, weights of one
    layer of generators.py:66-102), ids t%05d so sorted id order = chain order;
    optional seeded +-10% FLOP jitter."""
    h, s = hidden, seq
    heads = max(1, h // 64)
    flops = 24.0 * s * h * h + 4.0 * s * s * h + 5.0 * s * s * heads + 52.0 * s * h
    rng = random.Random(jitter_seed) if jitter_seed is not None else None
    nodes, edges, prev = [_val("x", per_sample=s * 8)], [], "x"
    for i in range(nb):
        t, v, w = f"t{i:05d}", f"v{i:05d}", f"w{i:05d}"
        f = flops if rng is None else flops * rng.uniform(0.9, 1.1)
        nodes += [pc.graph.Node(t, task=pc.graph.TaskInfo(op="layer", flops_per_sample=f, attrs={})),
                  _val(v, per_sample=s * h * 4),
                  _val(w, fixed=(12 * h * h + 13 * h) * 4, param=True)]
        edges += [(prev, t), (w, t), (t, v)]
        prev = v
    return pc.TaskGraph(nodes, edges, ["x"], [prev])


def c5_cluster(D):
    return max(1, D // 8), min(8, D)


def c5_blockset(nb, D, jitter_seed=None):
    """One block per layer (the tests' blockset_for pattern, k = 10**6)."""
    g = bert_layer_chain(nb, jitter_seed=jitter_seed)
    nodes, dpn = c5_cluster(D)
    cl = pc.ClusterSpec(nodes, dpn, int(32e9), 50e9, 10e9)
    part = pc.build_atomic_subcomponents(g)
    model = pc.CostModel(part.graph, pc.CostModelConfig(), cl)
    return pc.partition_blocks(part, model, k=10 ** 6)


def unpruned_visits(nb, calls):
    """Closed form of the reference's unpruned visit count."""
    tot = 0
    for (S, D, R, MB) in calls:
        A, B = nb - S + 1, D - S + 1
        tot += S * (A * (A + 1) // 2) * (B * (B + 1) // 2)
    return tot
