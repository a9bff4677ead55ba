"""Generate the golden fixtures from the REFERENCE itself.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
Imports the unmodified reference package from /root/reference/pkg/src and
records its outputs; the GPU box has no /root/reference, so the parity tests
read these committed JSON files instead.
"""

import json
import os
import random
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import pipecut  # noqa: E402

assert pipecut.__file__.startswith("/root/reference"), pipecut.__file__

import cases  # noqa: E402
from plans import result_doc  # noqa: E402
from paper_2103_16063_b200.search import enumerate_calls  # noqa: E402

pc = pipecut


def dump(name, doc):
    with open(os.path.join(HERE, name), "w") as fh:
        json.dump(doc, fh, indent=0, sort_keys=True)
        fh.write("\n")


def random_families():
    out = []
    fams = [("stages", 1234, 60), ("stages", 99, 60), ("stages", 5, 10), ("stages", 7, 25),
            ("search", 777, 120)]
    for fam, seed, count in fams:
        rng = random.Random(seed)
        gen = cases.stages_random_instance if fam == "stages" else cases.search_instance
        for i in range(count):
            bs, S, D, BS, R, MB = gen(rng)
            rec = {"family": fam, "seed": seed, "index": i, "args": [S, D, BS, R, MB]}
            for prune in (True, False):
                res = pc.form_stage_dp(bs, S, D, BS, R, MB,
                                       pc.SearchOptions(disable_pruning=not prune))
                rec["pruned" if prune else "unpruned"] = result_doc(res)
            rec["brute"] = result_doc(pc.brute_force_partition(bs, S, D, BS, R, MB))
            out.append(rec)
    dump("random_dp.json", out)


def configs():
    out = {}
    for name in ("C1", "C2", "C3", "C4"):
        part, model, k, batch, cl = cases.config_partition(name)
        t0 = time.time()
        bs = pc.partition_blocks(part, model, k)
        t1 = time.time()
        res = pc.form_stage(cl.num_nodes, cl.devices_per_node, batch, bs)
        t2 = time.time()
        out[name] = {"block_atoms": [list(g) for g in bs.block_atoms],
                     "costs": [[c.t_fwd_sec.hex(), c.t_bwd_sec.hex(), c.mem_bytes] for c in bs.costs],
                     "form_stage": result_doc(res),
                     "ref_seconds": {"partition_blocks": t1 - t0, "form_stage": t2 - t1}}
        print(name, out[name]["ref_seconds"], res.stats, flush=True)
    dump("configs.json", out)


def chains():
    out = {}
    for nb, D, seed in ((64, 8, None), (64, 8, 0), (32, 16, 1)):
        bs = cases.c5_blockset(nb, D, jitter_seed=seed)
        res = pc.form_stage(max(1, D // 8), min(8, D), 8 * D, bs,
                            pc.SearchOptions(disable_pruning=True))
        out[f"nb{nb}_D{D}_seed{seed}"] = result_doc(res)
        print(nb, D, seed, res.stats, flush=True)
    dump("chains.json", out)


def cost_tables():
    """Measured cost tables (costs.py:43-80, 130-148): partition_blocks, span
    profiles, form_stage_dp and form_stage with overrides."""
    out = []
    rng = random.Random(4242)
    for i in range(80):
        part, model, k, (nodes, dpn, S, D, BS, R, MB) = cases.cost_table_instance(rng)
        rec = {"index": i, "k": k, "args": [nodes, dpn, S, D, BS, R, MB]}
        try:
            bs = pc.partition_blocks(part, model, k)
        except pc.InfeasibleAtom as e:
            rec["error"] = ["InfeasibleAtom", str(e)]
            out.append(rec)
            continue
        rec["block_atoms"] = [list(g) for g in bs.block_atoms]
        rec["costs"] = [[c.t_fwd_sec.hex(), c.t_bwd_sec.hex(), c.mem_bytes] for c in bs.costs]
        nb = len(bs)
        shares = sorted({BS // (MB * R * d) for d in range(1, D - S + 2)} - {0})
        spans = {}
        for m in shares:
            for lo in range(nb):
                for hi in range(lo + 1, nb + 1):
                    for ck in (False, True):
                        c = bs.model.profile(bs.span(lo, hi), m, checkpointing=ck)
                        spans[f"{lo},{hi},{m},{int(ck)}"] = [c.t_fwd_sec.hex(), c.t_bwd_sec.hex(),
                                                             c.mem_bytes]
        rec["spans"] = spans
        if S <= nb:
            for prune in (True, False):
                res = pc.form_stage_dp(bs, S, D, BS, R, MB,
                                       pc.SearchOptions(disable_pruning=not prune))
                rec["dp_pruned" if prune else "dp_unpruned"] = result_doc(res)
            rec["brute"] = result_doc(pc.brute_force_partition(bs, S, D, BS, R, MB))
        rec["form_stage"] = result_doc(pc.form_stage(nodes, dpn, BS, bs))
        calls, _ = enumerate_calls(nodes, dpn, BS, nb)
        rec["calls"] = [[list(c), result_doc(pc.form_stage_dp(bs, c[0], c[1], BS, c[2], c[3]))]
                        for c in calls]
        out.append(rec)
    dump("cost_tables.json", out)


if __name__ == "__main__":
    what = sys.argv[1:] or ["random", "configs", "chains"]
    if "random" in what:
        random_families()
    if "chains" in what:
        chains()
    if "configs" in what:
        configs()
    if "cost_tables" in what:
        cost_tables()
