"""torchrun check: form_stage_sharded over N GPUs (NCCL) == single-GPU
form_stage == golden/reference, on C1-C4 and a C5 chain, plus budget errors.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port 29511 tools/check_sharded.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, world = dist.get_rank(), dist.get_world_size()

import cases  # noqa: E402
from paper_2103_16063_b200 import form_stage, form_stage_sharded, partition_blocks  # noqa: E402
from paper_2103_16063_b200._host import pipecut as pc  # noqa: E402
from plans import result_doc  # noqa: E402

gold = json.load(open(os.path.join(ROOT, "tests", "golden", "configs.json")))
ok = True
for name in ("C1", "C2", "C3", "C4"):
    part, model, k, batch, cl = cases.config_partition(name)
    bs = partition_blocks(part, model, k)
    got = result_doc(form_stage_sharded(cl.num_nodes, cl.devices_per_node, batch, bs))
    lvl = result_doc(form_stage_sharded(cl.num_nodes, cl.devices_per_node, batch, bs,
                                        speculative=False))
    same = got == gold[name]["form_stage"] == lvl
    ok &= same
    if rank == 0:
        print(f"{name}: sharded over {world} == golden: {same}", flush=True)
bs = cases.c5_blockset(128, 32, jitter_seed=2)
a = result_doc(form_stage_sharded(4, 8, 256, bs))
b = result_doc(form_stage(4, 8, 256, bs))
ok &= a == b
if rank == 0:
    print(f"C5 nb=128 D=32: sharded == single-GPU: {a == b}", flush=True)
small = cases.one_block_per_task(cases.chain([1.0] * 4), nodes=1, dpn=2)
for budget in (2, 20, 45, 80):
    def run(fn):
        try:
            r = fn(1, 2, 8, small, pc.SearchOptions(visit_budget=budget))
            return ("ok", r.stats.visits)
        except pc.SearchBudgetExceeded as e:
            return ("budget", e.visits)
    same = (run(form_stage_sharded) == run(pc.form_stage)
            == run(lambda *a, **k: form_stage_sharded(*a, speculative=False, **k)))
    ok &= same
# measured cost tables: golden form_stage of the reference (tests/golden/cost_tables.json)
import random  # noqa: E402

rng = random.Random(4242)
n_ct = 0
for rec in json.load(open(os.path.join(ROOT, "tests", "golden", "cost_tables.json"))):
    part, model, k, (nodes, dpn, S, D, BS, R, MB) = cases.cost_table_instance(rng)
    if "error" in rec:
        continue
    bs = partition_blocks(part, model, k)
    same = result_doc(form_stage_sharded(nodes, dpn, BS, bs)) == rec["form_stage"]
    ok &= same
    n_ct += same
if rank == 0:
    print(f"cost tables: {n_ct} sharded searches == golden", flush=True)
t = torch.tensor([1 if ok else 0], device="cuda")
dist.all_reduce(t, op=dist.ReduceOp.MIN)
if rank == 0:
    print("ALL OK" if t.item() == 1 else "MISMATCH", flush=True)
dist.destroy_process_group()
sys.exit(0 if t.item() == 1 else 1)
