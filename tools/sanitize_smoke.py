"""Every entry point on small inputs, for compute-sanitizer runs (memcheck,
racecheck, synccheck): DP/search (pruned, unpruned, budget), cost tables with
the pruning cut, brute force, validate/simulate, coarsening, sharded path."""
import os, random, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import cases
from paper_2103_16063_b200 import (brute_force_partition, form_stage, form_stage_dp,
                                   form_stage_sharded, partition_blocks)
from paper_2103_16063_b200._host import pipecut as pc
from paper_2103_16063_b200.simulate import simulate, validate_plan

bs = cases.c5_blockset(48, 16, jitter_seed=1)
r = form_stage(2, 8, 128, bs)
form_stage(2, 8, 128, bs, pc.SearchOptions(disable_pruning=True))
try:
    form_stage(2, 8, 128, bs, pc.SearchOptions(visit_budget=10 ** 5))
except pc.SearchBudgetExceeded:
    pass
form_stage_sharded(2, 8, 128, bs)
simulate(r.plan, bs)
validate_plan(r.plan, bs)
small = cases.c5_blockset(10, 8, jitter_seed=2)
brute_force_partition(small, 3, 8, 64, 1, 2)
rng = random.Random(4242)
for _ in range(12):
    part, model, k, (nodes, dpn, S, D, BS, R, MB) = cases.cost_table_instance(rng)
    try:
        b = partition_blocks(part, model, k)
    except pc.InfeasibleAtom:
        continue
    if S <= len(b):
        form_stage_dp(b, S, D, BS, R, MB)
    form_stage(nodes, dpn, BS, b)
rng = random.Random(5)
for _ in range(6):
    g = cases.layered_graph(rng)
    p, m = cases.blocks_inputs(g)
    try:
        partition_blocks(p, m, rng.randint(1, 6))
    except pc.CompactionStuck:
        pass
# refinement on the device: C1 (moves, rejected candidates), C4 (cluster
# kernel), a fan graph (dozens of levels); the bounded DP path on a small chain
from paper_2103_16063_b200.workloads import config_partition
for name in ("C1", "C4"):
    part, model, k, batch, cl = config_partition(name)
    b = partition_blocks(part, model, k)
    if name == "C1":
        form_stage(cl.num_nodes, cl.devices_per_node, batch, b)
p, m = cases.blocks_inputs(cases.fan_graph(random.Random(2), 90))
partition_blocks(p, m, 3)
os.environ["PIPECUT_B200_BOUND_MIN_VISITS"] = "0"
form_stage(4, 8, 256, cases.c5_blockset(128, 32, jitter_seed=3))
print("sanitize smoke done")
