"""partition_blocks + form_stage at paper scale (~15,000 atoms): host phases
vs the library call."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2103_16063_b200 import flatten as F
from paper_2103_16063_b200 import build_atomic_subcomponents, form_stage, partition_blocks
from paper_2103_16063_b200._host import pipecut as pc

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 1536
g = pc.gen_bert_like(1024, layers, 512, 30522)
t0 = time.perf_counter()
ref = pc.build_atomic_subcomponents(g)
t1 = time.perf_counter()
part = build_atomic_subcomponents(g)
t2 = time.perf_counter()
assert part.atoms == ref.atoms and part.graph == ref.graph and part.clone_origins == ref.clone_origins
cl = pc.ClusterSpec(32, 8, 32 * 10 ** 9, 50e9, 10e9)
model = pc.CostModel(part.graph, pc.CostModelConfig(), cl)
print(f"{layers} layers: {len(part.atoms)} atoms, {len(g.nodes)} nodes; atoms: reference "
      f"{1e3 * (t1 - t0):.0f} ms, C++ {1e3 * (t2 - t1):.0f} ms (same partition)", flush=True)
if "--warm-small" in sys.argv:
    g0 = pc.gen_bert_like(64, 2, 16, 100)
    p0 = pc.build_atomic_subcomponents(g0)
    partition_blocks(p0, pc.CostModel(p0.graph, pc.CostModelConfig(), cl), 4)
    print("warmed up on a small graph", flush=True)
for rep in range(2):
    F._ATOM_CACHE.clear()
    t2 = time.perf_counter()
    fa = F.flatten_atoms(part, model)
    t3 = time.perf_counter()
    bs = partition_blocks(part, model, 32)
    t4 = time.perf_counter()
    res = form_stage(32, 8, 2048, bs)
    t5 = time.perf_counter()
    print(f"flatten_atoms {1e3*(t3-t2):.0f} ms, partition_blocks (cached flatten) {1e3*(t4-t3):.0f} ms, "
          f"form_stage {1e3*(t5-t4):.0f} ms, {len(bs)} blocks, plan {res.plan is not None}", flush=True)
