"""CPU: the reference arm (baseline/ref_arm.py) runs the unmodified reference
without the repo's package, on the same workloads the GPU arm measures."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline"))

import ref_arm  # noqa: E402

from paper_2103_16063_b200 import workloads  # noqa: E402
from paper_2103_16063_b200.search import enumerate_calls  # noqa: E402


@pytest.mark.parametrize("nb,D,seed", [(24, 8, None), (40, 16, 0), (33, 64, 3)])
def test_chain_builders_agree(nb, D, seed):
    a = ref_arm.chain_blockset(nb, D, jitter_seed=seed)
    b = workloads.c5_blockset(nb, D, jitter_seed=seed)
    assert a.block_atoms == b.block_atoms
    assert [(c.t_fwd_sec.hex(), c.t_bwd_sec.hex(), c.mem_bytes) for c in a.costs] == \
        [(c.t_fwd_sec.hex(), c.t_bwd_sec.hex(), c.mem_bytes) for c in b.costs]
    assert a._cut_fixed == b._cut_fixed and a._cut_per_sample == b._cut_per_sample
    assert a.model.cluster == b.model.cluster


@pytest.mark.parametrize("nodes,dpn,bs,nb", [(1, 8, 64, 100), (32, 8, 2048, 4096),
                                             (128, 8, 8192, 300), (4, 2, 16, 5)])
def test_enumeration_agrees(nodes, dpn, bs, nb):
    assert ref_arm.enumerate_calls(nodes, dpn, bs, nb) == enumerate_calls(nodes, dpn, bs, nb)[0]


def test_configs_match_the_product_workloads():
    assert ref_arm.CONFIGS == workloads.CONFIGS


def test_reference_arm_loads_no_repo_code():
    code = ("import sys; sys.path.insert(0, 'baseline'); import ref_arm; "
            "r = ref_arm.sample(48, 16, 1, 20000); "
            "bad = [m for m in sys.modules if m.startswith('paper_2103_16063_b200') or "
            "m.startswith('oracle')]; assert not bad, bad; "
            "assert r['visits'] > 20000 and r['value'] > 0, r; print('ok')")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0 and out.stdout.strip() == "ok", out.stderr
