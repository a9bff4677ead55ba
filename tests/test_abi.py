"""CPU: the C-ABI library loads and exports every symbol include/pipecut_b200.h
declares; without a GPU the compute entry points refuse (no CPU fallback)."""

import ctypes as C
import os
import re

import pytest

from paper_2103_16063_b200 import _lib, abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    with open(os.path.join(ROOT, "include", "pipecut_b200.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(pc_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_python_exports():
    declared = set(_declared())
    assert declared == set(_lib.EXPORTS)
    assert {"pc_form_stage", "pc_form_stage_dp", "pc_run_calls", "pc_set_problem",
            "pc_profile_spans"} <= declared


def test_library_loads_and_exports_every_symbol():
    lib = _lib.load()
    for name in _declared() + list(_lib.EXPORTS):
        assert hasattr(lib, name), name


def test_struct_layouts_match_header():
    # sizes of the ABI structs as compiled by gcc from the header
    import subprocess
    import tempfile
    src = r'''
#include <stdio.h>
#include <stddef.h>
#include "pipecut_b200.h"
int main(void){printf("%zu %zu %zu %zu %zu %zu %zu\n", sizeof(pc_problem), sizeof(pc_plan),
 sizeof(pc_stats), sizeof(pc_call), sizeof(pc_call_result), offsetof(pc_problem, mem_budget),
 offsetof(pc_plan, objective));return 0;}
'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        with open(c, "w") as fh:
            fh.write(src)
        exe = os.path.join(d, "t")
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()
    got = [int(x) for x in out]
    want = [C.sizeof(abi.PcProblem), C.sizeof(abi.PcPlan), C.sizeof(abi.PcStats),
            C.sizeof(abi.PcCall), C.sizeof(abi.PcCallResult),
            abi.PcProblem.mem_budget.offset, abi.PcPlan.objective.offset]
    assert got == want


def test_no_cpu_fallback_without_device():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(_lib.DeviceUnavailable):
        _lib.Context(0)
