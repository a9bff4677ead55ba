import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)

# the host API is the unmodified reference installed in baseline/_ref (git-ignored);
# on a fresh checkout create it the way build() does (offline pip install)
if not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "pipecut")):
    import __graft_entry__

    __graft_entry__._ensure_reference_install()


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libpipecut_b200.so")
    config.addinivalue_line("markers", "slow: long-running parity sweep")


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    if not has_gpu():
        pytest.skip("no CUDA device")
    from paper_2103_16063_b200 import _lib
    return _lib.context(0)
