import os
import sys

import pytest

# Results the binding allocates start as NaN in tests (paper_1502_02389_b200.POISON_OUTPUTS):
# an element a kernel fails to write must not pass on a recycled buffer's stale value.
os.environ.setdefault("LIFT_POISON_OUTPUTS", "1")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Compile the native libraries once per session (no-op when up to date)."""
    import __graft_entry__
    __graft_entry__.build()
    yield


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    # A `-m gpu` run on a machine without a GPU would silently pass nothing; make it loud.
    if gpu_available():
        return
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(pytest.mark.skip(reason="no CUDA device in this container"))
