import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); parity tests proper")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(autouse=True)
def _checked_build_invariants():
    """Under TSIM_EXPECT_CHECKED=1 (tests/test_gpu_checked.py runs GPU tests
    against the -DTS_CHECKED library): after every test, the row kernel's
    invariant counters must be clean (ts_debug_checks, include/tsim.h)."""
    if os.environ.get("TSIM_EXPECT_CHECKED") != "1":
        yield
        return
    import paper_cs_0105004_b200 as tsim
    tsim.debug_checks(reset=True)
    yield
    checked, bits, first_group, count = tsim.debug_checks(reset=True)
    assert checked == 1, "TSIM_EXPECT_CHECKED=1 but the loaded library is not a checked build"
    assert count == 0, (f"row-kernel invariants violated: bits {bits:#x}, "
                        f"first group {first_group}, {count} violations")
