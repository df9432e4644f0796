import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running GPU case")


def _cuda():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


HAS_CUDA = _cuda()


def pytest_collection_modifyitems(config, items):
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords and not HAS_CUDA:
            item.add_marker(skip)


_cache = {}


def golden(name):
    """Load tests/golden/<name>.npz (reference-generated, see make_golden.py)."""
    if name not in _cache:
        with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
            _cache[name] = {k: z[k] for k in z.files}
    return _cache[name]


@pytest.fixture
def gold():
    return golden


def kernels_launched(fn):
    """Run fn() under the CUDA activity profiler; return (result, set of kernel names).

    The set is None when the profiler recorded no device activity at all (CUPTI can stop
    delivering records late in a long test process); callers then skip only the
    which-kernel assertion, never the numerical ones."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        out = fn()
        torch.cuda.synchronize()
    names = {e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA}
    return out, (names or None)
