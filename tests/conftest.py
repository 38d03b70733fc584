import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_tests")

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN_DIR = ROOT / "tests" / "golden"
REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running case")


@pytest.fixture(scope="session")
def golden():
    meta = json.loads((GOLDEN_DIR / "golden.json").read_text())
    arrays = np.load(GOLDEN_DIR / "golden.npz")
    return meta, arrays


@pytest.fixture(scope="session")
def oracle():
    import oracle as o

    o.lib()
    return o


@pytest.fixture(scope="session")
def reference():
    """The live reference package (container only; absent on the GPU box)."""
    if not REFERENCE_SRC.exists():
        pytest.skip("/root/reference not mounted")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.append(str(REFERENCE_SRC))
    import gasketmap.backends as backends  # noqa: F401
    import gasketmap

    return gasketmap


@pytest.fixture(scope="session")
def gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1706_04552_b200 as gm

    gm.native.lib()  # fails loudly if the sm_100a library is missing
    return gm


@pytest.fixture(autouse=True)
def _release_gpu_memory(request):
    """After every GPU test, hand the cached device memory back to the driver: the
    BASELINE-size cases allocate up to ~130 GB, and later tests that start their own
    processes on the same GPU (tests/test_bench_multirank.py) must find it free."""
    yield
    if request.node.get_closest_marker("gpu") is None:
        return
    torch = sys.modules.get("torch")
    if torch is not None and torch.cuda.is_available() and torch.cuda.is_initialized():
        import gc

        gc.collect()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
