import gzip
import json
import sys
from functools import lru_cache
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden" / "reference_golden.json.gz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: full-size (BASELINE) sizes")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(autouse=True)
def _release_cuda_cache(request):
    """Give cached device memory back after every GPU test, so the full-size
    tests (up to ~150 GiB) find HBM free."""
    yield
    if "gpu" in request.keywords:
        import gc

        import torch
        gc.collect()
        if torch.cuda.is_available():
            torch.cuda.synchronize()
            torch.cuda.empty_cache()


@lru_cache(maxsize=1)
def golden() -> dict:
    with gzip.open(GOLDEN, "rt") as f:
        return json.load(f)


@pytest.fixture(scope="session")
def ref_golden():
    return golden()
