import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN_DIR = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


@pytest.fixture(scope="session")
def golden():
    meta = json.loads((GOLDEN_DIR / "golden_v1.json").read_text())
    arrays = np.load(GOLDEN_DIR / "golden_v1.npz")
    return meta, arrays


@pytest.fixture(scope="session")
def native_lib():
    """Build (if stale) and load the C-ABI library."""
    from paper_1409_8116_b200 import _build, _native

    _build.build()
    if not cuda_ok():
        # (a CPU container has the toolchain: build the PyTorch extension too if it is stale;
        # the GPU box only ever uses the prebuilt files)
        _build.build_torch_ext()
    return _native.load()


@pytest.fixture
def rng():
    return np.random.default_rng(20240901)


def cuda_ok():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
