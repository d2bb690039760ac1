import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: full-size parity (seconds of CPU oracle work)")


def _has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


HAS_GPU = _has_gpu()


def pytest_collection_modifyitems(config, items):
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def port():
    from oracle import Port

    return Port()


@pytest.fixture(scope="session")
def ref():
    from oracle import Ref

    if not Ref.available():
        pytest.skip("reference build (oracle/_ref) not available")
    return Ref()


@pytest.fixture(scope="session")
def fq():
    import paper_2402_17985_b200 as fq

    fq.lib()  # loads libfqg.so or raises
    return fq


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round f64 -> bf16 -> f64 (round-to-nearest-even), the bench input format."""
    import torch

    return torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16).double().numpy()
