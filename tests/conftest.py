import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs on the GPU box")
    config.addinivalue_line("markers", "slow: long-running (full-size) test")


@pytest.fixture(scope="session")
def golden_hexes():
    from tests.pins import load_golden
    return {name: load_golden(name) for name in ("fig5_invalid", "fig6_valid", "fig7_invalid")}


@pytest.fixture(autouse=True)
def _release_cuda_cache(request):
    """Full-size GPU tests allocate tens of GB; hand cached blocks back between tests."""
    yield
    if request.node.get_closest_marker("gpu") is not None:
        try:
            import torch
            if torch.cuda.is_available():
                torch.cuda.synchronize()
                torch.cuda.empty_cache()
        except Exception:
            pass
