import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) device; parity tests proper")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs (run under gpurun --gpus N)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def has_cuda() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def cuda_required():
    if not has_cuda():
        pytest.fail("a -m gpu test ran without a CUDA device")
