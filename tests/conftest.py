import os
import sys

import pytest

# The in-process multi-rank tests (loopback / MOE_FLAG_P2P) drive G ranks on ONE GPU
# from G streams. A P2P rank's stream blocks on a wait-value until its peers have
# signalled; if two ranks' streams shared one hardware work queue, the waiting rank
# would also block its peer's signal (false dependency) -> deadlock. 32 queues (the
# maximum; default 8) give every stream of a group its own queue. Set before CUDA
# is initialised. (One process per GPU, the production layout, has no such aliasing.)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: full-size (BASELINE.json configs 1-2) cases")


@pytest.fixture(scope="session")
def cuda_available():
    import torch
    return torch.cuda.is_available()
