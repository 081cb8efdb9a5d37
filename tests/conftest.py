import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def pytest_sessionstart(session):
    # Checkers (oracle/) and the product library are built in-tree; on the GPU
    # box the prebuilt files travel with the snapshot and make is a no-op.
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=False,
                   stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    from paper_2210_06528_b200.build import build
    build()


def have_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def ctx():
    import paper_2210_06528_b200 as m
    if not have_gpu():
        pytest.skip("no CUDA device")
    return m.Context(0)
