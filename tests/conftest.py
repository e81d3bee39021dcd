"""Test configuration: the `gpu` marker gates tests that need a B200."""

from __future__ import annotations

import os
import pathlib
import sys

# One-GPU simulations of multi-rank nodes (OneGpuShardGroup) run every rank's
# kernels on its own stream and spin-wait across streams: each stream needs
# its own hardware queue, or a rank's push can sit behind another rank's wait
# (CUDA's default is 8 queues).  Read at CUDA context creation.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = pathlib.Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libvsb200.so")


def cuda_ok() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def golden():
    return GOLDEN


@pytest.fixture(scope="session")
def dev():
    if not cuda_ok():
        pytest.fail("GPU test selected but no CUDA device is visible")
    import torch

    from paper_1805_03709_b200 import build

    build.build()
    return torch.device("cuda", 0)
