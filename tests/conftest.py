"""Shared test configuration.

``-m gpu`` tests need a B200 and the in-tree CUDA library; everything else
runs on the CPU build container (oracle vs golden vectors, host logic, C-ABI
symbol surface, 2-rank gloo tests).
"""

import json
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 GPU and the built CUDA library")


def load_golden(name):
    return json.loads((GOLDEN / name).read_text())


@pytest.fixture(scope="session")
def golden():
    return load_golden


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if cuda_ok():
        return
    skip = pytest.mark.skip(reason="needs a CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
