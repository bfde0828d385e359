import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU and the built libirdn.so")


def _build_once():
    from oracle import oracle
    from paper_1201_3972_b200 import build

    oracle.build()
    build.build_scene()
    build.build_cuda()


_build_once()


def load_golden(name: str):
    """Yield (meta, input, output) for every case of tests/golden/<name>."""
    z = np.load(os.path.join(GOLDEN, name))
    meta = json.loads(str(z["meta"]))
    return [(m, z[f"in{i}"], z[f"out{i}"]) for i, m in enumerate(meta)]


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available() and torch.cuda.get_device_capability(0)[0] == 10
    except Exception:
        return False


@pytest.fixture(scope="session")
def cuda_ok():
    if not gpu_available():
        pytest.skip("needs a B200 GPU")
    return True


@pytest.fixture
def cuda_ok_or_none():
    """True when a B200 is visible, False otherwise (never skips)."""
    return bool(gpu_available())


@pytest.fixture(scope="session")
def reference_pkg():
    """The unmodified reference package (baseline/_ref, pip-installed from /root/reference)."""
    from paper_1201_3972_b200 import launcher

    try:
        return launcher.import_reference()
    except ImportError:
        pytest.skip("the reference is not installed in baseline/_ref")
