import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def _golden_path():
    return os.path.join(ROOT, "oracle", "_golden", "libgolden_rlwe.so")


@pytest.fixture(scope="session")
def golden_lib():
    """The golden C model (oracle).  Built on demand with `make -C oracle`."""
    import subprocess
    path = _golden_path()
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    from paper_2102_03494_b200.abi import Library
    return Library(path)


@pytest.fixture(scope="session")
def cuda_lib():
    from paper_2102_03494_b200.abi import cuda_library
    return cuda_library()
