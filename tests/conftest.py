import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def ref_lib():
    """The compiled reference oracle (oracle/_ref); built here if missing."""
    from oracle import ref
    if not ref.available():
        import subprocess
        if Path("/root/reference/proj").exists():
            subprocess.run(["make", "-C", str(ROOT / "oracle"), "-j8"], check=True,
                           capture_output=True)
    if not ref.available():
        pytest.skip("oracle/_ref not built and /root/reference absent")
    return ref


@pytest.fixture(scope="session")
def gpu_lib():
    from paper_1807_01769_b200 import api
    return api.load_library()
