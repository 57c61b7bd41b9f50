import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).parent))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity or statistical test")


@pytest.fixture(scope="session")
def koller():
    """The bundled student network with its textbook CPTs (package API types)."""
    from paper_1511_06416_b200.io import bundled_network_path, load_network_file

    return load_network_file(bundled_network_path("koller"))


@pytest.fixture(autouse=True)
def _checked_build_asserts():
    """Under SG_CHECKED_RUN=1 (tests/test_gpu_checked.py runs the parity suites
    against lib_checked.so): after every test, no device-side SG_DCHECK failed."""
    yield
    if os.environ.get("SG_CHECKED_RUN") == "1":
        from paper_1511_06416_b200 import _lib

        hits = {tu: line for tu, line in _lib.checked_lines().items() if line}
        assert not hits, f"device-side SG_DCHECK failed (translation unit: source line): {hits}"
