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
