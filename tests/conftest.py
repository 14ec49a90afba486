import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
for p in (str(ROOT), str(ROOT / "tests"), str(ROOT / "tools")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (runs on the B200 box)")


@pytest.fixture(scope="session")
def gpu():
    """An rt3d Session on cuda:0.  GPU tests fail loudly without a device."""
    from paper_1905_06700_b200.rt3d import Session
    s = Session(0)
    yield s
    s.close()
