import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a path")
    config.addinivalue_line("markers", "slow: full-size benchmark configs")


@pytest.fixture(scope="session", autouse=True)
def _built():
    from paper_2002_11302_b200 import build
    build.build_host()
    import oracle
    oracle.build(ref=Path("/root/reference/proj/src").is_dir())
    yield
