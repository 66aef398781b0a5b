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


@pytest.fixture(autouse=True)
def _release_device_memory():
    """GPU tests upload inputs through torch and keep per-test device
    contexts: return their memory after every test, so a large product later
    in the session (C5b bands: ~23 GB of workspace) does not fail on memory
    an earlier test still caches."""
    yield
    if "torch" in sys.modules:
        import gc
        import torch
        if torch.cuda.is_initialized():
            gc.collect()
            torch.cuda.empty_cache()
