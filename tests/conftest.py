import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running")
    # The forward stores label tiles only from D >= 1536 (ops.LABEL_STORE_MIN_D); the parity
    # cases use small D, so force the store path on for them (tests that need it off set "0").
    os.environ.setdefault("CCE_STORE_LABELS", "1")


def golden_cases():
    return sorted(p.stem for p in GOLDEN.glob("*.npz"))


@pytest.fixture(scope="session")
def cuda_device():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)
