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


@pytest.fixture(autouse=True)
def _fresh_library_state():
    """Every test starts without learned S-hat capacities (they are keyed by the head, so another
    test's data could size this one's slots) and without a pending label-range error."""
    try:
        from paper_2411_09009_b200 import ops
    except Exception:  # noqa: BLE001 - CPU-only collection without the package importable
        yield
        return
    ops._KEPT_HINT.clear()
    ops._IGNORED_HINT.clear()
    ops._LABEL_STATE.clear()
    yield


@pytest.fixture(scope="session")
def cuda_device():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)
