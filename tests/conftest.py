import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]
GOLDEN = REPO / "tests" / "golden"
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the CUDA path through the C ABI")
    config.addinivalue_line("markers", "slow: full-size configuration checks")


def golden_cases():
    return sorted(p.stem for p in GOLDEN.glob("*.npz"))


def load_golden(name):
    import json

    z = np.load(GOLDEN / f"{name}.npz")
    settings = json.loads(str(z["settings"]))
    return z, settings


@pytest.fixture(scope="session")
def evaluator():
    """One device context for the whole GPU session (fails loudly without a GPU)."""
    from paper_2105_01196_b200 import Evaluator, build

    build.build_ext()
    ev = Evaluator(0)
    yield ev
    ev.close()
