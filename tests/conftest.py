import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"

# the C-ABI library is a build artefact (git-ignored): build it once if this checkout lacks it
_LIB = ROOT / "paper_2510_13602_b200" / "libnosa_b200.so"
if not _LIB.exists():
    import subprocess
    subprocess.run(["make", "-j8", "-C", str(ROOT / "paper_2510_13602_b200" / "csrc")], check=True)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a); run with -m gpu")


@pytest.fixture
def golden():
    def load(name):
        return dict(np.load(GOLDEN / f"{name}.npz", allow_pickle=False))
    return load


@pytest.fixture
def rng():
    return np.random.default_rng(1234)
