import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"
REF_SRC = Path(os.environ.get("DASH_REF_SRC", "/root/reference/pkg/src"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libdash_b200.so")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    import json

    import numpy as np

    return {
        "structure": json.loads((GOLDEN / "structure.json").read_text()),
        "seeds": dict(np.load(GOLDEN / "seeds.npz")),
        "solvers": dict(np.load(GOLDEN / "solvers.npz")),
        "steps": dict(np.load(GOLDEN / "steps.npz")),
    }


@pytest.fixture(scope="session")
def reference():
    """The live reference package (only in the build container); skips elsewhere."""
    if not (REF_SRC / "blockshampoo").exists():
        pytest.skip("reference sources not present (GPU box)")
    sys.path.insert(0, str(REF_SRC))
    import blockshampoo.shampoo  # noqa: F401
    import blockshampoo

    return blockshampoo
