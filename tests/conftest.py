"""Shared fixtures. `-m "not gpu"` runs here (no GPU); `-m gpu` on a B200."""
import json
import pathlib
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running full-size parity")


@pytest.fixture(scope="session")
def golden():
    return json.loads((GOLDEN / "reference_vectors.json").read_text())


@pytest.fixture(scope="session")
def golden_arrays():
    with np.load(GOLDEN / "reference_arrays.npz") as z:
        return {k: z[k] for k in z.files}


def golden_params(rec):
    """Params as the reference saw them (ints were stored as decimal strings)."""
    out = {}
    for k, v in rec["params"].items():
        out[k] = int(v) if isinstance(v, str) else v
    return out
