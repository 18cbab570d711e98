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


TRANSFORMED = ("lognormal", "gumbel", "pareto", "weibull", "gpd")


def is_vectorized(rec):
    """The reference's default (numpy-vectorised) transform path: not bit-exact by design
    (continuous.py:364-410 uses np.exp/np.log); parity bar = 4 ulp (north star)."""
    return rec["dist"] in TRANSFORMED and not rec.get("bitexact", False)


def max_ulp(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    same = (a == b) | (np.isnan(a) & np.isnan(b))
    if same.all():
        return 0.0
    a, b = a[~same], b[~same]
    return float(np.max(np.abs(a - b) / np.spacing(np.maximum(np.abs(a), np.abs(b)))))


def vec_close(a, b):
    """The reference's own contract for its vectorised transforms vs the det_* route
    (pkg/tests/test_continuous.py:140-153): every element within 4 ulp or 1e-13
    absolute (cancellation in the transform), and >= 90 % within 4 ulp."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    ulp_ok = np.abs(a - b) <= 4 * np.spacing(np.maximum(np.abs(a), np.abs(b)))
    ulp_ok |= (a == b)
    return bool(np.all(ulp_ok | (np.abs(a - b) < 1e-13)) and ulp_ok.mean() > 0.9)
