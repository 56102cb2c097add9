import hashlib
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: N=2^16 oracle runs (seconds to a minute)")


def digest(rows) -> str:
    """SHA-256 of little-endian uint32 residues; matches tests/golden/make_golden.py."""
    a = np.asarray(rows)
    if hasattr(rows, "cpu"):
        a = rows.cpu().numpy()
    a = np.ascontiguousarray(np.asarray(a, dtype=np.uint64).astype("<u4"))
    return hashlib.sha256(a.tobytes()).hexdigest()


def load_json(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def load_npz(name):
    return np.load(os.path.join(GOLDEN, name))


@pytest.fixture(scope="session")
def golden_params():
    return load_json("params.json")
