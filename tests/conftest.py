import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = Path(__file__).resolve().parent / "golden" / "golden_v1.npz"
GOLDEN_NEXT = Path(__file__).resolve().parent / "golden" / "golden_next_v1.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="session")
def golden_next():
    return dict(np.load(GOLDEN_NEXT))


def unpack_records(g, prefix="rec_"):
    """Golden record arrays -> list of (n, edges, X, fs, y) tuples."""
    n, ne, edges, x, fs, y = (g[prefix + k] for k in ("n", "ne", "edges", "x", "fs", "y"))
    out, xo, eo = [], 0, 0
    for i in range(len(n)):
        e = [(int(a), int(b)) for a, b in edges[eo:eo + ne[i]]]
        out.append((int(n[i]), e, x[xo:xo + n[i]], fs[i], y[i]))
        xo += n[i]
        eo += ne[i]
    return out
