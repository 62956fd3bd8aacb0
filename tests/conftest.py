import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def oracle():
    import oracle as O
    return O.Oracle()


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference (oracle/_ref).  Present in the build container and, prebuilt, on the GPU box."""
    import oracle as O
    try:
        return O.Ref()
    except (FileNotFoundError, OSError):
        pytest.skip("oracle/_ref/libgempe_ref.so not available")


@pytest.fixture(scope="session")
def golden_fastmath():
    import oracle as O
    t = load_golden("numerics.json")["tables"]
    return O.fastmath_from_flat([float(v) for v in t["erf"]["flat"]], [float(v) for v in t["ratio"]["flat"]])


# ---- small graph builders in the spirit of the reference's tests/testutil.hpp ------------------------------

def ring(n):
    s = np.arange(n, dtype=np.uint32)
    return n, s, ((s + 1) % n).astype(np.uint32)


def clique_pair(k):
    e = []
    for off in (0, k):
        for i in range(k):
            for j in range(i + 1, k):
                e.append((off + i, off + j))
    e.append((0, k))
    e = np.array(e, np.uint32)
    return 2 * k, np.ascontiguousarray(e[:, 0]), np.ascontiguousarray(e[:, 1])


def er_graph(n, m, seed):
    from paper_2011_03479_b200.graphgen import Stream
    rng = Stream(seed, 77)
    chosen = {}
    while len(chosen) < m:
        a, b = (int(v) for v in rng.below(2, n))
        if a == b:
            continue
        chosen.setdefault((min(a, b), max(a, b)), None)
    e = np.array(list(chosen), np.uint32)
    return n, np.ascontiguousarray(e[:, 0]), np.ascontiguousarray(e[:, 1])


def star_plus_ring(n, hubs=2):
    """A few very-high-degree vertices (hub splitting) on top of a ring."""
    e = [(i, (i + 1) % n) for i in range(n)]
    for h in range(hubs):
        for v in range(n):
            if v != h and abs(v - h) not in (1, n - 1) and (v + h) % 3 != 0:
                e.append((h, v))  # two thirds of all vertices: high degree, yet non-edges remain
    seen = {}
    for a, b in e:
        seen.setdefault((min(a, b), max(a, b)), None)
    e = np.array(list(seen), np.uint32)
    return n, np.ascontiguousarray(e[:, 0]), np.ascontiguousarray(e[:, 1])


def rel_l2(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
