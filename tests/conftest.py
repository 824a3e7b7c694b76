import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libcommdet_cuda.so")
    config.addinivalue_line("markers", "slow: takes more than a few seconds")


@pytest.fixture(scope="session")
def golden():
    arr = np.load(os.path.join(GOLDEN, "golden.npz"))
    with open(os.path.join(GOLDEN, "manifest.json")) as f:
        man = json.load(f)
    return arr, man


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.lib()
    return O


@pytest.fixture(scope="session")
def ref(oracle):
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built (reference headers absent)")
    oracle.ref()
    return oracle


@pytest.fixture(scope="session")
def dev():
    """The product package bound to cuda:0 (GPU tests only)."""
    import paper_1304_4453_b200 as P
    P.load_library()
    return P


@pytest.fixture(scope="session")
def ctx(dev):
    return dev.default_context()


# ---- shared instance builders (numpy PCG64, weights exact in fp32) ---------
def rand_edges(rng, n, p, kind="int", loop_p=0.0):
    eu, ev, ew = [], [], []
    for u in range(n):
        vs = np.nonzero(rng.random(n - u - 1) < p)[0] + u + 1
        for v in vs:
            eu.append(u)
            ev.append(int(v))
            ew.append(weight(rng, kind))
        if loop_p > 0 and rng.random() < loop_p:
            eu.append(u)
            ev.append(u)
            ew.append(weight(rng, kind))
    if not eu:
        eu, ev, ew = [0], [min(1, n - 1)], [1.0]
    return np.array(eu, np.int32), np.array(ev, np.int32), np.array(ew, np.float64)


def weight(rng, kind):
    if kind == "unit":
        return 1.0
    if kind == "int":
        return float(rng.integers(1, 6))
    return float((int(rng.integers(0, 1 << 24)) + 1) * 2.0 ** -24)


BARBELL = [(0, 1, 1), (0, 2, 1), (1, 2, 1), (3, 4, 1), (3, 5, 1), (4, 5, 1), (2, 3, 1)]
TWO_TRIANGLES = [(0, 1, 1), (0, 2, 1), (1, 2, 1), (3, 4, 1), (3, 5, 1), (4, 5, 1)]
TRIANGLES = np.array([0, 0, 0, 1, 1, 1], np.int32)


def same_relation(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return bool(np.array_equal(a[:, None] == a[None, :], b[:, None] == b[None, :]))


def refines(a, b):
    a, b = np.asarray(a), np.asarray(b)
    sa = a[:, None] == a[None, :]
    sb = b[:, None] == b[None, :]
    return bool(np.all(~sa | sb))
