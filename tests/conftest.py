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
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: full-size runs")


@pytest.fixture(scope="session")
def ts():
    import paper_2303_08365_b200
    return paper_2303_08365_b200


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle.Oracle()


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.Reference.available():
        pytest.skip("reference library not built (oracle/_ref); run make -C oracle ref")
    return oracle.Reference()


def golden_index():
    with open(os.path.join(GOLDEN, "index.json")) as f:
        return json.load(f)


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    return z["cur"], z["prev"]


def bench_kernel(ts, name):
    return ts.find_benchmark(name).kernel


def random_grid(ts, orc, extent, halo, seed, dtype="f64"):
    """fill_random(seed) grid built by the oracle (test_util.hpp:66-70)."""
    g = (ts.Grid if dtype == "f64" else ts.GridF)(extent, halo)
    orc.fill_random(g, seed)
    return g


def bitwise_equal_interior(a, b):
    x = a.interior_view(a.parity)
    y = b.interior_view(b.parity)
    return x.tobytes() == y.tobytes()
