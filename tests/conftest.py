import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def golden_small():
    with np.load(os.path.join(GOLDEN, "golden_small.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden_hashes():
    import json
    with open(os.path.join(GOLDEN, "golden_hashes.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o
    if not os.path.exists(o.LIB_PATH):
        o.build()
    return o


@pytest.fixture
def rng():
    return np.random.default_rng(987654321)


def ttv_cases(golden_small, golden_hashes):
    """Yield (name, subs, vals, shape, x, k, error, expected-or-None) from the fixture."""
    for i, case in enumerate(golden_hashes["ttv_cases"]):
        g = golden_small
        exp = None
        if not case["error"]:
            exp = (g[f"t{i}_osubs"], g[f"t{i}_ovals"], tuple(int(v) for v in g[f"t{i}_oshape"]))
        yield (case["name"], g[f"t{i}_subs"], g[f"t{i}_vals"], tuple(int(v) for v in g[f"t{i}_shape"]),
               g[f"t{i}_x"], int(g[f"t{i}_k"]), case["error"], exp)
