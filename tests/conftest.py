import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_runs.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def product_lib():
    """The CUDA library, built in-tree (build() compiles it for sm_100a)."""
    import paper_2508_14568_b200 as pkg
    if not os.path.exists(pkg.LIB_PATH):
        pkg.build()
    return pkg.lib()


@pytest.fixture(scope="session")
def ctx():
    import paper_2508_14568_b200 as pkg
    if not os.path.exists(pkg.LIB_PATH):
        pkg.build()
    c = pkg.Context(seed=0)
    yield c
    c.close()


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle as O
    return O.Oracle(0)
