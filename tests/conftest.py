import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: larger-scale case (seconds to a minute)")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def corpus():
    return load_golden("corpus.json")["graphs"]


@pytest.fixture(scope="session")
def kron16():
    return load_golden("kronecker_s16.json")


@pytest.fixture(scope="session")
def kron_big():
    return load_golden("kronecker_big.json")


def edges_of(g):
    e = np.array(g["edges"], dtype=np.uint64).reshape(-1, 2)
    return e


def levels_list(lv):
    return [-1 if x == 0xFFFFFFFFFFFFFFFF else int(x) for x in lv]
