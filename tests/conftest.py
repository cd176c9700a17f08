import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def load_json(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_traces():
    return load_json("traces.json"), np.load(os.path.join(GOLDEN, "traces.npz"))


@pytest.fixture(scope="session")
def golden_batches():
    return load_json("batches.json"), np.load(os.path.join(GOLDEN, "batches.npz"))


@pytest.fixture(scope="session")
def golden_records():
    return load_json("records.json")


@pytest.fixture(scope="session")
def golden_seeds_keys():
    return load_json("seeds_keys.json")


@pytest.fixture(scope="session")
def golden_deltas():
    return load_json("deltas.json")


@pytest.fixture(scope="session")
def golden_optima():
    return load_json("optima.json")


@pytest.fixture(scope="session")
def oracle():
    import oracle as o

    o.build()
    return o


@pytest.fixture(scope="session")
def golden_config2_traces():
    return load_json("config2_traces.json")


@pytest.fixture(scope="session")
def golden_config_records():
    return load_json("config_records.json")


@pytest.fixture(scope="session")
def golden_optima_43_55():
    return load_json("optima_43_55.json")
