import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through liblbdd_b200.so)")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def instance_from_json(j):
    from paper_2304_06543_b200.instance import PenaltySpec, ProblemInstance, ServiceCenter
    centers = [ServiceCenter(i, j["capacity"][i], PenaltySpec(j["family"][i], list(j["params"][i])))
               for i in range(j["k"])]
    return ProblemInstance(centers, np.array(j["costs"], dtype=np.int32).reshape(j["n"], j["k"]))


@pytest.fixture(scope="session")
def oracle():
    import pyoracle
    return pyoracle.oracle()


@pytest.fixture(scope="session")
def reference():
    import pyoracle
    ref = pyoracle.reference()
    if ref is None:
        pytest.skip("oracle/_ref/liblbdd_ref.so not built (no /root/reference here)")
    return ref


@pytest.fixture(scope="session")
def dev():
    """The product's device API; fails (does not skip) when the CUDA library
    is missing on a GPU box."""
    from paper_2304_06543_b200 import solver
    if solver.device_count() < 1:
        pytest.skip("no CUDA device")
    return solver
