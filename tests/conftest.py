import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device")


def golden(name):
    d = np.load(os.path.join(GOLDEN, name + ".npz"))
    out = {k: d[k] for k in d.files if k != "meta"}
    out.update(json.loads(str(d["meta"])))
    return out


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import REF_SO, Ref
    if not os.path.exists(REF_SO) and not os.path.isdir("/root/reference/proj"):
        pytest.skip("reference library not built and /root/reference absent")
    return Ref()


@pytest.fixture(scope="session")
def ctx():
    from paper_1705_03524_b200 import swg
    return swg.Context(0)
