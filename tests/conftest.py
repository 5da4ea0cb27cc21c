import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box with -m gpu)")


@pytest.fixture(scope="session")
def port():
    from oracle import cpu
    return cpu.port()


@pytest.fixture(scope="session")
def ref():
    from oracle import cpu
    r = cpu.ref()
    if r is None:
        pytest.skip("oracle/_ref/libbinattn_ref.so not built (needs /root/reference)")
    return r


class Golden:
    def __init__(self, path):
        self.z = np.load(path)
        self.meta = json.loads(bytes(self.z["meta"]).decode())

    def case(self, name):
        pre = name + "/"
        return {k[len(pre):]: self.z[k] for k in self.z.files if k.startswith(pre)}


@pytest.fixture(scope="session")
def golden():
    return Golden(os.path.join(ROOT, "tests", "golden", "binattn_golden.npz"))
