import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

PRECS = ["f32", "f16", "e5m3", "e4m4"]
CASES = ["small", "blobs", "sub3_p5", "sift_mini"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def load_case(name):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    return {k: z[k] for k in z.files}


def index_from_case(c):
    from paper_2301_06672_b200.index import IvfPqIndex, PQCodebook

    return IvfPqIndex.from_csr(c["coarse"], PQCodebook(centers=c["centers"], p=int(c["p"])),
                               c["list_off"], c["ids"], c["codes"])


@pytest.fixture(scope="session")
def golden():
    return {name: load_case(name) for name in CASES}
