import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built liblrqmm.so")
    config.addinivalue_line("markers", "slow: multi-second CPU test")


@pytest.fixture(scope="session")
def golden_tables():
    rows = {}
    with open(os.path.join(ROOT, "tests", "golden", "paper_tables_2_3.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            d, b, dq, q110, q111, lr = line.split()
            rows[(d, int(b))] = dict(dq=float(dq), qt110=float(q110), qt111=float(q111), lrqmm=float(lr))
    return rows
