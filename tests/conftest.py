import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libtang.so")


def pytest_collection_modifyitems(config, items):
    # a gpu test on a box without CUDA is a skip only when explicitly deselected; when
    # selected with -m gpu it must run and fail loudly if the device or library is missing
    pass


@pytest.fixture(scope="session")
def table1():
    """Parsed tests/golden/table1.txt."""
    path = os.path.join(ROOT, "tests", "golden", "table1.txt")
    rules, tuples, grid, counts, trunc, inserts = [], [], {}, {}, [], []
    for line in open(path):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        f = line.split()
        if f[0] == "rule":
            rules.append((f[1], int(f[2]), f[3], f[4], int(f[5]), int(f[6])))
        elif f[0] == "tuple":
            tuples.append((f[1], int(f[2]), int(f[3]), f[4:]))
        elif f[0] == "grid":
            grid[int(f[1])] = f[2:]
        elif f[0] == "count":
            counts[f[1]] = int(f[2])
        elif f[0] == "truncate":
            trunc.append((f[1], int(f[2]), f[3]))
        elif f[0] == "insert":
            inserts.append((f[1], int(f[2]), f[3], f[4], f[5]))
    return dict(rules=rules, tuples=tuples, grid=grid, counts=counts, trunc=trunc, inserts=inserts)
