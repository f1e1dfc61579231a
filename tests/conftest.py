import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    return np.load(os.path.join(ROOT, "tests", "golden", "expm_golden.npz"))


@pytest.fixture(scope="session")
def lowrank_golden():
    import numpy as np
    return np.load(os.path.join(ROOT, "tests", "golden", "lowrank_golden.npz"))


def lowrank_cases(g):
    """(i, name, A1, A2, X, eps) for every case of lowrank_golden.npz."""
    offs, oo = g["offsets"], g["out_offsets"]
    for i in range(len(g["names"])):
        n, t = int(g["n"][i]), int(g["t"][i])
        A1 = g["A1"][offs[i]:offs[i + 1]].reshape(n, t)
        A2 = g["A2"][offs[i]:offs[i + 1]].reshape(t, n)
        X = g["X"][oo[i]:oo[i + 1]].reshape(n, n)
        yield i, str(g["names"][i]), A1, A2, X, float(g["eps"][i])
