import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a kernels")
    config.addinivalue_line("markers", "slow: larger shapes (seconds to a minute)")


@pytest.fixture(scope="session")
def oracle():
    from oracle.pyoracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.pyoracle import Reference, have_reference
    if not have_reference():
        pytest.skip("oracle/_ref/libparmf_ref.so not built (needs /root/reference at build time)")
    return Reference()


@pytest.fixture(scope="session")
def pmf():
    import paper_1511_02433_b200 as P
    return P


@pytest.fixture(scope="session")
def ml100k(oracle):
    """ML-100K-shape synthetic corpus (testutil.hpp synth_ratings, seed 777) with a 10% probe
    carved by carve_probe (seed 5) -- BASELINE.json configs[0]."""
    a = oracle.synth_ratings(943, 1682, 3, 100000, 777)
    train, probe = oracle.carve_probe(a, 10000, 5)
    return train, probe


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def frob_rel(x, y):
    return float(np.linalg.norm(np.asarray(x, np.float64) - np.asarray(y, np.float64)) /
                 max(np.linalg.norm(np.asarray(y, np.float64)), 1e-300))
