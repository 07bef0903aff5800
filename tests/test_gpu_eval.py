"""GPU evaluation kernels (model.hpp:103-167) vs the reference."""
import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu


def test_objective_golden_fixture(pmf, oracle):
    """tests/model_test.cpp:91-102 fixture (FP32 model): GPU objective == oracle FP32 objective."""
    t = [(0, 0, 4.0), (0, 2, 3.0), (1, 1, 5.0), (2, 0, 1.0)]
    A = pmf.RatingsMatrix.from_triplets(t, 3, 3)
    W = np.array([[0.5, -0.2], [1.0, 0.3], [-0.4, 0.8]], np.float32)
    H = np.array([[0.6, 0.1], [0.2, -0.7], [1.1, 0.4]], np.float32)
    obj = pmf.objective(pmf.FactorModel(W, H), A, 0.1)
    O = oracle.from_triplets(np.array(t, dtype=[("user", "<i4"), ("item", "<i4"), ("rating", "<f8")]), 3, 3)
    ref, _ = oracle.objective(O, W, H, 0.1)
    assert rel(obj, ref) < 1e-14
    assert abs(obj - 47.129999999999995) < 1e-5     # the double-precision golden value, FP32 factors


def test_rmse_cases(pmf):
    """tests/model_test.cpp:170-183."""
    W = np.zeros((3, 2), np.float32); H = np.zeros((3, 2), np.float32)
    W[0, 0] = 1.0; H[1, 0] = 4.0
    m = pmf.FactorModel(W, H)
    assert pmf.rmse(m, [(0, 1, 4.0)]) == 0.0
    assert pmf.rmse(m, [(0, 1, 2.0)]) == 2.0
    with pytest.raises(ValueError):
        pmf.rmse(m, [])
    with pytest.raises(IndexError):
        pmf.rmse(m, [(3, 0, 1.0)])


def test_rmse_and_objective_vs_reference_large(pmf, oracle, reference):
    """FP32 predict in sequential t (model.hpp:111-112) is bit-exact per entry; only the FP64
    summation order differs -> agreement to ~1e-13 relative."""
    t = oracle.synth_ratings(3000, 1500, 3, 200000, 99)
    tr, pr = oracle.carve_probe(t, 20000, 3)
    A = pmf.RatingsMatrix.from_triplets(tr, 3000, 1500)
    rng = np.random.default_rng(4)
    W = rng.uniform(-1, 1, (3000, 40)).astype(np.float32)
    H = rng.uniform(-1, 1, (1500, 40)).astype(np.float32)
    m = pmf.FactorModel(W, H)
    assert rel(pmf.rmse(m, pr), reference.rmse(W, H, pr)) < 1e-12
    M = reference.matrix(tr, 3000, 1500)
    assert rel(pmf.objective(m, A, 0.05), M.objective(W, H, 0.05)) < 1e-12
