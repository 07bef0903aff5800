"""CPU tests of the C-ABI library: it loads, exports every symbol include/pmf_gpu.h declares, its host
helpers (from_triplets, partition_balanced) match the reference, and without a GPU
every compute entry point fails loudly (no CPU fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "pmf_gpu.h")).read()
    return sorted(set(re.findall(r"^\s*(?:pmf_status|const char\*|int32_t)\s+(pmf_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol(pmf):
    syms = declared_symbols()
    assert len(syms) >= 30
    raw = C.CDLL(pmf.LIB_PATH)
    missing = [s for s in syms if not hasattr(raw, s)]
    assert not missing, missing
    assert pmf.lib.pmf_abi_version() == 1


def test_no_cpu_fallback_without_device(pmf, oracle, ml100k):
    if pmf.device_count() > 0:
        pytest.skip("a CUDA device is present")
    train, probe = ml100k
    A = pmf.RatingsMatrix.from_triplets(train, 943, 1682)
    for call in (lambda: pmf.ccdpp_train(pmf.CcdConfig(k=2, outer_iters=1, inner_iters=1), A, probe),
                 lambda: pmf.als_train(pmf.AlsConfig(k=2, outer_iters=1), A, probe),
                 lambda: pmf.rmse(pmf.FactorModel.zeros(943, 1682, 2), probe),
                 lambda: pmf.ccdpp_update_u(A, A.val_row, np.zeros(1682), 0.1),
                 lambda: pmf.Context(A)):
        with pytest.raises(RuntimeError, match="no CUDA device"):
            call()


def test_from_triplets_matches_reference(pmf, oracle, ml100k):
    train, _ = ml100k
    A = pmf.RatingsMatrix.from_triplets(train, 943, 1682)
    B = oracle.from_triplets(train, 943, 1682)
    for f in ("row_start", "col_of", "val_row", "col_start", "row_of", "val_col"):
        assert np.array_equal(getattr(A, f), getattr(B, f)), f
    # canonical: independent of input order (sparse.hpp:117-118)
    perm = np.random.default_rng(1).permutation(len(train))
    C2 = pmf.RatingsMatrix.from_triplets(train[perm], 943, 1682)
    assert np.array_equal(C2.col_of, A.col_of) and np.array_equal(C2.row_of, A.row_of)
    assert np.array_equal(C2.val_col, A.val_col)


def test_from_triplets_errors(pmf):
    with pytest.raises(IndexError):
        pmf.RatingsMatrix.from_triplets([(3, 0, 1.0)], 3, 3)
    with pytest.raises(IndexError):
        pmf.RatingsMatrix.from_triplets([(0, -1, 1.0)], 3, 3)
    with pytest.raises(ValueError, match=r"^duplicate rating for user 1, item 2$"):  # sparse.hpp:127-132
        pmf.RatingsMatrix.from_triplets([(2, 0, 1.0), (1, 2, 1.0), (2, 0, 3.0), (1, 2, 2.0)], 3, 3)
    with pytest.raises(ValueError):
        pmf.RatingsMatrix.from_triplets([(0, 0, float("inf"))], 3, 3)
    with pytest.raises(ValueError):
        pmf.RatingsMatrix.from_triplets([], -1, 3)
    E = pmf.RatingsMatrix.from_triplets([], 4, 2)
    assert E.nnz() == 0 and list(E.row_start) == [0] * 5


def test_partition_balanced_matches_reference(pmf, oracle):
    rng = np.random.default_rng(9)
    for count, p in ((50, 1), (50, 3), (2000, 8), (5, 9)):
        c = rng.integers(0, 500, count)
        assert np.array_equal(pmf.partition_balanced(c, p), oracle.partition_balanced(c, p))
    with pytest.raises(ValueError):
        pmf.partition_balanced([1, 2], 0)
    with pytest.raises(ValueError):
        pmf.partition_balanced([1, -2], 2)


def test_init_random_items_matches_reference(pmf, oracle):
    for n, k, seed in ((10, 5, 123), (1682, 10, 1), (7, 40, 2 ** 33 + 1)):
        assert np.array_equal(pmf.init_random_items(n, k, seed), oracle.init_random_items(n, k, seed))


def test_predict_host(pmf):
    W = np.zeros((2, 1), np.float32); H = np.zeros((2, 1), np.float32)
    W[0, 0] = 2.0; H[1, 0] = 3.0
    m = pmf.FactorModel(W, H)
    assert pmf.predict(m, 0, 1) == 6.0
    with pytest.raises(IndexError):
        pmf.predict(m, 2, 0)
