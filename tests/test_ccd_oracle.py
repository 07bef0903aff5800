"""Item/user-wise CCD (ccd.hpp:52-125, ccd_train :310-344): the C oracle's restatement pinned bit for
bit against the reference's own ccd_train (oracle/_ref) -- CPU only; the GPU path is checked against
this oracle in test_gpu_ccdw.py."""
import numpy as np


def test_ccd_oracle_matches_reference(oracle, reference, ml100k):
    train, probe = ml100k
    A = oracle.from_triplets(train, 943, 1682)
    M = reference.matrix(train, 943, 1682, "_f32")
    for k, lam, outer in [(10, 0.05, 3), (4, 0.0, 2)]:
        W, H, rows = oracle.ccd_train(A, k, lam, outer, 7, probe)
        W2, H2, rows2 = M.ccd_train(k, lam, outer, 7, probe)
        assert np.array_equal(W, W2) and np.array_equal(H, H2)
        assert np.array_equal(rows["objective"], rows2["objective"])
        assert np.array_equal(rows["rmse"], rows2["rmse"])


def test_ccd_oracle_double(oracle, reference):
    t = oracle.random_triplets(40, 30, 350, 71)
    A = oracle.from_triplets(t, 40, 30, real="_f64")
    M = reference.matrix(t, 40, 30, "_f64")
    W, H, rows = oracle.ccd_train(A, 3, 0.1, 4, 9, real="_f64")
    W2, H2, rows2 = M.ccd_train(3, 0.1, 4, 9)
    assert np.array_equal(W, W2) and np.array_equal(H, H2)
    assert np.all(np.diff(rows["objective"]) <= 0)  # exact 1-D minimisations never increase it
