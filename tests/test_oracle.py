"""CPU tests: pin the oracle (oracle/pmf_oracle.c) against the reference's golden vectors and against
the reference itself compiled here (oracle/_ref).  No GPU needed."""
import json
import math
import os

import numpy as np
import pytest

from conftest import rel

GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_trajectories.json")

# tests/oracle/gen_fixture_values.py:20-54 (frozen in tests/ccd_test.cpp:253-280)
FIX65 = [(0, 0, 5.0), (0, 2, 3.0), (0, 4, 1.0), (1, 1, 4.0), (1, 2, 2.0), (2, 0, 1.0), (2, 4, 5.0),
         (3, 1, 2.0), (3, 2, 4.5), (3, 4, 2.5), (5, 0, 3.5), (5, 1, 1.5), (5, 2, 2.0), (5, 4, 4.0)]
V0 = [0.8, -0.5, 1.2, 0.3, -1.0]
EXPECT_U = [2.0754716981132075, 0.22346368715083795, -2.4137931034482758, 0.68100358422939045, 0.0,
            0.13119533527696797]
EXPECT_V = [0.82163605483103141, 3.8874624185557933, 2.0249580990531117, 0.0, -0.72480018190921613]


def trips64(lst):
    from oracle.pyoracle import TRIP64
    return np.array(lst, dtype=TRIP64)


def test_golden_rank_one_fixture(oracle):
    A = oracle.from_triplets(trips64(FIX65), 6, 5, "_f64")
    u = oracle.update_u(A, A.val_row, V0, 0.1, "_f64")
    v = oracle.update_v(A, A.val_col, u, 0.1, "_f64")
    np.testing.assert_allclose(u, EXPECT_U, rtol=0, atol=1e-12)
    np.testing.assert_allclose(v, EXPECT_V, rtol=0, atol=1e-12)


def test_golden_objective_fixture(oracle):
    # tests/oracle/gen_fixture_values.py:11-18, tests/model_test.cpp:91-102
    A = oracle.from_triplets(trips64([(0, 0, 4.0), (0, 2, 3.0), (1, 1, 5.0), (2, 0, 1.0)]), 3, 3, "_f64")
    W = np.array([[0.5, -0.2], [1.0, 0.3], [-0.4, 0.8]])
    H = np.array([[0.6, 0.1], [0.2, -0.7], [1.1, 0.4]])
    obj, _ = oracle.objective(A, W, H, 0.1, "_f64")
    assert abs(obj - 47.129999999999995) <= 1e-12


def test_known_answers_ccdpp_stages(oracle):
    A = oracle.from_triplets(trips64([(0, 0, 1.0)]), 1, 1, "_f64")
    rr, rc = oracle.build_rhat(A, A.val_row, A.val_col, [2.0], [3.0], "_f64")
    assert rr[0] == 7.0 and rc[0] == 7.0  # ccd_test.cpp:203-210
    rr, rc, W, H = oracle.writeback(A, rr, rc, [2.0], [3.0], real="_f64")
    assert rr[0] == 1.0 and rc[0] == 1.0 and W[0, 0] == 2.0 and H[0, 0] == 3.0  # ccd_test.cpp:306-318
    A6 = oracle.from_triplets(trips64([(0, 0, 6.0)]), 1, 1, "_f64")
    assert oracle.update_u(A6, A6.val_row, [2.0], 0.0, "_f64")[0] == 3.0   # 6*2/2^2
    assert oracle.update_u(A6, A6.val_row, [0.0], 0.5, "_f64")[0] == 0.0   # v = 0 -> 0


def test_known_answers_dense(oracle, reference):
    m = np.array([[4.0, 2.0], [2.0, 3.0]])
    L = oracle.cholesky_factor(m)
    np.testing.assert_allclose(L, [[2.0, 0.0], [1.0, math.sqrt(2.0)]], atol=1e-15)
    x = oracle.cholesky_solve(L, [4.0, 5.0])
    np.testing.assert_allclose(x, [0.25, 1.5], atol=1e-14)
    with pytest.raises(ArithmeticError):
        oracle.cholesky_factor(np.array([[1.0, 2.0], [2.0, 1.0]]))
    with pytest.raises(ZeroDivisionError):
        oracle.cholesky_solve(np.array([[1.0, 0.0], [0.0, 0.0]]), [1.0, 1.0])
    rng = np.random.default_rng(17)
    for k in (1, 2, 5, 10):
        b = rng.uniform(-1, 1, (k, k))
        spd = b @ b.T + 0.1 * np.eye(k)
        assert np.array_equal(oracle.cholesky_factor(spd), reference.cholesky_factor(spd))
        rhs = rng.uniform(-3, 3, k)
        Lk = oracle.cholesky_factor(spd)
        assert np.array_equal(oracle.cholesky_solve(Lk, rhs), reference.cholesky_solve(Lk, rhs))


def test_als_known_answers(oracle):
    # als_test.cpp:14-29: empty row -> 0; k=1, A=4, h=2 -> w = 4*2/(4+lambda)
    A = oracle.from_triplets(trips64([(1, 0, 4.0)]), 3, 2, "_f64")
    out = oracle.als_half(A, 0, np.full((2, 2), 0.5), 0.1, "_f64")
    assert np.all(out[0] == 0.0)
    A1 = oracle.from_triplets(trips64([(0, 0, 4.0)]), 1, 1, "_f64")
    w = oracle.als_half(A1, 0, np.array([[2.0]]), 1e-12, "_f64")
    assert abs(w[0, 0] - 2.0) < 1e-9


def test_generators_match_reference(oracle, reference):
    assert np.array_equal(oracle.synth_ratings(300, 200, 3, 12500, 4242), reference.synth_ratings(300, 200, 3, 12500, 4242))
    assert np.array_equal(oracle.random_triplets(40, 30, 350, 71), reference.random_triplets(40, 30, 350, 71))
    assert np.array_equal(oracle.planted_full(20, 15, 2, 0.01, 42), reference.planted_full(20, 15, 2, 0.01, 42))
    d = oracle.synth_ratings(60, 40, 2, 1200, 17)
    for a, b in zip(oracle.carve_probe(d, 240, 4), reference.carve_probe(d, 240, 4)):
        assert np.array_equal(a, b)


def test_layout_and_init_match_reference(oracle, reference, ml100k):
    train, _ = ml100k
    A = oracle.from_triplets(train, 943, 1682)
    B = reference.matrix(train, 943, 1682).export()
    for f in ("row_start", "col_of", "val_row", "col_start", "row_of", "val_col", "xlink"):
        assert np.array_equal(getattr(A, f), getattr(B, f)), f
    for k, seed in ((10, 1), (40, 7), (3, 2 ** 40 + 5)):
        assert np.array_equal(oracle.init_random_items(50, k, seed), reference.init_random_items(50, k, seed))


def test_from_triplets_errors(oracle):
    with pytest.raises(IndexError):
        oracle.from_triplets(trips64([(3, 0, 1.0)]), 3, 3)
    with pytest.raises(ValueError):
        oracle.from_triplets(trips64([(0, 0, 1.0), (0, 0, 2.0)]), 3, 3)
    with pytest.raises(ValueError):
        oracle.from_triplets(trips64([(0, 0, float("nan"))]), 3, 3)


@pytest.mark.parametrize("real", ["_f32", "_f64"])
def test_ccdpp_bitwise_vs_reference(oracle, reference, ml100k, real):
    train, probe = ml100k
    A = oracle.from_triplets(train, 943, 1682, real)
    M = reference.matrix(train, 943, 1682, real)
    W, H, rows, rr, rc = oracle.ccdpp_train(A, 10, 0.05, 3, 15, 1, probe, real)
    W2, H2, rows2, rr2, rc2 = M.ccdpp_stage_loop(10, 0.05, 3, 15, 1, probe, workers=4)
    W3, H3, rows3 = M.ccdpp_train(10, 0.05, 3, 15, 1, probe, workers=4)
    assert np.array_equal(W, W2) and np.array_equal(H, H2) and np.array_equal(W, W3) and np.array_equal(H, H3)
    assert np.array_equal(rr, rr2) and np.array_equal(rc, rc2)
    for f in ("objective", "rmse"):
        assert np.array_equal(rows[f], rows2[f]) and np.array_equal(rows[f], rows3[f])
    assert np.array_equal(rows["train_rmse"], rows2["train_rmse"])


@pytest.mark.parametrize("real", ["_f32", "_f64"])
def test_als_bitwise_vs_reference(oracle, reference, ml100k, real):
    train, probe = ml100k
    A = oracle.from_triplets(train, 943, 1682, real)
    M = reference.matrix(train, 943, 1682, real)
    W, H, rows = oracle.als_train(A, 10, 0.05, 3, 1, probe, real)
    W2, H2, rows2 = M.als_train(10, 0.05, 3, 1, probe, workers=4)
    assert np.array_equal(W, W2) and np.array_equal(H, H2)
    assert np.array_equal(rows["objective"], rows2["objective"]) and np.array_equal(rows["rmse"], rows2["rmse"])


def test_oracle_matches_golden_file(oracle, ml100k):
    """The committed fixtures (made by the reference, tests/golden/make_golden.py) vs the oracle."""
    gold = json.load(open(GOLD))
    train, probe = ml100k
    A = oracle.from_triplets(train, 943, 1682, "_f32")
    _, _, rows, _, _ = oracle.ccdpp_train(A, 10, 0.05, 5, 15, 1, probe, "_f32")
    for r, g in zip(rows, gold["ccdpp_ml100k_k10_f32"]["rows"]):
        assert r["objective"] == g["objective"] and r["rmse"] == g["rmse"] and r["train_rmse"] == g["train_rmse"]
    _, _, rows = oracle.als_train(A, 10, 0.05, 5, 1, probe, "_f32")
    for r, g in zip(rows, gold["als_ml100k_k10_f32"]["rows"]):
        assert r["objective"] == g["objective"] and r["rmse"] == g["rmse"]
    # reference float vs double stay inside the parity band the GPU must meet
    for f in ("objective", "rmse", "train_rmse"):
        for a, b in zip(gold["ccdpp_ml100k_k10_f32"]["rows"], gold["ccdpp_ml100k_k10_f64"]["rows"]):
            assert rel(a[f], b[f]) < 1e-5


def test_partition_balanced_matches_reference(oracle, reference):
    rng = np.random.default_rng(3)
    for count, p in ((100, 1), (100, 4), (1000, 8), (7, 16), (0, 3)):
        costs = rng.integers(0, 1000, count)
        assert np.array_equal(oracle.partition_balanced(costs, p), reference.partition_balanced(costs, p))
