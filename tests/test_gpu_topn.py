"""GPU top_n (model.hpp:172-209) against the oracle restatement (pinned to the
reference in test_topn_oracle.py): items and scores bitwise, ties by ascending item, rated-item
exclusion from lists and from a RatingsMatrix, the reference's known answers and errors."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _check_batch(pmf, oracle, W, H, users, count, rated):
    items, scores, counts = pmf.top_n_batch(pmf.FactorModel(W, H), users, count, rated=rated)
    for u, i in enumerate(users):
        exp = oracle.top_n(W, H, int(i), count, rated[u])
        assert counts[u] == len(exp)
        assert list(items[u, :counts[u]]) == [j for j, _ in exp]
        assert scores[u, :counts[u]].tobytes() == np.array([s for _, s in exp], np.float32).tobytes()
        assert (items[u, counts[u]:] == -1).all()


def test_topn_known_answers(pmf):
    zero = pmf.FactorModel.zeros(2, 5, 2)
    assert [j for j, _ in pmf.top_n(zero, 0, 3, [1, 3])] == [0, 2, 4]
    m = pmf.FactorModel(np.array([[1.0]], np.float32), np.array([[1.0], [2.0], [3.0]], np.float32))
    assert pmf.top_n(m, 0, 2, []) == [(2, 3.0), (1, 2.0)]
    assert len(pmf.top_n(m, 0, 10, [0])) == 2
    with pytest.raises(ValueError):
        pmf.top_n(m, 0, 0, [])
    with pytest.raises(IndexError):
        pmf.top_n(m, 5, 1, [])
    # matrix overload (tests/model_test.cpp:224-233)
    a = pmf.RatingsMatrix.from_triplets([(0, 1, 5.0), (0, 3, 2.0), (1, 0, 1.0)], 2, 5)
    mm = pmf.FactorModel(np.array([[1.0], [0.0]], np.float32), np.arange(5, dtype=np.float32).reshape(5, 1))
    assert [j for j, _ in pmf.top_n(mm, a, 0, 5)] == [4, 2, 0]


@pytest.mark.parametrize("m,n,k,count", [(150, 700, 10, 10), (70, 257, 40, 100), (65, 1000, 3, 5), (3, 40, 64, 60)])
def test_topn_random_vs_oracle(pmf, oracle, m, n, k, count):
    rng = np.random.default_rng(m + n + k)
    W = rng.uniform(-1, 1, (m, k)).astype(np.float32)
    H = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    H[::5] = np.round(H[::5] * 2) / 2
    W[::3] = np.round(W[::3] * 2) / 2          # many exactly equal scores
    users = rng.permutation(m)[: max(1, m - 3)].astype(np.int32)
    rated = [np.sort(rng.choice(n, rng.integers(0, n // 3), replace=False)).astype(np.int32) for _ in users]
    _check_batch(pmf, oracle, W, H, users, count, rated)


@pytest.mark.parametrize("m,n,k,count", [(40, 300, 10, 300), (30, 257, 10, 1000), (20, 900, 100, 400),
                                         (12, 500, 200, 7), (9, 64, 3, 64)])
def test_topn_wide_vs_oracle(pmf, oracle, m, n, k, count):
    """count >= items (every unrated item ranked) and k x count past the tiled kernel's shared memory:
    the wide path (full scoring + stable segmented sort), same results."""
    rng = np.random.default_rng(m * n + k)
    W = rng.uniform(-1, 1, (m, k)).astype(np.float32)
    H = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    H[::4] = np.round(H[::4] * 2) / 2
    W[::3] = np.round(W[::3] * 2) / 2
    W[1] = 0.0                                   # +0 / -0 scores: ties by ascending item
    users = np.arange(m, dtype=np.int32)
    rated = [np.sort(rng.choice(n, rng.integers(0, n // 2), replace=False)).astype(np.int32) for _ in users]
    _check_batch(pmf, oracle, W, H, users, count, rated)


def test_topn_matrix_exclusion_vs_oracle(pmf, oracle, ml100k):
    train, _ = ml100k
    A = pmf.RatingsMatrix.from_triplets(train, 943, 1682)
    rng = np.random.default_rng(2)
    model = pmf.FactorModel(rng.normal(0, 1, (943, 10)).astype(np.float32),
                            rng.normal(0, 1, (1682, 10)).astype(np.float32))
    users = np.arange(943, dtype=np.int32)
    items, scores, counts = pmf.top_n_batch(model, users, 20, a=A)
    for i in range(0, 943, 37):
        rated = A.col_of[A.row_start[i]:A.row_start[i + 1]]
        exp = oracle.top_n(model.w, model.h, i, 20, rated)
        assert list(items[i, :counts[i]]) == [j for j, _ in exp]
        assert scores[i, :counts[i]].tobytes() == np.array([s for _, s in exp], np.float32).tobytes()
