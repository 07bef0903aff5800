"""top_n (model.hpp:172-209): the C oracle's restatement pinned against the reference's own top_n
(oracle/_ref) on the reference's known answers (tests/model_test.cpp:184-233) and random models with
ties -- CPU only; the GPU kernel is checked against this oracle in test_gpu_topn.py."""
import numpy as np
import pytest


def test_topn_known_answers(oracle):
    zero_w = np.zeros((2, 2), np.float32); zero_h = np.zeros((5, 2), np.float32)
    assert [j for j, _ in oracle.top_n(zero_w, zero_h, 0, 3, [1, 3])] == [0, 2, 4]   # ties -> ascending
    w = np.array([[1.0]], np.float32); h = np.array([[1.0], [2.0], [3.0]], np.float32)
    best = oracle.top_n(w, h, 0, 2)
    assert [(j, float(s)) for j, s in best] == [(2, 3.0), (1, 2.0)]
    assert len(oracle.top_n(w, h, 0, 10, [0])) == 2                                 # exhausted
    with pytest.raises(ValueError):
        oracle.top_n(w, h, 0, 0)
    with pytest.raises(IndexError):
        oracle.top_n(w, h, 5, 1)


def test_topn_oracle_matches_reference(oracle, reference):
    rng = np.random.default_rng(6)
    for m, n, k, count in [(4, 20, 3, 12), (3, 300, 7, 25), (2, 1000, 40, 1000)]:
        W = rng.uniform(-1, 1, (m, k)).astype(np.float32)
        H = rng.uniform(-1, 1, (n, k)).astype(np.float32)
        H[::7] = np.round(H[::7] * 2) / 2          # coarse rows: equal scores -> tie order matters
        for i in range(m):
            rated = np.sort(rng.choice(n, n // 5, replace=False)).astype(np.int32)
            a = oracle.top_n(W, H, i, count, rated)
            b = reference.top_n(W, H, i, count, rated)
            assert [(j, s.tobytes()) for j, s in a] == [(j, s.tobytes()) for j, s in b]
