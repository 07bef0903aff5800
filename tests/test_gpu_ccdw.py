"""GPU item/user-wise CCD (ccd.hpp:52-125, ccd_train :310-344) against the oracle
(pinned to the reference in test_ccd_oracle.py): per-iteration objective, train and probe RMSE within
1e-4 relative, factors within 1e-3 relative Frobenius (default: warp / CTA residual sweeps; PMF_CCD_GRAM=1,
k <= 40: each coordinate sweep as a Gauss-Seidel sweep on the row's normal equations with a tensor-core
gram; the reference's sums are sequential), objective non-increasing, edge cases, both paths."""
import numpy as np
import pytest

from conftest import frob_rel, rel

pytestmark = pytest.mark.gpu


def test_ccd_ml100k_vs_oracle(pmf, oracle, ml100k):
    train, probe = ml100k
    A = pmf.RatingsMatrix.from_triplets(train, 943, 1682)
    O = oracle.from_triplets(train, 943, 1682)
    cfg = pmf.CcdConfig(k=10, lam=0.05, outer_iters=4, inner_iters=15, seed=1)
    model, rep = pmf.ccd_train(cfg, A, probe)
    W, H, rows = oracle.ccd_train(O, 10, 0.05, 4, 1, probe)
    for r, g in zip(rep.rows, rows):
        assert rel(r.objective, g["objective"]) < 1e-4
        assert rel(r.rmse, g["rmse"]) < 1e-4
        assert rel(r.train_rmse, g["train_rmse"]) < 1e-4
    assert frob_rel(model.w, W) < 1e-3 and frob_rel(model.h, H) < 1e-3
    objs = [r.objective for r in rep.rows]
    assert all(b <= a * (1 + 1e-6) for a, b in zip(objs, objs[1:]))
    assert pmf.run_training(pmf.RunSpec(pmf.Algorithm.kCcd, k=10, lam=0.05, outer_iters=4, inner_iters=15,
                                        workers=1, seed=1), A, probe)[0] == model


def test_ccd_edges_vs_oracle(pmf, oracle):
    # empty rows / columns, lambda = 0 (den == 0 -> 0), a row longer than the register cache
    t = oracle.random_triplets(57, 41, 300, 9)
    t = np.concatenate([t, np.array([(60, j, 3.0) for j in range(41)] +
                                    [(i, 44, 2.0) for i in range(0, 70, 2)], dtype=t.dtype)])
    A = pmf.RatingsMatrix.from_triplets(t, 70, 45)
    O = oracle.from_triplets(t, 70, 45)
    for lam in (0.0, 0.2):
        model, rep = pmf.ccd_train(pmf.CcdConfig(k=3, lam=lam, outer_iters=3, inner_iters=1, seed=5), A)
        W, H, rows = oracle.ccd_train(O, 3, lam, 3, 5)
        for r, g in zip(rep.rows, rows):
            assert rel(r.objective, g["objective"]) < 1e-4
        assert frob_rel(model.w, W) < 1e-3 and frob_rel(model.h, H) < 1e-3
    with pytest.raises(ValueError):
        pmf.ccd_train(pmf.CcdConfig(k=0), A)


@pytest.mark.slow
def test_ccd_long_rows_vs_oracle(pmf, oracle):
    m, n = 300, 5000
    t = oracle.synth_ratings(m, n, 3, 400000, 3)   # rows of ~1300 entries: the uncached path
    A = pmf.RatingsMatrix.from_triplets(t, m, n)
    O = oracle.from_triplets(t, m, n)
    model, rep = pmf.ccd_train(pmf.CcdConfig(k=5, lam=0.05, outer_iters=2, inner_iters=1, seed=2), A)
    W, H, rows = oracle.ccd_train(O, 5, 0.05, 2, 2)
    for r, g in zip(rep.rows, rows):
        assert rel(r.objective, g["objective"]) < 1e-4
    assert frob_rel(model.w, W) < 1e-3 and frob_rel(model.h, H) < 1e-3


@pytest.mark.slow
def test_ccd_long_columns_vs_oracle(pmf, oracle):
    """Columns of more than 32K entries take the cluster kernel (8 CTAs per column, DSMEM reduction)."""
    rng = np.random.default_rng(4)
    m, n = 60000, 50
    rows, cols = [], []
    for j in range(n):
        cnt = 50000 if j % 5 == 0 else int(rng.integers(1, 3000))   # 10 columns above the threshold
        rows.append(rng.choice(m, cnt, replace=False)); cols.append(np.full(cnt, j))
    i = np.concatenate(rows); j = np.concatenate(cols)
    t = np.zeros(i.size, dtype=[("user", "<i4"), ("item", "<i4"), ("rating", "<f4")])
    t["user"], t["item"], t["rating"] = i, j, rng.integers(1, 6, i.size)
    A = pmf.RatingsMatrix.from_triplets(t, m, n)
    O = oracle.from_triplets(t, m, n)
    model, rep = pmf.ccd_train(pmf.CcdConfig(k=6, lam=0.05, outer_iters=3, inner_iters=1, seed=2), A)
    W, H, rws = oracle.ccd_train(O, 6, 0.05, 3, 2)
    for r, g in zip(rep.rows, rws):
        assert rel(r.objective, g["objective"]) < 1e-4
        assert rel(r.train_rmse, g["train_rmse"]) < 1e-4
    assert frob_rel(model.w, W) < 1e-3 and frob_rel(model.h, H) < 1e-3


def test_ccd_paths_vs_oracle(pmf, oracle, ml100k, monkeypatch):
    # default: the residual kernels; PMF_CCD_GRAM=1 (k <= 40): gram + Gauss-Seidel; k > 40 always residual
    train, probe = ml100k
    A = pmf.RatingsMatrix.from_triplets(train, 943, 1682)
    O = oracle.from_triplets(train, 943, 1682)
    for k, gram in ((12, True), (12, False), (44, True)):
        if gram:
            monkeypatch.setenv("PMF_CCD_GRAM", "1")
        else:
            monkeypatch.delenv("PMF_CCD_GRAM", raising=False)
        model, rep = pmf.ccd_train(pmf.CcdConfig(k=k, lam=0.1, outer_iters=2, inner_iters=1, seed=3), A, probe)
        W, H, rows = oracle.ccd_train(O, k, 0.1, 2, 3, probe)
        for r, g in zip(rep.rows, rows):
            assert rel(r.objective, g["objective"]) < 1e-4
            assert rel(r.rmse, g["rmse"]) < 1e-4
        assert frob_rel(model.w, W) < 1e-3 and frob_rel(model.h, H) < 1e-3


def test_ccd_set_model_rebuilds_residual(pmf, ml100k):
    """set_model on an item/user-wise CCD context rebuilds R = A - W H^T: iterating from an
    installed model tracks the uninterrupted run (residual rounding history differs only)."""
    train, probe = ml100k
    A = pmf.RatingsMatrix.from_triplets(train, 943, 1682)
    cfg = pmf.CcdConfig(k=10, lam=0.05, outer_iters=3, inner_iters=1, seed=1)
    ref = pmf.Context(A); ref.set_probe(probe); ref.ccd_begin(cfg)
    ref.ccd_iterate(1)
    m1 = ref.model()
    ref.ccd_iterate(1)
    o_ref, r_ref, _ = ref.metrics()
    ctx = pmf.Context(A); ctx.set_probe(probe); ctx.ccd_begin(cfg)
    ctx.set_model(m1)
    ctx.ccd_iterate(1)
    o, r, _ = ctx.metrics()
    assert rel(o, o_ref) < 1e-5 and rel(r, r_ref) < 1e-5
    # without the rebuild the second epoch would minimise against A - W0 H0^T (W0 = 0): far off
    ref.close(); ctx.close()
