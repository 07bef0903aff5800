"""Parity at every BASELINE.json config against the reference itself (oracle/_ref: parmf compiled from its
unmodified headers), on the bench's own bytes (bench.make_data -> datagen), all host cores.

* configs[1]  ALS k=10 on the ML-10M shape, 5 iterations            (als.hpp:188-233)
* configs[2]  CCD++ k=40, T=15 on the Netflix shape, 2 outer iterations (ccd.hpp:349-404)
* configs[3]  ALS k=40 on the Netflix shape, 2 iterations
* configs[4]  CCD++ k=100, T=15 on the Yahoo-Music shape, 1 outer iteration (2 in the committed
              artefact profiles/r02_parity_yahoo-ccdpp.json, scripts/parity_artifacts.py)
(configs[0], ML-100K, is covered against the committed reference trajectories in test_gpu_ccd.py.)

The reference runs through its stage API loop (tests/acceptance_test.cpp:150-171 pattern), which is
bitwise its ccdpp_train / als_train trajectory (tests/test_oracle.py) and also yields the per-iteration
train RMSE.  Criteria (north_star): per-iteration objective, probe RMSE and train RMSE
within 1e-4 relative of the reference's float run; final factors within 1e-3 relative Frobenius, or --
where the committed calibration shows the reference's own float and double runs further apart at
that shape -- within twice that float-vs-double distance."""
import json
import os

import numpy as np
import pytest

from conftest import ROOT, frob_rel, rel

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
CORES = os.cpu_count() or 1


def factor_tol(cfg, which, iters):
    """1e-3, or 2 x the reference's own float-vs-double factor distance after `iters` outer iterations
    at this shape (committed calibration: scripts/calibrate_ref.py -> profiles/r02_calib_CFG.json, or the
    float-vs-double column of scripts/parity_artifacts.py -> profiles/r02_parity_CFG.json)."""
    for name in (f"r02_calib_{cfg}.json", f"r02_parity_{cfg}.json"):
        p = os.path.join(ROOT, "profiles", name)
        if os.path.exists(p):
            cal = json.load(open(p))["factors_per_iteration"][iters - 1][f"{which}_f32_vs_f64"]
            return max(1e-3, 2.0 * cal)
    return 1e-3


def _data(cfg):
    import bench
    return bench.make_data(cfg)


def _compare(cfg, gpu_rows, ref_rows, model, W, H):
    assert len(gpu_rows) == len(ref_rows)
    for g, r in zip(gpu_rows, ref_rows):
        assert rel(g.objective, float(r["objective"])) <= 1e-4, (g.iteration, g.objective, r["objective"])
        assert rel(g.rmse, float(r["rmse"])) <= 1e-4, (g.iteration, g.rmse, r["rmse"])
        assert rel(g.train_rmse, float(r["train_rmse"])) <= 1e-4, (g.iteration, g.train_rmse, r["train_rmse"])
    assert frob_rel(model.w, W) <= factor_tol(cfg, "W", len(ref_rows))
    assert frob_rel(model.h, H) <= factor_tol(cfg, "H", len(ref_rows))


def test_ml10m_als_vs_reference(pmf, reference):
    train, probe = _data("ml10m-als")
    A = pmf.RatingsMatrix.from_triplets(train, 69878, 10677)
    model, rep = pmf.als_train(pmf.AlsConfig(k=10, lam=0.05, outer_iters=5, seed=1), A, probe)
    M = reference.matrix(train, 69878, 10677, "_f32")
    W, H, rows = M.als_epochs(10, 0.05, 5, 1, probe, workers=CORES)
    _compare("ml10m-als", rep.rows, rows, model, W, H)


@pytest.fixture(scope="module")
def netflix(reference):
    train, probe = _data("netflix-ccdpp")
    return train, probe, reference.matrix(train, 480189, 17770, "_f32")


def test_netflix_ccdpp_vs_reference(pmf, netflix):
    train, probe, M = netflix
    A = pmf.RatingsMatrix.from_triplets(train, 480189, 17770)
    model, rep = pmf.ccdpp_train(pmf.CcdConfig(k=40, lam=0.05, outer_iters=2, inner_iters=15, seed=1), A, probe)
    W, H, rows, _, _ = M.ccdpp_stage_loop(40, 0.05, 2, 15, 1, probe, workers=CORES)
    _compare("netflix-ccdpp", rep.rows, rows, model, W, H)


def test_netflix_als_vs_reference(pmf, netflix):
    train, probe, M = netflix
    A = pmf.RatingsMatrix.from_triplets(train, 480189, 17770)
    model, rep = pmf.als_train(pmf.AlsConfig(k=40, lam=0.05, outer_iters=2, seed=1), A, probe)
    W, H, rows = M.als_epochs(40, 0.05, 2, 1, probe, workers=CORES)
    _compare("netflix-als", rep.rows, rows, model, W, H)


def test_yahoo_ccdpp_vs_reference(pmf, reference):
    train, probe = _data("yahoo-ccdpp")
    A = pmf.RatingsMatrix.from_triplets(train, 1000990, 624961)
    model, rep = pmf.ccdpp_train(pmf.CcdConfig(k=100, lam=0.05, outer_iters=1, inner_iters=15, seed=1), A, probe)
    del A
    M = reference.matrix(train, 1000990, 624961, "_f32")
    W, H, rows, _, _ = M.ccdpp_stage_loop(100, 0.05, 1, 15, 1, probe, workers=CORES)
    _compare("yahoo-ccdpp", rep.rows, rows, model, W, H)


def test_netflix_skew_ccdpp_vs_reference(pmf, reference):
    """Power-law users at the Netflix shape (datagen user_skew 0.5: rows of up to thousands of entries,
    the skew of the real Netflix data), CCD++ k=40, 2 outer iterations."""
    train, probe = _data("netflix-skew-ccdpp")
    A = pmf.RatingsMatrix.from_triplets(train, 480189, 17770)
    assert np.diff(A.row_start).max() > 2000  # long CSR rows are exercised
    model, rep = pmf.ccdpp_train(pmf.CcdConfig(k=40, lam=0.05, outer_iters=2, inner_iters=15, seed=1), A, probe)
    M = reference.matrix(train, 480189, 17770, "_f32")
    W, H, rows, _, _ = M.ccdpp_stage_loop(40, 0.05, 2, 15, 1, probe, workers=CORES)
    _compare("netflix-skew-ccdpp", rep.rows, rows, model, W, H)
