"""The multi-rank library path on one GPU: a device group of 2 / 3 ranks in one process
(pmf_ctx_create_group; num_gpus > 1 in the whole-call API, the reference's `workers`, ccd.hpp:39,
als.hpp:30).  Every rank owns a CSR row block and a CSC column block from partition_balanced
(runtime.hpp:91-136) in the padded index space, and the all-gathers of u / v (CCD++) and of the W / H
blocks (ALS) are device-to-device pushes between the ranks' replicated vectors -- the same layouts,
row / column maps, out_off offsets and block exchanges the NCCL ranks use, with only the transport
swapped.  On a 1-GPU box the ranks share cuda:0 (loopback).

Each output's sum runs over the same segments and units in the same order whatever rank owns it, so
where the layouts keep one gather panel (these shapes) the trajectory is bitwise the one-device
trajectory -- the analogue of the reference's worker-count invariance (tests/ccd_test.cpp:347-367,
tests/als_test.cpp:137-156).  The objective sums the ranks' row-block losses in rank order (FP64), so
it agrees to ~1e-15 rather than bitwise."""
import numpy as np
import pytest

from conftest import frob_rel, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mid(oracle):
    data = oracle.synth_ratings(6000, 2500, 3, 400000, 99)
    train, probe = oracle.carve_probe(data, 20000, 7)
    return train, probe


def _same_rows(r1, r2, tol=1e-12):
    for a, b in zip(r1, r2):
        assert rel(a.objective, b.objective) <= tol
        assert rel(a.train_rmse, b.train_rmse) <= tol
        assert a.rmse == b.rmse  # probe RMSE over the (bitwise equal) replicated model


@pytest.mark.parametrize("gpus", [2, 3])
def test_ccdpp_group_bitwise(pmf, mid, gpus):
    train, probe = mid
    A = pmf.RatingsMatrix.from_triplets(train, 6000, 2500)
    cfg = dict(k=8, lam=0.05, outer_iters=2, inner_iters=4, seed=1)
    m1, r1 = pmf.ccdpp_train(pmf.CcdConfig(workers=1, **cfg), A, probe)
    mg, rg = pmf.ccdpp_train(pmf.CcdConfig(workers=gpus, **cfg), A, probe)
    assert np.array_equal(m1.w, mg.w) and np.array_equal(m1.h, mg.h)
    _same_rows(r1.rows, rg.rows)
    assert rg.workers == gpus


@pytest.mark.parametrize("gpus", [2, 3])
def test_als_group_bitwise(pmf, mid, gpus):
    train, probe = mid
    A = pmf.RatingsMatrix.from_triplets(train, 6000, 2500)
    cfg = dict(k=10, lam=0.05, outer_iters=2, seed=1)
    m1, r1 = pmf.als_train(pmf.AlsConfig(workers=1, **cfg), A, probe)
    mg, rg = pmf.als_train(pmf.AlsConfig(workers=gpus, **cfg), A, probe)
    assert np.array_equal(m1.w, mg.w) and np.array_equal(m1.h, mg.h)
    _same_rows(r1.rows, rg.rows)


def test_group_context_matches_oracle_and_dist_plan(pmf, oracle, mid):
    """The resident group context: block plan = pmf_dist_plan's, trajectory = the oracle's."""
    train, probe = mid
    A = pmf.RatingsMatrix.from_triplets(train, 6000, 2500)
    ctx = pmf.Context(A, gpus=2)
    ctx.set_probe(probe)
    ctx.ccdpp_begin(pmf.CcdConfig(k=6, lam=0.05, outer_iters=3, inner_iters=3, seed=2))
    ctx.ccdpp_iterate(3)
    o, r, tr = ctx.metrics()
    mdl = ctx.model()
    W, H = mdl.w, mdl.h
    ctx.close()
    OA = oracle.from_triplets(train, 6000, 2500)
    OW, OH, rows, _, _ = oracle.ccdpp_train(OA, 6, 0.05, 3, 3, 2, probe)
    assert rel(o, float(rows[-1]["objective"])) < 1e-4 and rel(r, float(rows[-1]["rmse"])) < 1e-4
    assert frob_rel(W, OW) < 1e-3 and frob_rel(H, OH) < 1e-3


def test_group_multi_panel_layouts(pmf, oracle):
    """Gather spaces wider than one shared-memory panel (CSR: 40,000 items): the padded index space
    moves panel boundaries, so per-output sums may regroup -- within FP32 rounding of one device."""
    data = oracle.synth_ratings(3000, 40000, 3, 300000, 5)
    train, probe = oracle.carve_probe(data, 10000, 3)
    A = pmf.RatingsMatrix.from_triplets(train, 3000, 40000)
    cfg = dict(k=6, lam=0.05, outer_iters=2, inner_iters=3, seed=1)
    m1, r1 = pmf.ccdpp_train(pmf.CcdConfig(workers=1, **cfg), A, probe)
    mg, rg = pmf.ccdpp_train(pmf.CcdConfig(workers=2, **cfg), A, probe)
    for a, b in zip(r1.rows, rg.rows):
        assert rel(a.objective, b.objective) < 1e-5 and rel(a.rmse, b.rmse) < 1e-5
    assert frob_rel(mg.w, m1.w) < 1e-4 and frob_rel(mg.h, m1.h) < 1e-4


def test_group_rejects_bad_workers(pmf, mid):
    train, probe = mid
    A = pmf.RatingsMatrix.from_triplets(train, 6000, 2500)
    with pytest.raises(ValueError, match="workers must be >= 1"):
        pmf.Context(A, gpus=0)
