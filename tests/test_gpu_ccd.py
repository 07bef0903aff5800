"""GPU parity tests for the CCD++ path (ccd.hpp:133-404) through the C-ABI, against the reference's
golden vectors, the committed reference trajectories and the oracle on the same seeded inputs.

Tolerances (north_star / SURVEY.md 8c): per-iteration objective, train RMSE and probe RMSE within
1e-4 relative of the reference float run; factors within 1e-3 relative Frobenius error.  FP32
reduction order differs from the reference's sequential sums, so results are not bitwise."""
import json
import os

import numpy as np
import pytest

import datagen

from conftest import frob_rel, rel

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_trajectories.json")))

FIX65 = [(0, 0, 5.0), (0, 2, 3.0), (0, 4, 1.0), (1, 1, 4.0), (1, 2, 2.0), (2, 0, 1.0), (2, 4, 5.0),
         (3, 1, 2.0), (3, 2, 4.5), (3, 4, 2.5), (5, 0, 3.5), (5, 1, 1.5), (5, 2, 2.0), (5, 4, 4.0)]
V0 = [0.8, -0.5, 1.2, 0.3, -1.0]
EXPECT_U = [2.0754716981132075, 0.22346368715083795, -2.4137931034482758, 0.68100358422939045, 0.0,
            0.13119533527696797]
EXPECT_V = [0.82163605483103141, 3.8874624185557933, 2.0249580990531117, 0.0, -0.72480018190921613]


def test_golden_rank_one_updates(pmf):
    """tests/ccd_test.cpp:253-280 / acceptance C2 (frozen from gen_fixture_values.py), FP32 band."""
    A = pmf.RatingsMatrix.from_triplets(FIX65, 6, 5)
    u = pmf.ccdpp_update_u(A, A.val_row, V0, 0.1)
    v = pmf.ccdpp_update_v(A, A.val_col, u, 0.1)
    np.testing.assert_allclose(u, EXPECT_U, rtol=2e-6, atol=1e-6)
    np.testing.assert_allclose(v, EXPECT_V, rtol=2e-6, atol=1e-6)
    assert u[4] == 0.0 and v[3] == 0.0  # empty row / column -> 0


def test_closed_form_stage_answers(pmf):
    one = pmf.RatingsMatrix.from_triplets([(0, 0, 1.0)], 1, 1)
    rr, rc = pmf.ccdpp_build_rhat(one, one.val_row, one.val_col, [2.0], [3.0])
    assert rr[0] == 7.0 and rc[0] == 7.0                       # ccd_test.cpp:203-210: 1 + 2*3
    rr, rc = pmf.ccdpp_writeback(one, rr, rc, [2.0], [3.0])
    assert rr[0] == 1.0 and rc[0] == 1.0                       # ccd_test.cpp:306-318: 7 - 2*3
    six = pmf.RatingsMatrix.from_triplets([(0, 0, 6.0)], 1, 1)
    assert pmf.ccdpp_update_u(six, six.val_row, [2.0], 0.0)[0] == 3.0    # 6*2/2^2
    assert pmf.ccdpp_update_u(six, six.val_row, [0.0], 0.5)[0] == 0.0    # v = 0 -> 0
    assert pmf.ccdpp_update_u(six, six.val_row, [0.0], 0.0)[0] == 0.0    # den == 0 -> 0


def test_build_rhat_skip_and_oracle(pmf, oracle):
    """build skips rows with u_i == 0 (ccd.hpp:142) and matches the oracle bitwise in both layouts."""
    t = oracle.random_triplets(9, 7, 30, 31)
    A = pmf.RatingsMatrix.from_triplets(t, 9, 7)
    O = oracle.from_triplets(t, 9, 7)
    rng = np.random.default_rng(5)
    u = rng.uniform(-1, 1, 9).astype(np.float32); u[[1, 4]] = 0.0
    v = rng.uniform(-1, 1, 7).astype(np.float32)
    r0 = rng.uniform(-2, 2, A.nnz()).astype(np.float32)
    r0c = r0[np.argsort(O.xlink)]  # same residual in CSC order
    rr, rc = pmf.ccdpp_build_rhat(A, r0, r0c, u, v)
    er, ec = oracle.build_rhat(O, r0, r0c, u, v)
    assert np.array_equal(rr, er) and np.array_equal(rc, ec)
    assert np.array_equal(rc[O.xlink], rr)  # layouts bitwise equal through the cross-link
    wr, wc = pmf.ccdpp_writeback(A, rr, rc, u, v)
    xr, xc, _, _ = oracle.writeback(O, er, ec, u, v)
    assert np.array_equal(wr, xr) and np.array_equal(wc, xc)


def test_update_u_v_vs_oracle_random(pmf, oracle):
    t = oracle.random_triplets(300, 200, 6000, 12)
    A = pmf.RatingsMatrix.from_triplets(t, 300, 200)
    O = oracle.from_triplets(t, 300, 200)
    rng = np.random.default_rng(1)
    v = rng.uniform(-1, 1, 200).astype(np.float32)
    u_gpu = pmf.ccdpp_update_u(A, A.val_row, v, 0.05)
    u_ref = oracle.update_u(O, O.val_row, v, 0.05)
    np.testing.assert_allclose(u_gpu, u_ref, rtol=1e-5, atol=1e-6)
    v_gpu = pmf.ccdpp_update_v(A, A.val_col, u_ref, 0.05)
    v_ref = oracle.update_v(O, O.val_col, u_ref, 0.05)
    np.testing.assert_allclose(v_gpu, v_ref, rtol=1e-5, atol=1e-6)


def _check_rows(rep_rows, gold_rows, tol=1e-4):
    for r, g in zip(rep_rows, gold_rows):
        assert rel(r.objective, g["objective"]) < tol, (r, g)
        assert rel(r.train_rmse, g["train_rmse"]) < tol, (r, g)
        if not np.isnan(g["rmse"]):
            assert rel(r.rmse, g["rmse"]) < tol, (r, g)


def test_ccdpp_ml100k_trajectory(pmf, oracle, ml100k):
    """BASELINE configs[0]: ML-100K shape, k=10, lambda=0.05, 5 outer x 15 inner."""
    train, probe = ml100k
    A = pmf.RatingsMatrix.from_triplets(train, 943, 1682)
    model, rep = pmf.ccdpp_train(pmf.CcdConfig(k=10, lam=0.05, outer_iters=5, inner_iters=15, seed=1), A, probe)
    assert len(rep.rows) == 5
    _check_rows(rep.rows, GOLD["ccdpp_ml100k_k10_f32"]["rows"])
    _check_rows(rep.rows, GOLD["ccdpp_ml100k_k10_f64"]["rows"])
    O = oracle.from_triplets(train, 943, 1682)
    W, H, rows, _, _ = oracle.ccdpp_train(O, 10, 0.05, 5, 15, 1, probe)
    assert frob_rel(model.w, W) < 1e-3 and frob_rel(model.h, H) < 1e-3
    # reported metrics are the metrics of the returned model (oracle evaluates the GPU factors)
    obj, loss = oracle.objective(O, model.w, model.h, float(np.float32(0.05)))
    assert rel(rep.rows[-1].objective, obj) < 1e-12
    assert rel(rep.rows[-1].rmse, oracle.rmse(model.w, model.h, probe)) < 1e-12


def test_ccdpp_deterministic(pmf, ml100k):
    train, probe = ml100k
    A = pmf.RatingsMatrix.from_triplets(train, 943, 1682)
    cfg = pmf.CcdConfig(k=4, lam=0.05, outer_iters=2, inner_iters=3, seed=6)
    m1, r1 = pmf.ccdpp_train(cfg, A, probe)
    m2, r2 = pmf.ccdpp_train(cfg, A, probe)
    assert m1 == m2
    assert [r.objective for r in r1.rows] == [r.objective for r in r2.rows]


def test_small_exact_fixture_and_residual(pmf, oracle):
    """random_triplets(40,30,350,71), k=3, lambda=0.1, 4 x 3 (tests/ccd_test.cpp:369-397): factors and
    the final residual vs the reference, residual true to the factors, layouts bitwise equal."""
    t = oracle.random_triplets(40, 30, 350, 71)
    A = pmf.RatingsMatrix.from_triplets(t, 40, 30)
    O = oracle.from_triplets(t, 40, 30)
    g = GOLD["ccdpp_small_k3_f32"]
    ctx = pmf.Context(A)
    ctx.ccdpp_begin(pmf.CcdConfig(k=3, lam=0.1, outer_iters=4, inner_iters=3, seed=9))
    for it in range(4):
        ctx.ccdpp_iterate(1)
        obj, _, tr = ctx.metrics()
        assert rel(obj, g["rows"][it]["objective"]) < 1e-4
    model = ctx.model()
    assert frob_rel(model.w, np.array(g["W"]).reshape(40, 3)) < 1e-3
    assert frob_rel(model.h, np.array(g["H"]).reshape(30, 3)) < 1e-3
    rr, rc = ctx.residual()
    assert np.array_equal(rc[O.xlink], rr)      # both layouts bitwise equal (testutil.hpp:266-272)
    pred = np.einsum("ik,ik->i", model.w[np.repeat(np.arange(40), np.diff(O.row_start))].astype(np.float64),
                     model.h[O.col_of].astype(np.float64))
    assert np.max(np.abs(rr - (O.val_row - pred))) < 1e-4   # residual_max_error, FP32 band
    assert frob_rel(rr, np.array(g["r_row"])) < 1e-3
    ctx.close()


def test_planted_recovery(pmf, oracle):
    """acceptance C6 / ccd_test.cpp:332-345: planted rank-2 20x15, lambda=1e-6, 15 x 15."""
    t = oracle.planted_full(20, 15, 2, 0.01, 42)
    A = pmf.RatingsMatrix.from_triplets(t, 20, 15)
    _, rep = pmf.ccdpp_train(pmf.CcdConfig(k=2, lam=1e-6, outer_iters=15, inner_iters=15, seed=3), A)
    assert rep.final_objective <= 1e-6
    assert np.isnan(rep.final_rmse)


def test_monotone_objective(pmf, oracle):
    t = oracle.random_triplets(60, 45, 900, 505)
    A = pmf.RatingsMatrix.from_triplets(t, 60, 45)
    _, rep = pmf.ccdpp_train(pmf.CcdConfig(k=3, lam=0.1, outer_iters=10, inner_iters=2, seed=21), A)
    objs = [r.objective for r in rep.rows]
    assert all(b <= a * (1 + 1e-5) for a, b in zip(objs, objs[1:]))


def test_edge_cases(pmf):
    # empty rows and columns, single entry, lambda = 0 with empty rows (den == 0 -> 0)
    t = [(0, 0, 3.0), (2, 3, 1.0), (2, 0, 2.0)]
    A = pmf.RatingsMatrix.from_triplets(t, 5, 6)
    model, rep = pmf.ccdpp_train(pmf.CcdConfig(k=2, lam=0.0, outer_iters=2, inner_iters=2, seed=1), A)
    assert np.all(model.w[[1, 3, 4]] == 0) and np.all(model.h[[1, 2, 4, 5]] == 0)
    assert np.all(np.isfinite(model.w)) and np.all(np.isfinite(model.h))
    # empty matrix
    E = pmf.RatingsMatrix.from_triplets([], 3, 4)
    model, rep = pmf.ccdpp_train(pmf.CcdConfig(k=2, lam=0.1, outer_iters=1, inner_iters=1), E)
    assert rep.rows[0].objective == pytest.approx(0.1 * float((model.h.astype(np.float64) ** 2).sum()), rel=1e-6)


def test_validation_errors(pmf):
    A = pmf.RatingsMatrix.from_triplets([(0, 0, 1.0)], 2, 2)
    with pytest.raises(ValueError):
        pmf.ccdpp_train(pmf.CcdConfig(k=0), A)
    with pytest.raises(ValueError):
        pmf.ccdpp_train(pmf.CcdConfig(lam=-1.0), A)
    with pytest.raises(ValueError):
        pmf.ccdpp_train(pmf.CcdConfig(), A, [(5, 0, 1.0)])   # probe outside dims (ccd.hpp:298-303)


@pytest.mark.slow
def test_multi_panel_layout_vs_oracle(pmf, oracle):
    """A shape whose CSC side needs several shared-memory row panels (m > 18.7K rows) and split
    units (columns longer than 4096 entries): exercises the partial / finalize path."""
    m, n = 60000, 300
    t = oracle.synth_ratings(m, n, 3, 600000, 99)
    A = pmf.RatingsMatrix.from_triplets(t, m, n)
    O = oracle.from_triplets(t, m, n)
    cfg = pmf.CcdConfig(k=3, lam=0.05, outer_iters=2, inner_iters=3, seed=4)
    model, rep = pmf.ccdpp_train(cfg, A)
    W, H, rows, _, _ = oracle.ccdpp_train(O, 3, 0.05, 2, 3, 4)
    for r, g in zip(rep.rows, rows):
        assert rel(r.objective, g["objective"]) < 1e-4
    assert frob_rel(model.w, W) < 1e-3 and frob_rel(model.h, H) < 1e-3


def test_distributed_context_single_rank_nccl(pmf, ml100k):
    """pmf_ctx_create_dist with a 1-rank NCCL communicator: the all-gathers run inside the captured
    CUDA graph and the result equals the plain context bit-for-bit."""
    train, probe = ml100k
    A = pmf.RatingsMatrix.from_triplets(train, 943, 1682)
    cfg = pmf.CcdConfig(k=5, lam=0.05, outer_iters=2, inner_iters=3, seed=2)
    a = pmf.Context(A)
    a.ccdpp_begin(cfg)
    a.ccdpp_iterate(2)
    b = pmf.Context(A, rank=0, world=1, nccl_id=pmf.nccl_unique_id())
    b.ccdpp_begin(cfg)
    b.ccdpp_iterate(2)
    assert a.model() == b.model()
    assert a.metrics()[0] == b.metrics()[0]
    b.als_begin(pmf.AlsConfig(k=5, lam=0.05, outer_iters=1, seed=2))
    b.als_iterate(1)
    a.als_begin(pmf.AlsConfig(k=5, lam=0.05, outer_iters=1, seed=2))
    a.als_iterate(1)
    assert a.model() == b.model()
    a.close()
    b.close()


@pytest.mark.slow
def test_global_gather_layout_vs_oracle(pmf, oracle):
    """Many short rows over a wide item space (Yahoo-like sparsity): both sides fall back to the
    non-panel layout that gathers the factor vectors from global memory with 32-bit indices."""
    m, n = 40000, 70000
    t = oracle.random_triplets(m, n, 400000, 5)
    A = pmf.RatingsMatrix.from_triplets(t, m, n)
    O = oracle.from_triplets(t, m, n)
    cfg = pmf.CcdConfig(k=4, lam=0.05, outer_iters=2, inner_iters=3, seed=8)
    model, rep = pmf.ccdpp_train(cfg, A)
    W, H, rows, _, _ = oracle.ccdpp_train(O, 4, 0.05, 2, 3, 8)
    for r, g in zip(rep.rows, rows):
        assert rel(r.objective, g["objective"]) < 1e-4
    assert frob_rel(model.w, W) < 1e-3 and frob_rel(model.h, H) < 1e-3


@pytest.mark.slow
def test_split_promote_wide_panels_residual(pmf, oracle):
    """Both gather spaces wider than one shared-memory panel (> 56K): the 14 plain sweeps of a step
    stage one vector per panel, and the promote (2 / 3 staged vectors, ccd.hpp:133-151 + :209-214)
    runs as a residual pass over 2 sub-panels + a plain sweep.  Trajectory vs the oracle, residual
    layouts bitwise equal (testutil.hpp:266-272) and true to the factors."""
    m, n = 62000, 60000
    t = oracle.random_triplets(m, n, 2_500_000, 13)
    A = pmf.RatingsMatrix.from_triplets(t, m, n)
    O = oracle.from_triplets(t, m, n)
    ctx = pmf.Context(A)
    lay = ctx.layout_info()
    for side in ("csr", "csc"):
        assert lay[side]["n_panels"] == 2 and not lay[side]["promote_fused"] and lay[side]["rmw_sub"] == 2
    k, outer, inner = 3, 2, 3
    ctx.ccdpp_begin(pmf.CcdConfig(k=k, lam=0.05, outer_iters=outer, inner_iters=inner, seed=4))
    W, H, rows, _, _ = oracle.ccdpp_train(O, k, 0.05, outer, inner, 4)
    for it in range(outer):
        ctx.ccdpp_iterate(1)
        assert rel(ctx.metrics()[0], rows[it]["objective"]) < 1e-4
    model = ctx.model()
    assert frob_rel(model.w, W) < 1e-3 and frob_rel(model.h, H) < 1e-3
    rr, rc = ctx.residual()
    assert np.array_equal(rc[O.xlink], rr)
    ri = np.repeat(np.arange(m), np.diff(O.row_start))
    pred = np.einsum("ik,ik->i", model.w[ri].astype(np.float64), model.h[O.col_of].astype(np.float64))
    assert np.max(np.abs(rr - (O.val_row - pred))) < 1e-4
    ctx.close()


def test_release_cached_memory(pmf, ml100k):
    """Destroyed contexts' device blocks are cached (no cudaFree in the next call) and returned to the
    driver on request; training after the release allocates afresh and gives the same model."""
    train, probe = ml100k
    A = pmf.RatingsMatrix.from_triplets(train, 943, 1682)
    cfg = pmf.CcdConfig(k=5, lam=0.05, outer_iters=2, inner_iters=3, seed=2)
    m1, _ = pmf.ccdpp_train(cfg, A, probe)
    assert pmf.release_cached_memory() > 0
    assert pmf.release_cached_memory() == 0
    m2, _ = pmf.ccdpp_train(cfg, A, probe)
    assert m1 == m2


def test_alloc_cache_off_same_model(pmf, tmp_path):
    """PMF_NO_ALLOC_CACHE=1 (plain cudaMalloc, pageable layout arrays through the staging buffers) trains
    the same model bit for bit as the cached device blocks + page-locked layout blocks (5M ratings: the
    layout arrays are above the 16 MB page-locked threshold)."""
    import subprocess
    import sys
    m, n = 30000, 2000
    train, _ = datagen.synth_ratings(m, n, 3, 5_000_000, 1000, 11)
    A = pmf.RatingsMatrix.from_triplets(train, m, n)
    cfg = pmf.CcdConfig(k=4, lam=0.05, outer_iters=2, inner_iters=3, seed=2)
    m1, _ = pmf.ccdpp_train(cfg, A)
    np.save(tmp_path / "train.npy", train)
    code = (
        "import sys, numpy as np; sys.path.insert(0, sys.argv[1]); import paper_1511_02433_b200 as P\n"
        "t = np.load(sys.argv[2]); A = P.RatingsMatrix.from_triplets(t, 30000, 2000)\n"
        "m, _ = P.ccdpp_train(P.CcdConfig(k=4, lam=0.05, outer_iters=2, inner_iters=3, seed=2), A)\n"
        "np.save(sys.argv[3], m.w); np.save(sys.argv[4], m.h)\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PMF_NO_ALLOC_CACHE="1")
    subprocess.run([sys.executable, "-c", code, root, str(tmp_path / "train.npy"), str(tmp_path / "w.npy"),
                    str(tmp_path / "h.npy")], check=True, env=env, timeout=300)
    assert np.array_equal(np.load(tmp_path / "w.npy"), m1.w) and np.array_equal(np.load(tmp_path / "h.npy"), m1.h)


def test_set_model_rebuilds_residual(pmf, oracle, ml100k):
    """set_model installs a model together with its residual (A - W H^T, ascending t): the residual
    read back matches the oracle's from-scratch residual, and iterating from the installed model
    follows an uninterrupted run (the stored residual differs only by rounding history)."""
    train, probe = ml100k
    A = pmf.RatingsMatrix.from_triplets(train, 943, 1682)
    cfg = pmf.CcdConfig(k=10, lam=0.05, outer_iters=3, inner_iters=15, seed=1)
    ref = pmf.Context(A); ref.set_probe(probe); ref.ccdpp_begin(cfg)
    ref.ccdpp_iterate(1)
    m1 = ref.model()
    ref.ccdpp_iterate(1)
    o_ref, r_ref, _ = ref.metrics()
    ctx = pmf.Context(A); ctx.set_probe(probe); ctx.ccdpp_begin(cfg)
    ctx.set_model(m1)
    rr, rc = ctx.residual()
    exp = A.val_row.astype(np.float64) - np.einsum(
        "ek,ek->e", m1.w[np.repeat(np.arange(943), np.diff(A.row_start))].astype(np.float64),
        m1.h[A.col_of].astype(np.float64))
    assert np.max(np.abs(rr - exp)) < 1e-4
    assert np.array_equal(rr[np.argsort(oracle.from_triplets(train, 943, 1682).xlink)], rc)
    ctx.ccdpp_iterate(1)
    o, r, _ = ctx.metrics()
    assert rel(o, o_ref) < 1e-5 and rel(r, r_ref) < 1e-5
    ref.close(); ctx.close()


@pytest.mark.parametrize("k,T", [(10, 15), (1, 1), (33, 2)])
def test_small_path_matches_graph_schedule(ml100k, k, T):
    """ML-100K runs its whole outer iteration as one cluster kernel (small_kernels.cu); PMF_SMALL=0 keeps
    the CUDA-graph schedule of the large shapes.  Same layouts and per-entry arithmetic, different sum
    order: the trajectories agree to FP32 rounding, and each keeps its two residual copies bitwise equal
    (checked by the other tests of this file on the default path)."""
    import json
    import os
    import subprocess
    import sys
    code = r'''
import json, sys
sys.path.insert(0, sys.argv[1])
import paper_1511_02433_b200 as P
from oracle.pyoracle import Oracle
O = Oracle()
a = O.synth_ratings(943, 1682, 3, 100000, 777)
train, probe = O.carve_probe(a, 10000, 5)
A = P.RatingsMatrix.from_triplets(train, 943, 1682)
ctx = P.Context(A)
ctx.set_probe(probe)
ctx.ccdpp_begin(P.CcdConfig(k=int(sys.argv[2]), lam=0.05, outer_iters=3, inner_iters=int(sys.argv[3]), seed=1))
rows = []
for _ in range(3):
    ctx.ccdpp_iterate(1)
    rows.append(list(ctx.metrics()))
print(json.dumps({"rows": rows, "launches": ctx.launch_count()}))
'''
    from conftest import ROOT
    out = {}
    for flag in ("1", "0"):
        r = subprocess.run([sys.executable, "-c", code, ROOT, str(k), str(T)], env=dict(os.environ, PMF_SMALL=flag),
                           capture_output=True, text=True, timeout=240)
        assert r.returncode == 0, r.stderr[-2000:]
        out[flag] = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["1"]["launches"] == 1 and out["0"]["launches"] > 2 * T * k - 1
    for a, b in zip(out["1"]["rows"], out["0"]["rows"]):
        for x, y in zip(a, b):
            assert abs(x - y) <= 1e-5 * abs(y)
