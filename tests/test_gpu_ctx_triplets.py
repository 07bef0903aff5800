"""Contexts built straight from triplets (pmf_ctx_create_from_triplets: CSR / CSC built and kept on the
device, layout streams filled on the device) against contexts from the host-built
RatingsMatrix: the layouts are the same, so CCD++, ALS and item/user-wise CCD give BITWISE the same
metrics, factors and residuals; every layout mode is exercised (one panel, several panels, wide panels
with the split promote / flat sweeps, gathers from global memory); and the input errors are the
reference's (sparse.hpp:82-92, :127-132)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _synth(m, n, per_row, seed):
    rng = np.random.default_rng(seed)
    rows, cols = [], []
    for i in range(m):
        k = int(rng.integers(max(1, per_row // 2), per_row * 3 // 2 + 1))
        cols.append(np.sort(rng.choice(n, min(k, n), replace=False)))
        rows.append(np.full(len(cols[-1]), i))
    t = np.zeros(sum(len(c) for c in cols), dtype=[("user", "<i4"), ("item", "<i4"), ("rating", "<f4")])
    t["user"] = np.concatenate(rows)
    t["item"] = np.concatenate(cols)
    t["rating"] = rng.integers(1, 6, len(t))
    return t[rng.permutation(len(t))]


def _pair(pmf, t, m, n):
    host = pmf.Context(pmf.RatingsMatrix.from_triplets(t, m, n))
    dev = pmf.Context.from_triplets(t, m, n)
    assert host.layout_info() == dev.layout_info()
    return host, dev


def _same(a, b):
    assert np.array_equal(np.array(a.metrics()), np.array(b.metrics()), equal_nan=True)  # (rmse: NaN, no probe)
    ma, mb = a.model(), b.model()
    assert np.array_equal(ma.w, mb.w) and np.array_equal(ma.h, mb.h)


def _run_all(pmf, t, m, n, k, probe=None, ccd=True, als=True):
    host, dev = _pair(pmf, t, m, n)
    for c in (host, dev):
        if probe is not None:
            c.set_probe(probe)
        c.ccdpp_begin(pmf.CcdConfig(k=k, lam=0.05, outer_iters=2, inner_iters=3, seed=1))
        c.ccdpp_iterate(2)
    _same(host, dev)
    rh, rd = host.residual(), dev.residual()
    assert np.array_equal(rh[0], rd[0]) and np.array_equal(rh[1], rd[1])
    if als:
        for c in (host, dev):
            c.als_begin(pmf.AlsConfig(k=k, lam=0.05, outer_iters=2, seed=1))
            c.als_iterate(2)
        _same(host, dev)
    if ccd:
        for c in (host, dev):
            c.ccd_begin(pmf.CcdConfig(k=k, lam=0.05, outer_iters=2, inner_iters=1, seed=1))
            c.ccd_iterate(2)
        _same(host, dev)
    return host.layout_info()


def test_ml100k_bitwise(pmf, ml100k):
    train, probe = ml100k
    li = _run_all(pmf, train, 943, 1682, 10, probe)
    assert li["csr"]["n_panels"] == 1 and li["csc"]["n_panels"] == 1


def test_several_panels_bitwise(pmf):
    t = _synth(60000, 3000, 40, 5)   # CSC gathers over 60K users: several panels, fused promote
    li = _run_all(pmf, t, 60000, 3000, 8)
    assert li["csc"]["n_panels"] > 1 and li["csc"]["promote_fused"]


@pytest.mark.slow
def test_wide_panels_split_promote_bitwise(pmf):
    t = _synth(20000, 400000, 80, 6)   # CSR gathers over 400K items, ~11 entries per segment: flat sweeps
    li = _run_all(pmf, t, 20000, 400000, 6, ccd=False)
    assert li["csr"]["n_panels"] > 1 and not li["csr"]["promote_fused"] and li["csr"]["rmw_sub"] > 1


def test_global_gathers_bitwise(pmf):
    t = _synth(20000, 400000, 6, 7)    # too short for panels: 32-bit indices, gathers from global memory
    li = _run_all(pmf, t, 20000, 400000, 4, ccd=False, als=False)
    assert not li["csr"]["smem"] and not li["csr"]["idx16"]


def test_empty_and_edge_shapes(pmf):
    t = np.array([(0, 0, 1.0), (2, 3, 2.0), (2, 1, 5.0)], dtype=[("user", "<i4"), ("item", "<i4"), ("rating", "<f4")])
    _run_all(pmf, t, 4, 5, 2)   # empty rows / columns
    c = pmf.Context.from_triplets(t[:0], 3, 2)   # no ratings
    c.ccdpp_begin(pmf.CcdConfig(k=2, lam=0.1, outer_iters=1, inner_iters=1, seed=1))
    c.ccdpp_iterate(1)
    assert c.metrics()[0] >= 0.0


def test_errors_match_host_builder(pmf):
    dt = [("user", "<i4"), ("item", "<i4"), ("rating", "<f4")]
    cases = [np.array([(0, 0, 1.0), (5, 0, 1.0)], dtype=dt),          # user out of range
             np.array([(0, 0, 1.0), (0, 9, 1.0)], dtype=dt),          # item out of range
             np.array([(0, 0, 1.0), (1, 1, np.nan)], dtype=dt),       # non-finite
             np.array([(1, 1, 1.0), (0, 0, 1.0), (1, 1, 2.0)], dtype=dt)]  # duplicate
    for t in cases:
        with pytest.raises(Exception) as eh:
            pmf.RatingsMatrix.from_triplets(t, 3, 3)
        with pytest.raises(Exception) as ed:
            pmf.Context.from_triplets(t, 3, 3)
        assert type(eh.value) is type(ed.value) and str(eh.value) == str(ed.value)


@pytest.mark.slow
def test_netflix_shape_bitwise(pmf):
    """BASELINE configs[2] bytes (bench.make_data): one CCD++ outer iteration (k=40, T=15) and one ALS
    iteration on a context from triplets and on one from the host matrix -- bitwise the same."""
    import bench
    train, probe = bench.make_data("netflix-ccdpp")
    host, dev = _pair(pmf, train, 480189, 17770)
    for c in (host, dev):
        c.set_probe(probe)
        c.ccdpp_begin(pmf.CcdConfig(k=40, lam=0.05, outer_iters=1, inner_iters=15, seed=1))
        c.ccdpp_iterate(1)
    _same(host, dev)
    for c in (host, dev):
        c.als_begin(pmf.AlsConfig(k=40, lam=0.05, outer_iters=1, seed=1))
        c.als_iterate(1)
    _same(host, dev)
    host.close()
    dev.close()


def test_large_k_bitwise(pmf, ml100k):
    """k > 64: ALS on the CTA-per-system path (als_big_kernels.cu) reads the device CSR / CSC the same way."""
    train, probe = ml100k
    _run_all(pmf, train, 943, 1682, 72, probe, ccd=False)
