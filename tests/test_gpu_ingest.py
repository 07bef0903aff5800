"""GPU ingestion: RatingsMatrix::from_triplets (sparse.hpp:73-149) built on the
device must equal the host build -- itself pinned to the reference (tests/test_abi.py) -- bit for bit,
and raise the same errors with the same messages (sparse.hpp:82-92 input-order validation,
:127-132 first duplicate in row order)."""
import numpy as np
import pytest

import datagen

pytestmark = pytest.mark.gpu
FIELDS = ("row_start", "col_of", "val_row", "col_start", "row_of", "val_col")


def _same(A, B):
    for f in FIELDS:
        assert np.array_equal(getattr(A, f), getattr(B, f)), f


def test_from_triplets_gpu_matches_host(pmf, oracle, ml100k):
    train, _ = ml100k
    _same(pmf.RatingsMatrix.from_triplets(train, 943, 1682, device=True),
          pmf.RatingsMatrix.from_triplets(train, 943, 1682))
    perm = np.random.default_rng(3).permutation(len(train))
    _same(pmf.RatingsMatrix.from_triplets(train[perm], 943, 1682, device=True),
          pmf.RatingsMatrix.from_triplets(train, 943, 1682))
    # empty rows and columns, shapes that are not powers of two
    t = oracle.random_triplets(57, 41, 300, 9)
    _same(pmf.RatingsMatrix.from_triplets(t, 70, 45, device=True), pmf.RatingsMatrix.from_triplets(t, 70, 45))
    E = pmf.RatingsMatrix.from_triplets([], 4, 2, device=True)
    assert E.nnz() == 0 and list(E.row_start) == [0] * 5 and list(E.col_start) == [0] * 3


@pytest.mark.slow
def test_from_triplets_gpu_large(pmf):
    train, _ = datagen.synth_ratings(200000, 30000, 3, 3_000_000, 0, 11)
    _same(pmf.RatingsMatrix.from_triplets(train, 200000, 30000, device=True),
          pmf.RatingsMatrix.from_triplets(train, 200000, 30000))


@pytest.mark.parametrize("trip,m,n,exc", [
    ([(0, 0, 1.0), (5, 0, 1.0), (0, 9, 1.0)], 3, 3, IndexError),       # first bad: user 5
    ([(0, 0, 1.0), (0, 9, 1.0), (5, 0, 1.0)], 3, 3, IndexError),       # first bad: item 9
    ([(0, -1, 1.0)], 3, 3, IndexError),
    ([(1, 1, 1.0), (0, 0, float("nan"))], 3, 3, ValueError),
    ([(2, 1, 1.0), (0, 2, 2.0), (2, 1, 3.0), (0, 2, 1.0)], 3, 3, ValueError),  # duplicates: user 0 first
])
def test_from_triplets_gpu_errors(pmf, trip, m, n, exc):
    with pytest.raises(exc) as host:
        pmf.RatingsMatrix.from_triplets(trip, m, n)
    with pytest.raises(exc) as dev:
        pmf.RatingsMatrix.from_triplets(trip, m, n, device=True)
    assert str(dev.value) == str(host.value)
