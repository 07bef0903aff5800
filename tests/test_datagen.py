"""The benchmark corpus generator (datagen/synth.cpp, tests/testutil.hpp:91-132 recipe on per-user
streams): exact counts, sorted unique (user, item), 1..5 stars, Zipf-skewed items, deterministic in
the seed; the power-law-user variant."""
import numpy as np

import datagen


def test_synth_ratings_recipe():
    tr, pr = datagen.synth_ratings(2000, 500, 3, 60000, 3000, 11)
    assert len(tr) == 60000 and len(pr) == 3000
    allt = np.concatenate([tr, pr])
    key = allt["user"].astype(np.int64) * 500 + allt["item"]
    assert len(np.unique(key)) == len(key)
    assert set(np.unique(allt["rating"])) <= {1.0, 2.0, 3.0, 4.0, 5.0}
    k_tr = tr["user"].astype(np.int64) * 500 + tr["item"]
    assert np.all(np.diff(k_tr) > 0)
    cnt = np.bincount(allt["item"], minlength=500)
    assert cnt[:10].sum() > cnt[-100:].sum()
    tr2, pr2 = datagen.synth_ratings(2000, 500, 3, 60000, 3000, 11)
    assert np.array_equal(tr, tr2) and np.array_equal(pr, pr2)


def test_synth_ratings_skewed_users():
    """user_skew > 0: power-law row lengths, the heaviest rows dense (every item), still exact and unique."""
    tr, pr = datagen.synth_ratings(5000, 800, 3, 400000, 4000, 3, user_skew=0.6)
    assert len(tr) == 400000 and len(pr) == 4000
    allt = np.concatenate([tr, pr])
    key = allt["user"].astype(np.int64) * 800 + allt["item"]
    assert len(np.unique(key)) == len(key)
    rows = np.bincount(allt["user"], minlength=5000)
    assert rows.max() == 800 and rows.max() > 8 * np.median(rows)
    assert np.all(np.diff(tr["user"].astype(np.int64) * 800 + tr["item"]) > 0)
