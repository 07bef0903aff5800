"""Wall time of top_n_batch (pmf_top_n, copies included) for every user of the Netflix-shape matrix
(k=40, count=10, rated items excluded).  The reference's top_n is timed by `bench.py --impl reference`."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1511_02433_b200 as P  # noqa: E402

train, probe = bench.make_data("netflix-ccdpp")
A = P.RatingsMatrix.from_triplets(train, *bench.CONFIGS["netflix-ccdpp"][:2])
rng = np.random.default_rng(1)
model = P.FactorModel(rng.normal(0, 0.3, (A.m, 40)).astype(np.float32), rng.normal(0, 0.3, (A.n, 40)).astype(np.float32))
users = np.arange(A.m, dtype=np.int32)
P.top_n_batch(model, users[:1000], 10, a=A)  # warm-up
for rep in range(2):
    t0 = time.perf_counter()
    items, scores, counts = P.top_n_batch(model, users, 10, a=A)
    print(f"top_n_batch all {A.m} users: {time.perf_counter() - t0:.3f} s", file=sys.stderr)
