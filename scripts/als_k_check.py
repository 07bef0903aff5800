"""ALS seconds per outer iteration at the Netflix shape for a given k (experiment helper, not a bench line):
    python scripts/als_k_check.py K [iters]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1511_02433_b200 as P  # noqa: E402

k = int(sys.argv[1])
it = int(sys.argv[2]) if len(sys.argv) > 2 else 3
train, probe = bench.make_data("netflix-als")
A = P.RatingsMatrix.from_triplets(train, 480189, 17770)
ctx = P.Context(A)
ctx.set_probe(probe)
ctx.als_begin(P.AlsConfig(k=k, lam=0.05, outer_iters=it + 1, seed=1))
ctx.als_iterate(1)
t = list(ctx.als_iterate(it))
print(f"k={k} ALS s/iter {np.mean(t):.5f} metrics {ctx.metrics()}")
