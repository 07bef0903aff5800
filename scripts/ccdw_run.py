"""Item/user-wise CCD epochs at the Netflix shape (experiment / ncu helper, not a bench line):
    python scripts/ccdw_run.py [epochs] [k]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1511_02433_b200 as P  # noqa: E402

ep = int(sys.argv[1]) if len(sys.argv) > 1 else 3
k = int(sys.argv[2]) if len(sys.argv) > 2 else 40
train, probe = bench.make_data("netflix-ccdpp")
A = P.RatingsMatrix.from_triplets(train, 480189, 17770)
ctx = P.Context(A)
ctx.set_probe(probe)
ctx.ccd_begin(P.CcdConfig(k=k, lam=0.05, outer_iters=ep + 1, inner_iters=1, seed=1))
ctx.ccd_iterate(1)
t = list(ctx.ccd_iterate(ep))
print(f"ccd k={k} s/epoch {np.mean(t):.5f} {t} metrics {ctx.metrics()}")
