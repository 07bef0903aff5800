"""ML-100K CCD++ (configs[0] shape) per-iteration device time of the one-kernel small path at several
inner iteration counts T and ranks k: separates the per-sweep cost from the per-step cost."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1511_02433_b200 as P  # noqa: E402

train, probe = bench.make_data("ml100k-ccdpp")
m, n = bench.CONFIGS["ml100k-ccdpp"][:2]
A = P.RatingsMatrix.from_triplets(train, m, n)
for k, T in ((10, 1), (10, 5), (10, 15), (20, 15), (5, 15)):
    ctx = P.Context(A)
    ctx.ccdpp_begin(P.CcdConfig(k=k, lam=0.05, outer_iters=20, inner_iters=T, seed=1))
    ctx.ccdpp_iterate(3)
    t = np.median(ctx.ccdpp_iterate(10))
    print(f"k={k:3d} T={T:3d}: {t * 1e3:.3f} ms/iter, {t * 1e6 / (k * (2 * T + 1)):.2f} us per phase")
    ctx.close()
