"""Item/user-wise CCD epoch time at the Netflix (k=40) and ML-10M (k=10) shapes on the device.  The
reference's ccd_train is timed by `bench.py --impl reference`."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1511_02433_b200 as P  # noqa: E402

for cfg in ("netflix-ccdpp", "ml10m-als"):
    m, n, ntr, npr, k, *_ = bench.CONFIGS[cfg]
    k = 40 if cfg.startswith("netflix") else 10
    train, probe = bench.make_data(cfg)
    A = P.RatingsMatrix.from_triplets(train, *bench.CONFIGS[cfg][:2])
    ctx = P.Context(A)
    ctx.ccd_begin(P.CcdConfig(k=k, lam=0.05, outer_iters=3, inner_iters=1, seed=1))
    secs = ctx.ccd_iterate(3)
    print(f"{cfg} k={k}: GPU CCD epoch s {list(secs)} metrics {ctx.metrics()}", file=sys.stderr)
    ctx.close()
