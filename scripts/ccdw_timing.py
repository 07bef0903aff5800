"""Item/user-wise CCD epoch time at the Netflix shape (k=40) on the device, and the reference's
ccd_train on the ML-10M shape (single worker, as the reference always runs it)."""
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
    train, probe, A = bench.make_data(cfg)
    ctx = P.Context(A)
    ctx.ccd_begin(P.CcdConfig(k=k, lam=0.05, outer_iters=3, inner_iters=1, seed=1))
    secs = ctx.ccd_iterate(3)
    print(f"{cfg} k={k}: GPU CCD epoch s {list(secs)} metrics {ctx.metrics()}", file=sys.stderr)
    ctx.close()
    if cfg.startswith("ml10m"):
        from oracle.pyoracle import Reference
        M = Reference().matrix(train, m, n, "_f32")
        t0 = time.perf_counter()
        W, H, rows = M.ccd_train(k, 0.05, 1, 1)
        print(f"{cfg} reference ccd_train 1 epoch: {rows['seconds'][0]:.2f} s (1 worker)", file=sys.stderr)
