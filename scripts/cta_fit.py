"""Fits per-CTA sweep time = a*entries + b_long*n_long + b_mid*n_mid + b_short*n_short + c from one
profiled sweep (pmf_ctx_debug_sweep_profile) per side; prints the coefficients in entry units."""
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
import paper_1511_02433_b200 as P  # noqa: E402

train, probe, A = bench.make_data(sys.argv[1] if len(sys.argv) > 1 else "netflix-ccdpp")
ctx = P.Context(A)
ctx.ccdpp_begin(P.CcdConfig(k=40, lam=0.05, outer_iters=1, inner_iters=15, seed=1))
ctx.ccdpp_iterate(1)
for side in (0, 1):
    rows = []
    for rep in range(3):
        clk, st = ctx.debug_sweep_profile(side, False)
        rows.append((clk[:, 1] - clk[:, 0]) / 1e3)
    d = np.median(np.array(rows), axis=0)
    X = np.column_stack([st[:, 3], st[:, 0], st[:, 1], st[:, 2], np.ones(len(d))]).astype(float)
    coef, *_ = np.linalg.lstsq(X, d, rcond=None)
    pred = X @ coef
    a = coef[0]
    print(f"side {side}: us/entry {a:.3e}  per-unit overhead in entries: long {coef[1]/a:.1f} mid {coef[2]/a:.1f} "
          f"short {coef[3]/a:.1f}  const {coef[4]:.1f} us; fit rms {np.sqrt(np.mean((pred-d)**2)):.2f} us; "
          f"dur min {d.min():.1f} max {d.max():.1f}")
    np.save(f"gpurun_out/cta_side{side}.npy", np.column_stack([d, st]))
