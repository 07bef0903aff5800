"""Short, fixed workload for ncu captures (never a bench number): build the synthetic Netflix-shape
matrix, create the device context, run `--iters` CCD++ outer iterations (CUDA graph) and optionally
`--als` ALS epochs.

    ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 0 -c 4 \
        -o gpurun_out/prof python scripts/profile_run.py --iters 1
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1511_02433_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="netflix-ccdpp")
    ap.add_argument("--iters", type=int, default=1)
    ap.add_argument("--als", type=int, default=0)
    ap.add_argument("--profiling", action="store_true", help="per-sweep event timing (no graph)")
    ap.add_argument("--k", type=int, default=0, help="override the config's rank (fewer launches)")
    ap.add_argument("--cta", action="store_true", help="per-CTA timing of one plain / promote sweep per side")
    a = ap.parse_args()
    if a.cta:
        return cta_profile(a.config)
    m, n, ntr, npr, k, lam, inner, solver, skew = bench.CONFIGS[a.config]
    k = a.k or k
    train, probe = bench.make_data(a.config)
    A = P.RatingsMatrix.from_triplets(train, m, n)
    ctx = P.Context(A)
    if a.iters:
        ctx.ccdpp_begin(P.CcdConfig(k=k, lam=lam, outer_iters=a.iters, inner_iters=15, seed=1))
        if a.profiling:
            ctx.set_profiling(True)
        t0 = time.perf_counter()
        secs = ctx.ccdpp_iterate(a.iters)
        print("ccdpp iter s:", list(secs), "wall", time.perf_counter() - t0, file=sys.stderr)
        if a.profiling:
            print(ctx.kernel_stats(), file=sys.stderr)
    if a.als:
        ctx.als_begin(P.AlsConfig(k=k, lam=lam, outer_iters=a.als, seed=1))
        print("als iter s:", list(ctx.als_iterate(a.als)), file=sys.stderr)




def cta_profile(config):
    """python scripts/profile_run.py --cta [--config C]: per-CTA time spread of one plain / promote
    sweep per side (after one outer iteration at rank 4)."""
    import numpy as np
    m, n = bench.CONFIGS[config][:2]
    train, probe = bench.make_data(config)
    A = P.RatingsMatrix.from_triplets(train, m, n)
    ctx = P.Context(A)
    for side, li in ctx.layout_info().items():
        print(f"layout {side}: " + " ".join(f"{k}={v}" for k, v in li.items()))
    ctx.ccdpp_begin(P.CcdConfig(k=4, lam=0.05, outer_iters=1, inner_iters=15, seed=1))
    ctx.ccdpp_iterate(1)
    for side in (0, 1):
        for promote in (False, True):
            clk, st = ctx.debug_sweep_profile(side, promote)
            t0 = clk[:, 0].min()
            dur = (clk[:, 1] - clk[:, 0]) / 1e3
            end = (clk[:, 1] - t0) / 1e3
            print(f"side {side} promote {promote}: kernel {end.max():.1f} us; CTA dur min {dur.min():.1f} "
                  f"avg {dur.mean():.1f} max {dur.max():.1f}; start spread {(clk[:, 0].max() - t0) / 1e3:.1f} us")
            order = np.argsort(-dur)
            for c in list(order[:6]) + list(order[-3:]):
                print(f"   cta {c:3d} dur {dur[c]:7.1f} us  long {st[c, 0]:5d} mid {st[c, 1]:5d} short {st[c, 2]:5d} "
                      f"entries {st[c, 3]:8d} pieces {st[c, 4]} panel {st[c, 5]}")


if __name__ == "__main__":
    main()
