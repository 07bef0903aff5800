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
    a = ap.parse_args()
    m, n, ntr, npr, k, lam, inner, solver = bench.CONFIGS[a.config]
    train, probe, A = bench.make_data(a.config)
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


if __name__ == "__main__":
    main()
