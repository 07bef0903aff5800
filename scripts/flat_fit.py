"""Per-CTA timing of the flat (segmented-stream) plain sweeps with the static partition (PMF_STEAL=0),
dumped with each CTA's entries and units for fitting the flat partition cost model:
    PMF_STEAL=0 python scripts/flat_fit.py --config yahoo-ccdpp > gpurun_out/flat_fit.json"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1511_02433_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="yahoo-ccdpp")
a = ap.parse_args()
train, probe = bench.make_data(a.config)
A = P.RatingsMatrix.from_triplets(train, *bench.CONFIGS[a.config][:2])
ctx = P.Context(A)
ctx.ccdpp_begin(P.CcdConfig(k=2, lam=0.05, outer_iters=1, inner_iters=15, seed=1))
ctx.ccdpp_iterate(1)
out = {}
for side in (0, 1):
    runs = []
    for rep in range(3):
        clk, st = ctx.debug_sweep_profile(side, False)
        runs.append(((clk[:, 1] - clk[:, 0]) / 1e3).tolist())
    dur = [min(x) for x in zip(*runs)]
    out[side] = {"dur_us": dur, "units": (st[:, 0] + st[:, 1] + st[:, 2]).tolist(), "entries": st[:, 3].tolist(),
                 "pieces": st[:, 4].tolist()}
print(json.dumps(out))
