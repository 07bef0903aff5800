#!/bin/bash
for sp in 0 1 2 3; do
  echo "== PMF_SPLIT_PROMOTE=$sp"
  PMF_SPLIT_PROMOTE=$sp python - <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import bench, paper_1511_02433_b200 as P
train, probe, A = bench.make_data("netflix-ccdpp")
ctx = P.Context(A); ctx.set_probe(probe)
ctx.ccdpp_begin(P.CcdConfig(k=40, lam=0.05, outer_iters=1, inner_iters=15, seed=1))
ctx.ccdpp_iterate(2)
print("graph iter s:", [round(x, 4) for x in ctx.ccdpp_iterate(2)], "metrics", ctx.metrics())
PY
done
