#!/bin/bash
# ALS timing at Netflix k=40 (tensor-core 3xTF32 gram vs SIMT FP32 gram) + ML-100K parity vs oracle.
for mode in tc simt; do
  if [ $mode = simt ]; then export PMF_ALS_SIMT=1; else unset PMF_ALS_SIMT; fi
  echo "== $mode"
  python - <<'PY'
import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
import bench, paper_1511_02433_b200 as P
from oracle.pyoracle import Oracle
O = Oracle()
d = O.synth_ratings(943, 1682, 3, 100000, 777); tr, pr = O.carve_probe(d, 10000, 5)
A = P.RatingsMatrix.from_triplets(tr, 943, 1682); OA = O.from_triplets(tr, 943, 1682)
m, rep = P.als_train(P.AlsConfig(k=10, lam=0.05, outer_iters=5, seed=1), A, pr)
W, H, rows = O.als_train(OA, 10, 0.05, 5, 1, pr)
print("ml100k k=10 max rel obj/rmse:", max(abs(r.objective - g["objective"]) / g["objective"] for r, g in zip(rep.rows, rows)),
      max(abs(r.rmse - g["rmse"]) / g["rmse"] for r, g in zip(rep.rows, rows)))
for k in (40, 32, 20):
    m, rep = P.als_train(P.AlsConfig(k=k, lam=0.05, outer_iters=3, seed=1), A, pr)
    W, H, rows = O.als_train(OA, k, 0.05, 3, 1, pr)
    print(f"ml100k k={k} max rel obj/rmse:", max(abs(r.objective - g["objective"]) / g["objective"] for r, g in zip(rep.rows, rows)),
          max(abs(r.rmse - g["rmse"]) / g["rmse"] for r, g in zip(rep.rows, rows)))
train, probe, A = bench.make_data("netflix-ccdpp")
ctx = P.Context(A); ctx.set_probe(probe)
ctx.als_begin(P.AlsConfig(k=40, lam=0.05, outer_iters=1, seed=1))
s = ctx.als_iterate(3)
print("netflix k=40 ALS s/iter:", [round(x, 4) for x in s], "metrics", ctx.metrics())
PY
done
