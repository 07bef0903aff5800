#!/bin/bash
# ALS timing at Netflix k=40 (tensor-core 3xTF32 gram vs SIMT FP32 gram); parity lives in tests/test_gpu_als.py.
for mode in tc simt; do
  if [ $mode = simt ]; then export PMF_ALS_SIMT=1; else unset PMF_ALS_SIMT; fi
  echo "== $mode"
  python - <<'PY'
import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
import bench, paper_1511_02433_b200 as P
train, probe, A = bench.make_data("netflix-ccdpp")
ctx = P.Context(A); ctx.set_probe(probe)
ctx.als_begin(P.AlsConfig(k=40, lam=0.05, outer_iters=1, seed=1))
s = ctx.als_iterate(3)
print("netflix k=40 ALS s/iter:", [round(x, 4) for x in s], "metrics", ctx.metrics())
PY
done
