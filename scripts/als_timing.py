"""ALS s/iter at Netflix k=40 (env knobs: PMF_ALS_EXACT=3 previous Cholesky, =2 no factorisation)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
import paper_1511_02433_b200 as P  # noqa: E402

train, probe, A = bench.make_data("netflix-ccdpp")
ctx = P.Context(A)
ctx.set_probe(probe)
ctx.als_begin(P.AlsConfig(k=40, lam=0.05, outer_iters=1, seed=1))
s = ctx.als_iterate(3)
print(os.environ.get("PMF_ALS_EXACT", "-"), "netflix k=40 ALS s/iter:", [round(x, 5) for x in s], "metrics",
      ctx.metrics())
