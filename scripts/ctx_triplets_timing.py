"""Netflix shape: a ready context from triplets on the device (pmf_ctx_create_from_triplets) vs through the
host RatingsMatrix + pmf_ctx_create; same layouts, one CCD++ iteration each, bitwise-equal metrics."""
import time, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, bench, paper_1511_02433_b200 as P
trn, probe = bench.make_data("netflix-ccdpp")
m, n = 480189, 17770
P.Context.from_triplets(trn[:100000], m, n).close()
for rep in range(2):
    t0 = time.perf_counter(); cd = P.Context.from_triplets(trn, m, n); td = time.perf_counter() - t0
    t0 = time.perf_counter(); ch = P.Context(P.RatingsMatrix.from_triplets(trn, m, n)); th = time.perf_counter() - t0
    print("ctx device", round(td, 3), "via host", round(th, 3), "same layouts", cd.layout_info() == ch.layout_info())
    for c in (cd, ch):
        c.set_probe(probe); c.ccdpp_begin(P.CcdConfig(k=40, lam=0.05, outer_iters=1, inner_iters=15, seed=1)); c.ccdpp_iterate(1)
    print("metrics equal", cd.metrics() == ch.metrics(), cd.metrics())
    cd.close(); ch.close()
