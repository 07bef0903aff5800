"""End-to-end ccdpp_train timing at Netflix k=40 (3 outer iterations), repeated; PMF_VERBOSE=1 prints
the setup / iterate / download breakdown."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
import paper_1511_02433_b200 as P  # noqa: E402

train, probe = bench.make_data("netflix-ccdpp")
A = P.RatingsMatrix.from_triplets(train, 480189, 17770)
reps = int(os.environ.get("REPS", "3"))
for rep in range(reps):
    t0 = time.perf_counter()
    model, rep_ = P.ccdpp_train(P.CcdConfig(k=40, lam=0.05, outer_iters=int(os.environ.get("ITERS", "5")), inner_iters=15, seed=1), A, probe)
    print("e2e wall", round(time.perf_counter() - t0, 3), file=sys.stderr)
    del model
