import sys, os, time
sys.path.insert(0, os.getcwd())
import bench, paper_1511_02433_b200 as P
train, probe, A = bench.make_data("netflix-ccdpp")
for rep in range(2):
    t0 = time.perf_counter()
    model, rep_ = P.ccdpp_train(P.CcdConfig(k=40, lam=0.05, outer_iters=3, inner_iters=15, seed=1), A, probe)
    print("e2e wall", time.perf_counter() - t0, file=sys.stderr)
