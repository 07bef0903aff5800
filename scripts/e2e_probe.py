"""Breakdown of the end-to-end pmf_ccdpp_train call at Netflix shape (PMF_VERBOSE=1 prints setup)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import bench, paper_1511_02433_b200 as P
train, probe, A = bench.make_data("netflix-ccdpp")
for K in (1, 3):
    t0 = time.perf_counter()
    m, rep = P.ccdpp_train(P.CcdConfig(k=40, lam=0.05, outer_iters=K, inner_iters=15, seed=1), A, probe)
    wall = time.perf_counter() - t0
    print(f"K={K}: wall {wall:.3f} s, setup {rep.setup_seconds:.3f}, train {rep.train_seconds:.3f}, lib wall {rep.wall_seconds:.3f}")
