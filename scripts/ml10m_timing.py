import sys, os
sys.path.insert(0, os.getcwd())
import bench, paper_1511_02433_b200 as P
train, probe, A = bench.make_data("ml10m-als")
ctx = P.Context(A); ctx.set_probe(probe)
ctx.als_begin(P.AlsConfig(k=10, lam=0.05, outer_iters=1, seed=1)); ctx.als_iterate(1)
a = ctx.als_iterate(3)
ctx.ccd_begin(P.CcdConfig(k=10, lam=0.05, outer_iters=1, inner_iters=1, seed=1)); ctx.ccd_iterate(1)
c = ctx.ccd_iterate(3)
print(os.environ.get("PMF_ALS_CHUNK", "auto"), "ml10m ALS ms", [round(1e3*x, 3) for x in a], "CCD ms", [round(1e3*x, 3) for x in c])
