import sys, os, time
sys.path.insert(0, os.getcwd())
import bench, paper_1511_02433_b200 as P
import numpy as np
train, probe = bench.make_data("netflix-ccdpp")
A = P.RatingsMatrix.from_triplets(train, *bench.CONFIGS["netflix-ccdpp"][:2])
for rep in range(2):
    t0 = time.perf_counter(); t = P._as_triplets(train); t1 = time.perf_counter()
    Ag = P.RatingsMatrix.from_triplets(train, 480189, 17770, device=True); t2 = time.perf_counter()
    Ah = P.RatingsMatrix.from_triplets(train, 480189, 17770); t3 = time.perf_counter()
    print("as_triplets %.3f gpu %.3f host %.3f" % (t1 - t0, t2 - t1, t3 - t2), file=sys.stderr)
