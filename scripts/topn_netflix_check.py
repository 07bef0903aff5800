"""top_n at Netflix shape against the reference itself: a model from 2 CCD++ iterations on the B200,
then the top-10 unrated items of 200 sampled users from pmf_top_n and from the reference's top_n
(model.hpp:172-209, rated items excluded).  Items and scores must be bitwise equal.  Writes
gpurun_out/topn_netflix_check.json."""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1511_02433_b200 as P  # noqa: E402
from oracle.pyoracle import Reference  # noqa: E402


def main():
    train, probe = bench.make_data("netflix-ccdpp")
    A = P.RatingsMatrix.from_triplets(train, *bench.CONFIGS["netflix-ccdpp"][:2])
    model, _ = P.ccdpp_train(P.CcdConfig(k=40, lam=0.05, outer_iters=2, inner_iters=15, seed=1), A, probe)
    rng = np.random.default_rng(5)
    users = np.sort(rng.choice(A.m, 200, replace=False)).astype(np.int32)
    items, scores, counts = P.top_n_batch(model, users, 10, a=A)
    ref = Reference()
    t0 = time.time()
    equal = 0
    for x, i in enumerate(users):
        rated = A.col_of[A.row_start[i]:A.row_start[i + 1]]
        r = ref.top_n(model.w, model.h, int(i), 10, rated)
        ri = np.array([t[0] for t in r], np.int32)
        rs = np.array([t[1] for t in r], np.float32)
        ok = counts[x] == len(r) and np.array_equal(items[x, :len(r)], ri) and \
            np.array_equal(scores[x, :len(r)].view(np.uint32), rs.view(np.uint32))
        equal += bool(ok)
    t_ref = time.time() - t0
    out = {"users": len(users), "bitwise_equal": equal, "reference_s_per_user": t_ref / len(users)}
    print(json.dumps(out))
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/topn_netflix_check.json", "w") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    main()
