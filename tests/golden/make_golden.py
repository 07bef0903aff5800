"""Generates the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs the parmf headers compiled in place (oracle/_ref/libparmf_ref.so, built by oracle/Makefile
from /root/reference/proj/include) on the seeded synthetic inputs of BASELINE.json configs[0] and on
the reference's own small test fixtures, and freezes per-iteration objective / probe RMSE / train
RMSE plus factor checksums.  The inputs are regenerated bit-identically from seeds by the
reference's own testutil generators, so only outputs are stored.

    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.pyoracle import Reference  # noqa: E402


def checksums(x):
    x = np.asarray(x, np.float64)
    return {"sum": float(x.sum()), "sumsq": float((x * x).sum()), "first": [float(v) for v in x.ravel()[:8]]}


def rows_to_json(rows):
    return [{"iteration": int(r["iteration"]), "objective": float(r["objective"]), "rmse": float(r["rmse"]),
             "train_rmse": float(r["train_rmse"])} for r in rows]


def main():
    R = Reference()
    out = {}
    # BASELINE.json configs[0]: ML-100K shape, 10% probe, k=10, lambda=0.05, 5 outer x 15 inner
    data = R.synth_ratings(943, 1682, 3, 100000, 777)
    train, probe = R.carve_probe(data, 10000, 5)
    for real in ("_f32", "_f64"):
        M = R.matrix(train, 943, 1682, real)
        W, H, rows, rr, rc = M.ccdpp_stage_loop(10, 0.05, 5, 15, 1, probe, workers=4)
        out["ccdpp_ml100k_k10" + real] = {
            "config": {"m": 943, "n": 1682, "nnz_total": 100000, "probe": 10000, "gen_seed": 777, "probe_seed": 5,
                       "k": 10, "lambda": 0.05, "outer": 5, "inner": 15, "seed": 1},
            "rows": rows_to_json(rows), "W": checksums(W), "H": checksums(H),
            "residual_row": checksums(rr)}
        W, H, rows = M.als_epochs(10, 0.05, 5, 1, probe, workers=4)
        out["als_ml100k_k10" + real] = {
            "config": {"m": 943, "n": 1682, "k": 10, "lambda": 0.05, "outer": 5, "seed": 1},
            "rows": rows_to_json(rows), "W": checksums(W), "H": checksums(H)}
    # tests/ccd_test.cpp:332-345 / acceptance C6: planted rank-2 20x15, k=2, lambda=1e-6, 15 x 15
    planted = R.planted_full(20, 15, 2, 0.01, 42)
    M = R.matrix(planted, 20, 15, "_f32")
    W, H, rows = M.ccdpp_train(2, 1e-6, 15, 15, 3, None, workers=2)
    out["ccdpp_planted_f32"] = {"rows": rows_to_json(rows)}
    W, H, rows = M.als_train(2, 1e-6, 15, 3, None, workers=2)
    out["als_planted_f32"] = {"rows": rows_to_json(rows)}
    # small exact fixture: random_triplets(40, 30, 350, 71) (tests/ccd_test.cpp:369-397), k=3
    small = R.random_triplets(40, 30, 350, 71)
    M = R.matrix(small, 40, 30, "_f32")
    W, H, rows, rr, rc = M.ccdpp_stage_loop(3, 0.1, 4, 3, 9, None, workers=2)
    out["ccdpp_small_k3_f32"] = {"rows": rows_to_json(rows), "W": W.ravel().tolist(), "H": H.ravel().tolist(),
                                 "r_row": rr.tolist(), "r_col": rc.tolist()}
    W, H, rows = M.als_epochs(3, 0.1, 4, 9, None, workers=2)
    out["als_small_k3_f32"] = {"rows": rows_to_json(rows), "W": W.ravel().tolist(), "H": H.ravel().tolist()}
    with open(os.path.join(HERE, "reference_trajectories.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", os.path.join(HERE, "reference_trajectories.json"))


if __name__ == "__main__":
    main()
