"""Netflix-shape parity against the reference itself: per-iteration objective, probe RMSE and train RMSE
of the B200 path and of the reference (parmf compiled from its headers, oracle/_ref, all host threads) on
the same synthetic Netflix-shape data (bench.make_data: 480,189 x 17,770, 99M ratings), CCD++ (k = 40,
T = 15), ALS and item/user-wise CCD (k = 40), plus the relative Frobenius distance of the factors.  Writes
gpurun_out/<config>_trajectory.json.  OUTER_CCD / OUTER_ALS / OUTER_CCDW set the iteration counts (3 / 2 / 2), ALGOS the algorithms;
CONFIG=yahoo-ccdpp runs the Yahoo-Music shape (k = 100, CCD++ only: the ALS kernels take k <= 64)."""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1511_02433_b200 as P  # noqa: E402
from oracle.pyoracle import Reference, RefMatrix  # noqa: E402


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def frob(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(np.asarray(b, np.float64)))


def main():
    oc = int(os.environ.get("OUTER_CCD", "3"))
    oa = int(os.environ.get("OUTER_ALS", "2"))
    cfg = os.environ.get("CONFIG", "netflix-ccdpp")
    m, n, _, _, k, *_ = bench.CONFIGS[cfg]
    train, probe = bench.make_data(cfg)
    A = P.RatingsMatrix.from_triplets(train, *bench.CONFIGS[cfg][:2])
    ref = Reference()
    workers = os.cpu_count() or 1
    RA = RefMatrix(ref, train, m, n, "_f32")
    out = {"workers": workers, "config": f"{cfg} synthetic, k={k}, lambda=0.05, seed 1"}
    ow = int(os.environ.get("OUTER_CCDW", "2"))
    algos = os.environ.get("ALGOS", "ccdpp,als,ccd").split(",")
    ref_cache = {}
    for algo in [a for a in algos if a == "ccdpp" or k <= 64]:
        t0 = time.time()
        if algo == "ccdpp":
            model, rep = P.ccdpp_train(P.CcdConfig(k=k, lam=0.05, outer_iters=oc, inner_iters=15, seed=1), A, probe)
        elif algo == "als":
            model, rep = P.als_train(P.AlsConfig(k=k, lam=0.05, outer_iters=oa, seed=1), A, probe)
        else:  # item/user-wise CCD (ccd.hpp:310-344), residual form; ccd_gram: PMF_CCD_GRAM=1
            if algo == "ccd_gram":
                os.environ["PMF_CCD_GRAM"] = "1"
            model, rep = P.ccd_train(P.CcdConfig(k=k, lam=0.05, outer_iters=ow, inner_iters=1, seed=1), A, probe)
            os.environ.pop("PMF_CCD_GRAM", None)
        t_gpu = time.time() - t0
        t0 = time.time()
        # the stage-API loop / epoch loop: bitwise the reference's ccdpp_train / als_train trajectory
        # (tests/test_oracle.py) and their rows also carry the train RMSE
        if algo == "ccdpp":
            W, H, rows, _, _ = RA.ccdpp_stage_loop(k, 0.05, oc, 15, 1, probe, workers)
        elif algo == "als":
            W, H, rows = RA.als_epochs(k, 0.05, oa, 1, probe, workers)
        elif "ccd" not in ref_cache:  # (ccd_train's rows have no train RMSE: the final one is compared)
            W, H, rows = ref_cache["ccd"] = RA.ccd_train(k, 0.05, ow, 1, probe)
        else:
            W, H, rows = ref_cache["ccd"]
        t_ref = time.time() - t0
        its = []
        for r, g in zip(rep.rows, rows):
            its.append({"iteration": r.iteration, "objective": [r.objective, float(g["objective"])],
                        "rel_objective": rel(r.objective, float(g["objective"])),
                        "rel_probe_rmse": rel(r.rmse, float(g["rmse"])),
                        "rel_train_rmse": rel(r.train_rmse, float(g["train_rmse"]))})
            print(f"{algo} iter {r.iteration}: objective {r.objective:.8g} vs {float(g['objective']):.8g} "
                  f"(rel {its[-1]['rel_objective']:.2e}), probe rmse rel {its[-1]['rel_probe_rmse']:.2e}, "
                  f"train rmse rel {its[-1]['rel_train_rmse']:.2e}", flush=True)
        # final train RMSE of both models, evaluated by the same (reference-pinned) rmse kernel
        tr_gpu = P.rmse(model, train)
        tr_ref = P.rmse(P.FactorModel(np.ascontiguousarray(W, np.float32), np.ascontiguousarray(H, np.float32)), train)
        out[algo] = {"iterations": its, "frob_rel_W": frob(model.w, W), "frob_rel_H": frob(model.h, H),
                     "final_train_rmse": [tr_gpu, tr_ref], "rel_final_train_rmse": rel(tr_gpu, tr_ref),
                     "gpu_wall_s": round(t_gpu, 2), "reference_wall_s": round(t_ref, 2)}
        print(f"{algo}: factors rel Frobenius W {out[algo]['frob_rel_W']:.2e} H {out[algo]['frob_rel_H']:.2e}; "
              f"wall GPU {t_gpu:.1f} s (incl. setup) vs reference {t_ref:.1f} s", flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/{cfg.split('-')[0]}_trajectory.json", "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
