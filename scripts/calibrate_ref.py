"""Reference float-vs-double calibration at a BASELINE shape (CPU only; test infrastructure).

Runs the reference (parmf compiled from its unmodified headers, oracle/_ref) in float AND double on the
bench corpus of CONFIG (bench.make_data -> datagen), through its stage API loop (the same trajectory as
ccdpp_train / als_train, tests/acceptance_test.cpp:150-171 pattern), and records per outer iteration
the relative Frobenius distance of the float and double factors and the relative differences of the
metrics.  That distance is what FP32 reduction order alone does to the factors at that shape; the
parity tests (tests/test_gpu_configs.py) allow the GPU factors twice it where it exceeds 1e-3.

    python scripts/calibrate_ref.py CONFIG [OUTER] > profiles/r02_calib_CONFIG.json
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from oracle.pyoracle import Reference  # noqa: E402


def frob(x, y):
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    return float(np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300))


def main():
    cfg = sys.argv[1]
    outer = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    m, n, ntr, npr, k, lam, inner, solver, skew = bench.CONFIGS[cfg]
    cores = os.cpu_count() or 1
    train, probe = bench.make_data(cfg)
    out = {"config": cfg, "m": m, "n": n, "nnz": int(len(train)), "probe": int(len(probe)), "k": k, "lambda": lam,
           "inner_iters": inner if solver == "ccdpp" else None, "outer_iters": outer, "workers": cores,
           "what": "reference float vs reference double (oracle/_ref), same bytes, stage-API loop"}
    R = Reference()
    hist, rows_by = {}, {}
    for real in ("_f32", "_f64"):
        t0 = time.perf_counter()
        M = R.matrix(train, m, n, real)
        if solver == "ccdpp":
            _, _, rows, _, _, Wh, Hh = M.ccdpp_stage_loop(k, lam, outer, inner, 1, probe, workers=cores, history=True)
        else:
            _, _, rows, Wh, Hh = M.als_epochs(k, lam, outer, 1, probe, workers=cores, history=True)
        rows_by[real] = [{"objective": float(r["objective"]), "rmse": float(r["rmse"]),
                          "train_rmse": float(r["train_rmse"]), "seconds": float(r["seconds"])} for r in rows]
        out["ref" + real] = {"rows": rows_by[real], "wall_s": round(time.perf_counter() - t0, 1)}
        hist[real] = (Wh, Hh)
        del M
        print(f"[calib] {cfg} reference{real} done in {time.perf_counter() - t0:.0f}s", file=sys.stderr, flush=True)
    for key in ("objective", "rmse", "train_rmse"):
        out[f"rel_{key}_f32_vs_f64"] = [abs(a[key] - b[key]) / abs(b[key])
                                        for a, b in zip(rows_by["_f32"], rows_by["_f64"])]
    (Wf, Hf), (Wd, Hd) = hist["_f32"], hist["_f64"]
    out["factors_per_iteration"] = [{"iteration": it + 1, "W_f32_vs_f64": frob(Wf[it], Wd[it]),
                                     "H_f32_vs_f64": frob(Hf[it], Hd[it])} for it in range(outer)]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
