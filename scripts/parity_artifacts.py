"""Large-shape parity artefacts against the reference itself (run on the GPU box; never a bench number).

For each config: the reference (parmf compiled from its headers, oracle/_ref) in float AND double, on
all host cores, through its stage API loop (tests/acceptance_test.cpp:150-171 pattern -- bitwise the
same trajectory as ccdpp_train / als_train, plus per-iteration train RMSE), and the B200 library on
the same bytes (datagen corpus of bench.py).  Records per-iteration objective / probe RMSE / train
RMSE of all three runs, their relative differences, and the relative Frobenius distances of the
final factors: GPU vs float, GPU vs double, and float vs double -- the last one is the calibration of
what FP32 reduction order alone does to the factors at that shape.

    python scripts/parity_artifacts.py CONFIG [OUTER] [--f32-only] > gpurun_out/parity_CONFIG.json

--f32-only skips the reference's double run (its float-vs-double distance is then taken from the
committed calibration profiles/r02_calib_CONFIG.json, scripts/calibrate_ref.py).
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1511_02433_b200 as P  # noqa: E402
from oracle.pyoracle import Reference  # noqa: E402


def frob(x, y):
    x = np.asarray(x, np.float64); y = np.asarray(y, np.float64)
    return float(np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300))


def rows_of(rows):
    return [{"objective": float(r["objective"]), "rmse": float(r["rmse"]), "train_rmse": float(r["train_rmse"]),
             "seconds": float(r["seconds"])} for r in rows]


def main():
    cfg = sys.argv[1]
    m, n, ntr, npr, k, lam, inner, solver, skew = bench.CONFIGS[cfg]
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    f32_only = "--f32-only" in sys.argv
    outer = int(args[1]) if len(args) > 1 else 2
    cores = os.cpu_count() or 1
    train, probe = bench.make_data(cfg)
    out = {"config": cfg, "m": m, "n": n, "nnz": int(len(train)), "probe": int(len(probe)), "k": k, "lambda": lam,
           "inner_iters": inner if solver == "ccdpp" else None, "outer_iters": outer, "workers": cores}
    # B200: the resident context, the model read back after every outer iteration
    A = P.RatingsMatrix.from_triplets(train, m, n)
    t0 = time.perf_counter()
    ctx = P.Context(A)
    ctx.set_probe(probe)
    if solver == "ccdpp":
        ctx.ccdpp_begin(P.CcdConfig(k=k, lam=lam, outer_iters=outer, inner_iters=inner, seed=1))
    else:
        ctx.als_begin(P.AlsConfig(k=k, lam=lam, outer_iters=outer, seed=1))
    grows, gmodels = [], []
    for it in range(outer):
        sec = (ctx.ccdpp_iterate if solver == "ccdpp" else ctx.als_iterate)(1)[0]
        o, r, t = ctx.metrics()
        grows.append({"objective": o, "rmse": r, "train_rmse": t, "seconds": float(sec)})
        mm = ctx.model()
        gmodels.append((mm.w.copy(), mm.h.copy()))
    ctx.close()
    out["gpu"] = {"rows": grows, "wall_s": time.perf_counter() - t0}
    del A
    R = Reference()
    hist = {}
    for real in (("_f32",) if f32_only else ("_f32", "_f64")):
        t0 = time.perf_counter()
        M = R.matrix(train, m, n, real)
        if solver == "ccdpp":
            W, H, rows, _, _, Wh, Hh = M.ccdpp_stage_loop(k, lam, outer, inner, 1, probe, workers=cores,
                                                          history=True)
        else:
            W, H, rows, Wh, Hh = M.als_epochs(k, lam, outer, 1, probe, workers=cores, history=True)
        out["ref" + real] = {"rows": rows_of(rows), "wall_s": time.perf_counter() - t0}
        hist[real] = (Wh, Hh)
        del M
        print(f"[parity] {cfg} reference{real} done in {time.perf_counter() - t0:.0f}s", file=sys.stderr, flush=True)
    if f32_only:
        cal = json.load(open(os.path.join(ROOT, "profiles", f"r02_calib_{cfg}.json")))
        out["ref_f64"] = cal["ref_f64"]
        out["ref_f64"]["source"] = f"profiles/r02_calib_{cfg}.json (same bytes, reference double run)"
    for key in ("objective", "rmse", "train_rmse"):
        for a, b in (("gpu", "ref_f32"), ("gpu", "ref_f64"), ("ref_f32", "ref_f64")):
            out[f"rel_{key}_{a}_vs_{b}"] = [abs(g[key] - f[key]) / abs(f[key]) for g, f in
                                            zip(out[a]["rows"], out[b]["rows"])]
    Wf, Hf = hist["_f32"]
    if f32_only:
        out["factors_per_iteration"] = [
            dict({"iteration": it + 1, "W_gpu_vs_f32": frob(gmodels[it][0], Wf[it]),
                  "H_gpu_vs_f32": frob(gmodels[it][1], Hf[it])},
                 **{k: v for k, v in cal["factors_per_iteration"][it].items() if k.endswith("f32_vs_f64")})
            for it in range(outer)]
    else:
        Wd, Hd = hist["_f64"]
        out["factors_per_iteration"] = [
            {"iteration": it + 1,
             "W_gpu_vs_f32": frob(gmodels[it][0], Wf[it]), "H_gpu_vs_f32": frob(gmodels[it][1], Hf[it]),
             "W_gpu_vs_f64": frob(gmodels[it][0], Wd[it]), "H_gpu_vs_f64": frob(gmodels[it][1], Hd[it]),
             "W_f32_vs_f64": frob(Wf[it], Wd[it]), "H_f32_vs_f64": frob(Hf[it], Hd[it])} for it in range(outer)]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
