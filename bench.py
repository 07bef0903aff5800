"""bench.py -- seconds per outer iteration of CCD++ at synthetic Netflix shape, k=40 (BASELINE configs[2]),
with the other BASELINE configs as extra keys of the same line.

BASELINE.json metric: "sec/outer-iter (CCD++, ALS) at Netflix shape k=40, %HBM peak; RMSE vs CPU ref".
A "step" is one outer iteration (ccd.hpp:370-398): for t in 0..k-1 the rank-one step (fused promote,
15 x (u-sweep, v-sweep), deferred writeback).  Workload: CCD++ k=40, lambda=0.05, T=15 on the
480,189 x 17,770 synthetic Netflix shape, 99,072,112 training ratings + 1,408,395 probe (datagen/).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config NAME] [--quick]

* ``--impl ours`` (default): the B200 library.  ``value`` = device time per outer iteration (CUDA events
  around the captured graph, max over ranks); ``e2e`` = the public API with host buffers (N=1: the
  whole-call pmf_ccdpp_train, copies / layout build / per-iteration metrics / model download inside;
  N>1: every rank's resident NCCL context built from host buffers); ``roofline`` = the v-sweep's
  algorithmic bytes per launch / its CUDA-event time; ``cpu_baseline`` = the reference
  (parmf headers compiled in oracle/_ref) on the host cores, one measured steady-state outer
  iteration.  At N=1 the other BASELINE configs ride along: ``ml100k`` (configs[0], GPU vs the
  reference on 1 and all host cores), ``ml10m_als`` (configs[1]), ``als`` (configs[3]), ``yahoo``
  (configs[4]), plus ``netflix_skew`` (power-law users), ``ccd`` (item/user-wise CCD) and ``ingest``.
* ``--impl reference``: the reference's own ccdpp_train<float> (ccd.hpp:349) through oracle/_ref on
  all host cores, W warm-up + K timed whole outer iterations in one call, each iteration's seconds from
  its own TrainReport (solver stages, metrics excluded).  It never loads the product library.

Multi-GPU: ``--gpus N`` without a torchrun environment relaunches itself under torch.distributed.run
(one process per GPU, NCCL); each rank owns a CSR row block and a CSC column block (strong scaling of
the fixed problem) and u / v are all-gathered over NCCL inside the captured graph.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (m, n, n_train, n_probe, k, lambda, inner, solver, user_skew)
    "netflix-ccdpp": (480189, 17770, 99072112, 1408395, 40, 0.05, 15, "ccdpp", 0.0),
    "netflix-als": (480189, 17770, 99072112, 1408395, 40, 0.05, 1, "als", 0.0),
    "yahoo-ccdpp": (1000990, 624961, 252800275, 4003960, 100, 0.05, 15, "ccdpp", 0.0),
    "ml10m-als": (69878, 10677, 9900000, 100000, 10, 0.05, 1, "als", 0.0),
    "ml100k-ccdpp": (943, 1682, 90000, 10000, 10, 0.05, 15, "ccdpp", 0.0),
    "netflix-skew-ccdpp": (480189, 17770, 99072112, 1408395, 40, 0.05, 15, "ccdpp", 0.5),
}
GEN_SEED, MODEL_SEED = 777, 1
DATA_NOTE = ("synthetic, datagen/synth.cpp (tests/testutil.hpp:91-132 recipe -- planted rank 3 + biases + "
             "noise, 1..5 stars, Zipf(0.8) items -- on per-user splitmix64 streams, users ~N(mean, mean) "
             "counts{skew}, probe carved per user), seed 777; model seed 1; both arms read the same bytes")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.proc, self.lines = device, None, []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def make_data(cfg_name):
    """(train, probe) Triplet<float> arrays of a config -- datagen only (no product library)."""
    import datagen
    m, n, ntr, npr, *_, skew = CONFIGS[cfg_name]
    t0 = time.perf_counter()
    train, probe = datagen.synth_ratings(m, n, 3, ntr, npr, GEN_SEED, user_skew=skew)
    log(f"[bench] data {cfg_name}: {m}x{n} train={len(train)} probe={len(probe)} in {time.perf_counter() - t0:.1f}s")
    return train, probe


def ccd_bytes(N, m, n, k, T):
    """SURVEY.md 8(d) algorithmic bytes (FP32 values, int32 indices, int64 offsets)."""
    u = 8 * N + 12 * m + 4 * n
    v = 8 * N + 12 * n + 4 * m
    per_iter = k * (T * (16 * N + 16 * (m + n)) + 8 * N)
    return u, v, per_iter


def als_flops(N, m, n, k):
    """2 [2 N (k(k+1)/2 + k) + (m + n)(k^3/6 + k^2)] per ALS iteration."""
    return 2.0 * (2.0 * N * (k * (k + 1) / 2 + k) + (m + n) * (k ** 3 / 6 + k * k))


# ALS is issue / latency-bound (ncu: 50-56 % issue slots busy, profiles/r02_ncu_als_*): its roofline object
# reports the useful FP32-equivalent flops against both compute ceilings it could be held to
# -- the FP32 SIMT peak (148 SMs x 128 lanes x 2 flops at the 1,965 MHz max clock) and the dense TF32
# tensor peak measured with tcgen05 (scripts/micro/umma_rate.cu: 2,046 MAC / cycle / SM).
FP32_SIMT_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12
TF32_TENSOR_PEAK_TFLOPS = 148 * 2046 * 2 * 1.965e9 / 1e12


def als_roofline(fl, seconds):
    ach = fl / seconds / 1e12
    return {"bound": "issue (instruction / latency)", "achieved": round(ach, 2), "unit": "TFLOP/s",
            "peak": round(FP32_SIMT_PEAK_TFLOPS, 1), "frac": round(ach / FP32_SIMT_PEAK_TFLOPS, 4),
            "peak_source": "FP32 SIMT peak (148 x 128 x 2 x 1.965 GHz); the dense TF32 tensor peak measured with "
                           "tcgen05 is also given",
            "tf32_tensor_peak": round(TF32_TENSOR_PEAK_TFLOPS, 1),
            "frac_of_tf32_tensor": round(ach / TF32_TENSOR_PEAK_TFLOPS, 4),
            "flops_per_iter": fl, "note": "useful FP32-equivalent flops: 2 [2N(k(k+1)/2 + k) + (m + n)(k^3/6 + k^2)]"}


def ccd_epoch_roofline(N, k, seconds, hbm):
    """item/user-wise CCD: SURVEY 8(d) algorithmic bytes 8N per coordinate t per side."""
    b = 2 * k * 8 * N
    return {"bound": "hbm", "achieved": round(b / seconds / 1e9, 1), "unit": "GB/s", "peak": hbm,
            "frac": round(b / seconds / 1e9 / hbm, 4), "algorithmic_bytes_per_epoch": b,
            "note": "latency-bound: a coordinate-by-coordinate chain per row / column; rows and columns up to 8K "
                    "entries keep their residual in registers and gather the opposing factor 8 / 4 coordinates "
                    "at a time, longer columns stream (profiles/r02_ncu_ccdw.txt)"}


def barrier(dist):
    if dist:
        import torch.distributed as td
        td.barrier()


def max_over_ranks(dist, x):
    if not dist:
        return float(x)
    import torch
    import torch.distributed as td
    t = torch.tensor([float(x)], dtype=torch.float64)
    td.all_reduce(t, op=td.ReduceOp.MAX)
    return float(t.item())


# ---- the reference (oracle/_ref: parmf compiled from its unmodified headers) -------------------------

def ref_matrix(train, m, n):
    from oracle.pyoracle import Reference
    t0 = time.perf_counter()
    M = Reference().matrix(train, m, n, "_f32")
    log(f"[bench] reference RatingsMatrix::from_triplets {time.perf_counter() - t0:.1f}s")
    return M


def ref_train_rows(M, solver, k, lam, inner, outer, workers, probe):
    """The reference's own ccdpp_train / als_train<float> (ccd.hpp:349, als.hpp:188): per-iteration
    TrainReport rows (seconds = solver stages, metrics excluded)."""
    if solver == "ccdpp":
        _, _, rows = M.ccdpp_train(k, lam, outer, inner, MODEL_SEED, probe, workers=workers)
    else:
        _, _, rows = M.als_train(k, lam, outer, MODEL_SEED, probe, workers=workers)
    return rows


def reference_arm(args, world, rank):
    if rank != 0:
        return
    m, n, ntr, npr, k, lam, inner, solver, skew = CONFIGS[args.config]
    cores = os.cpu_count() or 1
    train, probe = make_data(args.config)
    M = ref_matrix(train, m, n)
    W, K = max(0, args.warmup), max(1, args.steps)
    t0 = time.perf_counter()
    rows = ref_train_rows(M, solver, k, lam, inner, W + K, cores, probe)
    wall = time.perf_counter() - t0
    secs = [float(x) for x in rows["seconds"][W:]]
    v = float(np.mean(secs))
    sample = (f"{solver}_train<float> (parmf, oracle/_ref) with workers={cores}: {W} warm-up + {K} timed whole "
              f"outer iterations in one call on the full matrix, seconds from its TrainReport rows")
    line = {"impl": "reference", "metric": f"sec/outer-iter {solver} (lower is better)", "value": v, "unit": "s/outer-iter",
            "n_gpus": 0, "steps": K, "warmup": W, "ms_per_step": v * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_of(args, world),
            "cpu_baseline": {"value": v, "unit": "s/outer-iter", "cores": cores, "kind": "reference", "sample": sample},
            "e2e": {"value": v, "unit": "s/outer-iter", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "per_step_s": secs, "call_wall_s": round(wall, 2),
            "quality": {"objective": float(rows["objective"][-1]), "probe_rmse": float(rows["rmse"][-1])}}
    print(json.dumps(line), flush=True)


def workload_of(args, world):
    m, n, ntr, npr, k, lam, inner, solver, skew = CONFIGS[args.config]
    return {"workload": f"{solver}-{args.config.split('-')[0]}-k{k}", "m": m, "n": n, "nnz_train": ntr, "probe": npr,
            "k": k, "lambda": lam, "inner_iters": inner if solver == "ccdpp" else None, "solver": solver,
            "data": DATA_NOTE.format(skew=f", power law {skew} on users" if skew else ""),
            "l2": "inputs larger than L2 (CSR+CSC residual >= 1.6 GB >> 126 MB L2), no flush needed",
            "parallelism": f"row/col blocks x{world}"}


# ---- the B200 library ----------------------------------------------------------------------------

def ccdpp_roofline(ctx, iterate, N, m, n, k, inner, value, hbm, cfg_name):
    """Dominant-kernel roofline: one uncaptured iteration with CUDA events around every sweep."""
    ub, vb, per_iter = ccd_bytes(N, m, n, k, inner)
    ctx.set_profiling(True)
    iterate(1)
    st = ctx.kernel_stats()
    ctx.set_profiling(False)
    # per launch: the T sweeps of a step, the first one with the promote RMW (+4N)
    u_bytes = st["usweep_launches"] * ub + k * 4 * N
    v_bytes = st["vsweep_launches"] * vb + k * 4 * N
    u_ach = u_bytes / (st["usweep_ms"] * 1e-3) / 1e9
    v_ach = v_bytes / (st["vsweep_ms"] * 1e-3) / 1e9
    dom = "v-sweep" if st["vsweep_ms"] >= st["usweep_ms"] else "u-sweep"
    ach = v_ach if dom == "v-sweep" else u_ach
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = tr.get(cfg_name, {}).get(dom)
    except Exception:
        pass
    return {"bound": "hbm", "kernel": dom, "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
            "frac": round(ach / hbm, 4), "traffic": traffic,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)",
            "whole_iteration": {"achieved": round(per_iter / value / 1e9, 1),
                                "frac": round(per_iter / value / 1e9 / hbm, 4),
                                "algorithmic_bytes_per_iter": per_iter},
            "usweep": {"ms": st["usweep_ms"], "launches": st["usweep_launches"], "gbs": round(u_ach, 1)},
            "vsweep": {"ms": st["vsweep_ms"], "launches": st["vsweep_launches"], "gbs": round(v_ach, 1)}}


def run_ours(args, rank, world, dist):
    import paper_1511_02433_b200 as P
    m, n, ntr, npr, k, lam, inner, solver, skew = CONFIGS[args.config]
    device = int(os.environ.get("LOCAL_RANK", "0"))
    train, probe = make_data(args.config)
    A = P.RatingsMatrix.from_triplets(train, m, n)
    N = A.nnz()
    nccl_id = None
    if world > 1:
        import torch.distributed as td
        obj = [P.nccl_unique_id() if rank == 0 else None]
        td.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    t0 = time.perf_counter()
    ctx = P.Context(A, device=device, rank=rank, world=world, nccl_id=nccl_id)
    log(f"[bench] context (layouts + upload) {time.perf_counter() - t0:.1f}s")
    for side, li in ctx.layout_info().items():
        log(f"[bench] layout {side}: " + " ".join(f"{a}={b}" for a, b in li.items()))
    ctx.set_probe(probe)
    hbm = peaks().get("hbm_gbs", 6544.7)
    if solver == "ccdpp":
        ctx.ccdpp_begin(P.CcdConfig(k=k, lam=lam, outer_iters=max(1, args.steps), inner_iters=inner, seed=MODEL_SEED))
        iterate = ctx.ccdpp_iterate
    else:
        ctx.als_begin(P.AlsConfig(k=k, lam=lam, outer_iters=max(1, args.steps), seed=MODEL_SEED))
        iterate = ctx.als_iterate
    iterate(args.warmup)
    barrier(dist)
    with ClockSampler(device) as clk:
        secs = iterate(args.steps)
    times = [max_over_ranks(dist, s) for s in secs]
    launches = ctx.launch_count()
    obj, rmse, trmse = ctx.metrics()
    value = float(np.mean(times))
    res = dict(value=value, times=times, launches=launches, objective=obj, rmse=rmse, train_rmse=trmse,
               clocks=clk.summary(), roofline=None)
    if solver == "ccdpp":
        res["roofline"] = ccdpp_roofline(ctx, iterate, N, m, n, k, inner, value, hbm, args.config)
    else:
        res["roofline"] = als_roofline(als_flops(N, m, n, k), value)
    res.update(ctx=ctx, nccl_id=nccl_id, A=A, probe=probe, train=train)
    return res


def e2e_whole_call(args, A, probe):
    """N=1: the public whole-call API (pmf_ccdpp_train / pmf_als_train) on HOST buffers: upload, device
    layout build, K outer iterations with per-iteration metrics, model download -- host clock."""
    import paper_1511_02433_b200 as P
    m, n, ntr, npr, k, lam, inner, solver, skew = CONFIGS[args.config]
    K = max(1, args.steps)

    def call(outer):
        if solver == "ccdpp":
            return P.ccdpp_train(P.CcdConfig(k=k, lam=lam, outer_iters=outer, inner_iters=inner, seed=MODEL_SEED),
                                 A, probe)
        return P.als_train(P.AlsConfig(k=k, lam=lam, outer_iters=outer, seed=MODEL_SEED), A, probe)

    # the first call in the process pays one-time costs (module loads, pinning the host layout blocks,
    # the device block cache): measured and reported, then the timed call
    t0 = time.perf_counter()
    call(1)
    cold = time.perf_counter() - t0
    t0 = time.perf_counter()
    _, rep = call(K)
    wall = time.perf_counter() - t0
    return {"value": wall / K, "unit": "s/outer-iter", "h2d_bytes_per_step": int(rep.h2d_bytes / K),
            "d2h_bytes_per_step": int(rep.d2h_bytes / K), "setup_seconds": round(rep.setup_seconds, 3),
            "final_rmse": rep.final_rmse, "api": "pmf_ccdpp_train (whole call, host buffers)",
            "cold_first_call_1iter_s": round(cold, 3),
            "note": "one untimed 1-iteration call first (cold_first_call_1iter_s): the process-wide device "
                    "block cache and page-locked layout pool it warms serve the timed call"}


def e2e_dist(args, rank, world, dist, A, probe, nccl_id):
    """N>1: every rank builds its resident NCCL context from host buffers (layout build + upload + NCCL
    init), runs K iterations with per-iteration metrics; rank 0 downloads the model.  Host clock,
    max over ranks."""
    import paper_1511_02433_b200 as P
    m, n, ntr, npr, k, lam, inner, solver, skew = CONFIGS[args.config]
    K = max(1, args.steps)
    device = int(os.environ.get("LOCAL_RANK", "0"))
    import torch.distributed as td
    obj = [P.nccl_unique_id() if rank == 0 else None]
    td.broadcast_object_list(obj, src=0)
    barrier(dist)
    t0 = time.perf_counter()
    ctx = P.Context(A, device=device, rank=rank, world=world, nccl_id=obj[0])
    ctx.set_probe(probe)
    if solver == "ccdpp":
        ctx.ccdpp_begin(P.CcdConfig(k=k, lam=lam, outer_iters=K, inner_iters=inner, seed=MODEL_SEED))
    else:
        ctx.als_begin(P.AlsConfig(k=k, lam=lam, outer_iters=K, seed=MODEL_SEED))
    for _ in range(K):
        (ctx.ccdpp_iterate if solver == "ccdpp" else ctx.als_iterate)(1)
        ctx.metrics()
    if rank == 0:
        ctx.model()
    ctx.close()
    wall = max_over_ranks(dist, time.perf_counter() - t0)
    return {"value": wall / K, "unit": "s/outer-iter", "api": "pmf_ctx_create_dist per rank (host buffers)",
            "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
            "note": "layout build + upload + NCCL init + K iterations with metrics + model download"}


def side_gpu(P, cfg_name, warm=1, steps=3, profile=False):
    """Device s/outer-iter of another config on this GPU (+ whole-iteration roofline for CCD++)."""
    m, n, ntr, npr, k, lam, inner, solver, skew = CONFIGS[cfg_name]
    train, probe = make_data(cfg_name)
    A = P.RatingsMatrix.from_triplets(train, m, n)
    ctx = P.Context(A)
    ctx.set_probe(probe)
    if solver == "ccdpp":
        ctx.ccdpp_begin(P.CcdConfig(k=k, lam=lam, outer_iters=steps, inner_iters=inner, seed=MODEL_SEED))
        it = ctx.ccdpp_iterate
    else:
        ctx.als_begin(P.AlsConfig(k=k, lam=lam, outer_iters=steps, seed=MODEL_SEED))
        it = ctx.als_iterate
    it(warm)
    ts = list(it(steps))
    o, r, t = ctx.metrics()
    v = float(np.mean(ts))
    out = {"config": cfg_name, "value": v, "unit": "s/outer-iter", "per_step_s": ts, "objective": o,
           "probe_rmse": r, "train_rmse": t, "launches_per_iter": ctx.launch_count()}
    hbm = peaks().get("hbm_gbs", 6544.7)
    if solver == "ccdpp":
        _, _, per_iter = ccd_bytes(A.nnz(), m, n, k, inner)
        out["roofline_whole_iteration"] = {"achieved_gbs": round(per_iter / v / 1e9, 1),
                                           "frac": round(per_iter / v / 1e9 / hbm, 4), "peak": hbm}
        if profile:
            rf = ccdpp_roofline(ctx, it, A.nnz(), m, n, k, inner, v, hbm, cfg_name)
            out["usweep"], out["vsweep"] = rf["usweep"], rf["vsweep"]
    else:
        fl = als_flops(A.nnz(), m, n, k)
        out["useful_tflops"] = round(fl / v / 1e12, 2)
        out["roofline"] = als_roofline(fl, v)
    ctx.close()
    return out, train, probe, A


def ref_side(train, probe, cfg_name, outer, workers):
    m, n, ntr, npr, k, lam, inner, solver, skew = CONFIGS[cfg_name]
    M = ref_matrix(train, m, n)
    rows = ref_train_rows(M, solver, k, lam, inner, outer, workers, probe)
    return [float(x) for x in rows["seconds"]], rows


def extras_n1(args, res):
    """The other BASELINE configs and SURVEY 8f rows on this GPU (N=1, rank 0)."""
    import paper_1511_02433_b200 as P
    cores = os.cpu_count() or 1
    m, n, ntr, npr, k, lam, inner, solver, skew = CONFIGS[args.config]
    ex = {}
    # configs[0]: ML-100K CCD++ k=10, 5 outer iterations, GPU vs the reference on 1 and all cores
    g, tr, pr, _ = side_gpu(P, "ml100k-ccdpp", warm=1, steps=5)
    s1, r1 = ref_side(tr, pr, "ml100k-ccdpp", 5, 1)
    sn, rn = ref_side(tr, pr, "ml100k-ccdpp", 5, cores)
    g["reference_1_worker"] = {"value": float(np.mean(s1)), "per_step_s": s1}
    g["reference_all_cores"] = {"value": float(np.mean(sn)), "per_step_s": sn, "workers": cores}
    g["reference_probe_rmse"] = float(r1["rmse"][-1])
    ex["ml100k"] = g
    # configs[1]: ML-10M ALS k=10
    g, tr, pr, _ = side_gpu(P, "ml10m-als", warm=1, steps=5)
    sn, rn = ref_side(tr, pr, "ml10m-als", 3, cores)
    g["reference_all_cores"] = {"value": float(np.mean(sn)), "per_step_s": sn, "workers": cores}
    g["reference_probe_rmse"] = float(rn["rmse"][-1])
    ex["ml10m_als"] = g
    if args.config == "netflix-ccdpp":
        ctx = res["ctx"]
        # configs[3]: ALS k=40 on the same Netflix-shape data and context
        ctx.als_begin(P.AlsConfig(k=k, lam=lam, outer_iters=1, seed=MODEL_SEED))
        ctx.als_iterate(1)
        ts = list(ctx.als_iterate(max(3, args.steps)))
        o, r, t = ctx.metrics()
        fl = als_flops(res["A"].nnz(), m, n, k)
        ex["als"] = {"config": "netflix-als", "value": float(np.mean(ts)), "unit": "s/outer-iter",
                     "launches_per_iter": ctx.launch_count(), "objective": o, "probe_rmse": r,
                     "useful_tflops": round(fl / float(np.mean(ts)) / 1e12, 2), "flops_per_iter": fl,
                     "roofline": als_roofline(fl, float(np.mean(ts)))}
        # item/user-wise CCD epochs (residual form) on the same context
        ctx.ccd_begin(P.CcdConfig(k=k, lam=lam, outer_iters=1, inner_iters=1, seed=MODEL_SEED))
        ctx.ccd_iterate(1)
        tc = list(ctx.ccd_iterate(3))
        ex["ccd"] = {"metric": "sec/epoch item/user-wise CCD k=40 Netflix shape (residual form)",
                     "value": float(np.mean(tc)), "unit": "s/epoch", "objective": ctx.metrics()[0],
                     "roofline": ccd_epoch_roofline(res["A"].nnz(), k, float(np.mean(tc)), peaks().get("hbm_gbs", 6544.7))}
        # RatingsMatrix::from_triplets on the GPU vs the host build (same bytes out)
        trn = res["train"]
        P.RatingsMatrix.from_triplets(trn[:100000], m, n, device=True)
        t0 = time.perf_counter()
        Ag = P.RatingsMatrix.from_triplets(trn, m, n, device=True)
        t_gpu = time.perf_counter() - t0
        t0 = time.perf_counter()
        Ah = P.RatingsMatrix.from_triplets(trn, m, n)
        t_host = time.perf_counter() - t0
        same = all(np.array_equal(getattr(Ag, f), getattr(Ah, f)) for f in
                   ("row_start", "col_of", "val_row", "col_start", "row_of", "val_col"))
        ex["ingest"] = {"from_triplets_gpu_s": round(t_gpu, 3), "from_triplets_host_s": round(t_host, 3),
                        "host_threads": cores, "bitwise_equal": bool(same), "nnz": int(len(trn))}
        del Ag, Ah
        # triplets -> a ready device context: the host matrix + pmf_ctx_create (layouts built on the host,
        # uploaded) vs pmf_ctx_create_from_triplets (CSR / CSC built and kept on the device, layout streams
        # filled there)
        P.Context.from_triplets(trn[:100000], m, n).close()
        t0 = time.perf_counter()
        cd = P.Context.from_triplets(trn, m, n)
        t_cdev = time.perf_counter() - t0
        li_dev = cd.layout_info()
        cd.close()
        t0 = time.perf_counter()
        ch = P.Context(P.RatingsMatrix.from_triplets(trn, m, n))
        t_chost = time.perf_counter() - t0
        li_host = ch.layout_info()
        ch.close()
        ex["ingest"].update({"ctx_from_triplets_device_s": round(t_cdev, 3), "ctx_via_host_matrix_s": round(t_chost, 3),
                             "same_layouts": li_dev == li_host})
    res["ctx"].close()
    if args.config == "netflix-ccdpp" and not args.quick:
        # configs[4]: Yahoo-Music CCD++ k=100; power-law users at Netflix shape
        ex["yahoo"], *_ = side_gpu(P, "yahoo-ccdpp", warm=1, steps=3, profile=True)
        ex["netflix_skew"], *_ = side_gpu(P, "netflix-skew-ccdpp", warm=1, steps=3, profile=True)
    return ex


def cpu_baseline_n1(args, res):
    """The reference on this box's host cores: ccdpp_train<float> for 2 outer iterations on the same
    matrix, iteration 2 (steady state: iteration 1 skips the build while W = 0) from its TrainReport."""
    m, n, ntr, npr, k, lam, inner, solver, skew = CONFIGS[args.config]
    cores = os.cpu_count() or 1
    try:
        secs, rows = ref_side(res["train"], res["probe"], args.config, 2, cores)
        return {"value": secs[-1], "unit": "s/outer-iter", "cores": cores, "kind": "reference",
                "sample": f"outer iteration 2 of the reference's {solver}_train<float> (2 iterations, "
                          f"workers={cores}) on the full matrix, measured (TrainReport seconds)",
                "iteration_1_s": secs[0], "probe_rmse": float(rows["rmse"][-1])}
    except Exception as e:  # reference library missing on this box
        return {"value": None, "unit": "s/outer-iter", "cores": cores, "kind": "reference",
                "sample": f"unavailable: {e}"}


def relaunch(args):
    """--gpus N outside torchrun: one process per GPU under torch.distributed.run (127.0.0.1)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + os.getpid() % 1000),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="netflix-ccdpp", choices=sorted(CONFIGS))
    ap.add_argument("--quick", action="store_true", help="skip the Yahoo / skewed-users side runs")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip every side measurement")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist = world > 1
    if dist:
        import torch.distributed as td
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        td.init_process_group("gloo")  # host-side barrier / max; the data path is NCCL inside the library
    if args.impl == "reference":
        reference_arm(args, world, rank)
        return
    m, n, ntr, npr, k, lam, inner, solver, skew = CONFIGS[args.config]
    res = run_ours(args, rank, world, dist)
    e2e = None
    if not args.no_e2e:
        if dist:
            e2e = e2e_dist(args, rank, world, dist, res["A"], res["probe"], res["nccl_id"])
        else:
            res["ctx"].close()  # measured with no other context alive
            e2e = e2e_whole_call(args, res["A"], res["probe"])
    extras = {}
    cpu = None
    if rank == 0 and not dist:
        if not args.no_extra:
            if not res["ctx"].h:
                import paper_1511_02433_b200 as P
                res["ctx"] = P.Context(res["A"])
                res["ctx"].set_probe(res["probe"])
            extras = extras_n1(args, res)
        if not args.no_cpu_baseline:
            cpu = cpu_baseline_n1(args, res)
    res["ctx"].close()
    if rank != 0:
        return
    v = res["value"]
    line = {"metric": f"sec/outer-iter {solver} (lower is better)", "value": v, "unit": "s/outer-iter", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_of(args, world), "roofline": res["roofline"], "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(res["launches"] * args.steps), "clocks": res["clocks"],
            "quality": {"objective": res["objective"], "probe_rmse": res["rmse"], "train_rmse": res["train_rmse"]},
            "per_step_s": res["times"]}
    line.update(extras)
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
