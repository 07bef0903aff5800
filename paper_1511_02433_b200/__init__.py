"""paper_1511_02433_b200 -- B200-native CCD++ / ALS matrix factorisation (arXiv 1511.02433).

Python mirror of the parmf reference interface (/root/reference/proj/include/parmf) over the C-ABI
of ``libpmf_gpu.so`` (include/pmf_gpu.h).  The names, argument meaning and error behaviour follow
the reference so the parity tests read like the reference's own tests:

=====================================  ==========================================================
reference (file:line)                  here
=====================================  ==========================================================
RatingsMatrix::from_triplets           RatingsMatrix.from_triplets         (sparse.hpp:73-149)
CcdConfig / AlsConfig                  CcdConfig / AlsConfig               (ccd.hpp:33, als.hpp:26)
ccdpp_train / als_train                ccdpp_train / als_train             (ccd.hpp:349, als.hpp:188)
run_training(RunSpec, A, probe)        run_training                        (bench.hpp:44-74)
objective / rmse / predict             objective / rmse / predict          (model.hpp:103-167)
init_random_items                      init_random_items (host, mt19937)   (model.hpp:86-93)
ccdpp_build_rhat / update_u / _v /     ccdpp_build_rhat / ccdpp_update_u / (ccd.hpp:235-271)
  writeback                              ccdpp_update_v / ccdpp_writeback
solve_user_row / solve_item_row        solve_user_rows / solve_item_rows   (als.hpp:72-108)
cholesky_factor / cholesky_solve       cholesky_solve_batched              (dense.hpp:74-131)
partition_balanced                     partition_balanced                  (runtime.hpp:91-136)
=====================================  ==========================================================

Exceptions map as the reference's: std::invalid_argument -> ValueError, std::out_of_range ->
IndexError, parmf::data_error -> DataError, parmf::not_positive_definite -> NotPositiveDefinite,
std::domain_error -> DomainError, CUDA/NCCL failures -> RuntimeError.

There is no CPU fallback: every compute call runs the sm_100a kernels of libpmf_gpu.so, and a
missing library or device raises.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field
from enum import Enum
from typing import List, Optional, Sequence

import numpy as np

__all__ = [
    "lib", "LIB_PATH", "TRIPLET", "RatingsMatrix", "CcdConfig", "AlsConfig", "FactorModel", "IterationRow",
    "TrainReport", "ccdpp_train", "als_train", "Algorithm", "RunSpec", "run_training", "rmse", "objective",
    "predict", "init_random_items", "ccdpp_build_rhat", "ccdpp_update_u", "ccdpp_update_v", "ccdpp_writeback",
    "solve_user_rows", "solve_item_rows", "cholesky_solve_batched", "partition_balanced",
    "Context", "DataError", "NotPositiveDefinite", "DomainError", "device_count", "nccl_unique_id", "dist_plan",
    "top_n", "top_n_batch", "ccd_train", "save_model", "load_model",
]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpmf_gpu.so")

# parmf::Triplet<float> (sparse.hpp:20-25) == pmf_triplet, 12 bytes
TRIPLET = np.dtype([("user", "<i4"), ("item", "<i4"), ("rating", "<f4")])
_ITER = np.dtype([("iteration", "<i4"), ("seconds", "<f8"), ("objective", "<f8"), ("rmse", "<f8"),
                  ("train_rmse", "<f8")], align=True)


class DataError(RuntimeError):
    """parmf::data_error (types.hpp:35-38)."""


class DomainError(ArithmeticError):
    """std::domain_error (dense.hpp:110-111)."""


class NotPositiveDefinite(DomainError):
    """parmf::not_positive_definite (types.hpp:41-44)."""


class _MatrixView(C.Structure):
    _fields_ = [("m", C.c_int32), ("n", C.c_int32), ("nnz", C.c_int64),
                ("row_start", C.c_void_p), ("col_of", C.c_void_p), ("val_row", C.c_void_p),
                ("col_start", C.c_void_p), ("row_of", C.c_void_p), ("val_col", C.c_void_p)]


class _CcdConfig(C.Structure):
    _fields_ = [("k", C.c_int32), ("lam", C.c_float), ("outer_iters", C.c_int32), ("inner_iters", C.c_int32),
                ("seed", C.c_uint64), ("num_gpus", C.c_int32), ("flags", C.c_int32)]


class _AlsConfig(C.Structure):
    _fields_ = [("k", C.c_int32), ("lam", C.c_float), ("outer_iters", C.c_int32), ("seed", C.c_uint64),
                ("num_gpus", C.c_int32), ("flags", C.c_int32)]


class _Totals(C.Structure):
    _fields_ = [("train_seconds", C.c_double), ("wall_seconds", C.c_double), ("final_objective", C.c_double),
                ("final_rmse", C.c_double), ("setup_seconds", C.c_double), ("h2d_bytes", C.c_int64),
                ("d2h_bytes", C.c_int64), ("kernel_launches", C.c_int64)]


class _LayoutInfo(C.Structure):
    _fields_ = [(f, C.c_int32) for f in ("n_panels", "panel_size", "smem", "idx16", "promote_fused", "rmw_sub",
                                         "sub_width", "n_units", "n_slots", "ctas")] + \
               [("n_entries", C.c_int64), ("n_real", C.c_int64)]


_P = C.c_void_p
_SIGS = {
    "pmf_last_error": ([], C.c_char_p),
    "pmf_abi_version": ([], C.c_int32),
    "pmf_device_count": ([], C.c_int32),
    "pmf_release_cached_memory": ([C.c_void_p], C.c_int),
    "pmf_ccdpp_train": ([_P, _P, _P, C.c_int64, _P, _P, _P, _P], C.c_int),
    "pmf_als_train": ([_P, _P, _P, C.c_int64, _P, _P, _P, _P], C.c_int),
    "pmf_ccd_train": ([_P, _P, _P, C.c_int64, _P, _P, _P, _P], C.c_int),
    "pmf_ctx_ccd_begin": ([_P, _P], C.c_int),
    "pmf_ctx_ccd_iterate": ([_P, C.c_int32, _P], C.c_int),
    "pmf_rmse": ([_P, _P, C.c_int32, C.c_int32, C.c_int32, _P, C.c_int64, _P], C.c_int),
    "pmf_objective": ([_P, _P, _P, C.c_int32, C.c_double, _P], C.c_int),
    "pmf_ctx_create": ([_P, C.c_int32, _P], C.c_int),
    "pmf_ctx_create_from_triplets": ([_P, C.c_int64, C.c_int32, C.c_int32, C.c_int32, _P], C.c_int),
    "pmf_ctx_create_dist": ([_P, C.c_int32, C.c_int32, C.c_int32, _P, _P], C.c_int),
    "pmf_ctx_create_group": ([_P, C.c_int32, _P, _P], C.c_int),
    "pmf_ctx_destroy": ([_P], C.c_int),
    "pmf_ctx_ccdpp_begin": ([_P, _P], C.c_int),
    "pmf_ctx_ccdpp_iterate": ([_P, C.c_int32, _P], C.c_int),
    "pmf_ctx_als_begin": ([_P, _P], C.c_int),
    "pmf_ctx_als_iterate": ([_P, C.c_int32, _P], C.c_int),
    "pmf_ctx_set_probe": ([_P, _P, C.c_int64], C.c_int),
    "pmf_ctx_metrics": ([_P, _P, _P, _P], C.c_int),
    "pmf_ctx_get_model": ([_P, _P, _P], C.c_int),
    "pmf_ctx_set_model": ([_P, _P, _P, C.c_int32], C.c_int),
    "pmf_ctx_get_residual": ([_P, _P, _P], C.c_int),
    "pmf_ctx_kernel_stats": ([_P, _P, _P, _P, _P], C.c_int),
    "pmf_ctx_set_profiling": ([_P, C.c_int32], C.c_int),
    "pmf_ctx_layout_info": ([_P, C.c_int32, _P], C.c_int),
    "pmf_ctx_launch_count": ([_P, _P], C.c_int),
    "pmf_ctx_debug_sweep_profile": ([_P, C.c_int32, C.c_int32, _P, _P, _P], C.c_int),
    "pmf_ccdpp_build_rhat": ([_P, _P, _P, _P, _P], C.c_int),
    "pmf_ccdpp_update_u": ([_P, _P, _P, _P, C.c_float], C.c_int),
    "pmf_ccdpp_update_v": ([_P, _P, _P, _P, C.c_float], C.c_int),
    "pmf_ccdpp_writeback": ([_P, _P, _P, _P, _P], C.c_int),
    "pmf_als_solve_rows": ([_P, C.c_int32, _P, C.c_int32, C.c_float, _P], C.c_int),
    "pmf_cholesky_solve_batched": ([C.c_int32, C.c_int32, _P, _P], C.c_int),
    "pmf_partition_balanced": ([_P, C.c_int32, C.c_int32, _P], C.c_int),
    "pmf_matrix_from_triplets": ([_P, C.c_int64, C.c_int32, C.c_int32, _P, _P, _P, _P, _P, _P], C.c_int),
    "pmf_matrix_from_triplets_gpu": ([_P, C.c_int64, C.c_int32, C.c_int32, _P, _P, _P, _P, _P, _P], C.c_int),
    "pmf_split_mask": ([_P, C.c_int64, C.c_double, C.c_uint64, _P, _P], C.c_int),
    "pmf_save_model": ([C.c_char_p, _P, _P, C.c_int64, C.c_int64, C.c_int64], C.c_int),
    "pmf_load_model": ([C.c_char_p, _P, _P, _P, _P, _P], C.c_int),
    "pmf_top_n": ([_P, _P, C.c_int32, C.c_int32, C.c_int32, _P, C.c_int32, C.c_int32, _P, _P, _P, _P, _P], C.c_int),
    "pmf_nccl_unique_id": ([_P], C.c_int),
    "pmf_dist_plan": ([_P, C.c_int32, _P, _P, _P, _P], C.c_int),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is not built (run `make -C {HERE}` or __graft_entry__.build()); "
                           "the B200 path has no fallback")
    L = C.CDLL(LIB_PATH)
    for name, (args, res) in _SIGS.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    if L.pmf_abi_version() != 1:
        raise RuntimeError("libpmf_gpu.so ABI mismatch")
    return L


lib = _load()


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _check(status: int):
    if status == 0:
        return
    msg = lib.pmf_last_error().decode(errors="replace")
    if status == 1:
        raise ValueError(msg)
    if status == 2:
        raise DataError(msg)
    if status == 4:
        raise NotPositiveDefinite(msg)
    if status == 5:
        raise IndexError(msg)
    if status == 6:
        raise DomainError(msg)
    raise RuntimeError(msg)


def device_count() -> int:
    return int(lib.pmf_device_count())


def release_cached_memory() -> int:
    """Returns the device blocks cached from destroyed contexts to the driver; bytes released."""
    n = C.c_int64(0)
    _check(lib.pmf_release_cached_memory(C.byref(n)))
    return int(n.value)


def _as_triplets(t) -> np.ndarray:
    if isinstance(t, np.ndarray) and t.dtype == TRIPLET and t.flags.c_contiguous:
        return t  # already the 12-byte Triplet<float> layout: passed zero-copy
    if isinstance(t, np.ndarray) and t.dtype.names and set(("user", "item", "rating")) <= set(t.dtype.names):
        out = np.empty(len(t), TRIPLET)
        out["user"], out["item"], out["rating"] = t["user"], t["item"], t["rating"]
        return out
    arr = np.asarray(list(t), dtype=object) if not isinstance(t, np.ndarray) else t
    out = np.empty(len(arr), TRIPLET)
    for x, (u, i, r) in enumerate(arr):
        out[x] = (u, i, r)
    return out


# ---------------------------------------------------------------------------------------------
# data (sparse.hpp, model.hpp)
# ---------------------------------------------------------------------------------------------

class RatingsMatrix:
    """Dual CSR/CSC ratings matrix (sparse.hpp:64-216) held as host numpy arrays."""

    def __init__(self, m, n, row_start, col_of, val_row, col_start, row_of, val_col):
        self.m, self.n = int(m), int(n)
        self.row_start = np.ascontiguousarray(row_start, np.int64)
        self.col_of = np.ascontiguousarray(col_of, np.int32)
        self.val_row = np.ascontiguousarray(val_row, np.float32)
        self.col_start = np.ascontiguousarray(col_start, np.int64)
        self.row_of = np.ascontiguousarray(row_of, np.int32)
        self.val_col = np.ascontiguousarray(val_col, np.float32)
        self._view = _MatrixView(self.m, self.n, self.nnz(), _ptr(self.row_start), _ptr(self.col_of),
                                 _ptr(self.val_row), _ptr(self.col_start), _ptr(self.row_of), _ptr(self.val_col))

    @staticmethod
    def from_triplets(triplets, m: int, n: int, device: bool = False) -> "RatingsMatrix":
        """Canonical CSR+CSC (sparse.hpp:73-149); IndexError (out_of_range) / ValueError (duplicate,
        non-finite).  device=True builds it on the GPU (pmf_matrix_from_triplets_gpu, bitwise equal)."""
        if m < 0 or n < 0:
            raise ValueError("matrix dimensions must be non-negative")
        t = _as_triplets(triplets)
        nnz = len(t)
        rs = np.empty(m + 1, np.int64); co = np.empty(nnz, np.int32); vr = np.empty(nnz, np.float32)
        cs = np.empty(n + 1, np.int64); ro = np.empty(nnz, np.int32); vc = np.empty(nnz, np.float32)
        fn = lib.pmf_matrix_from_triplets_gpu if device else lib.pmf_matrix_from_triplets
        _check(fn(_ptr(t), nnz, m, n, _ptr(rs), _ptr(co), _ptr(vr), _ptr(cs), _ptr(ro), _ptr(vc)))
        return RatingsMatrix(m, n, rs, co, vr, cs, ro, vc)

    def rows(self):
        return self.m

    def cols(self):
        return self.n

    def nnz(self):
        return int(self.row_start[-1]) if len(self.row_start) else 0

    def row_nnz(self, i):
        return int(self.row_start[i + 1] - self.row_start[i])

    def col_nnz(self, j):
        return int(self.col_start[j + 1] - self.col_start[j])

    def view(self):
        return C.byref(self._view)

    def to_triplets(self) -> np.ndarray:
        out = np.empty(self.nnz(), TRIPLET)
        out["user"] = np.repeat(np.arange(self.m, dtype=np.int32), np.diff(self.row_start))
        out["item"] = self.col_of
        out["rating"] = self.val_row
        return out


@dataclass
class FactorModel:
    """Rank-k model, W m x k and H n x k row-major float32 (model.hpp:24-72)."""
    w: np.ndarray
    h: np.ndarray

    @staticmethod
    def zeros(m, n, k):
        if k < 1:
            raise ValueError("rank must be >= 1")
        return FactorModel(np.zeros((m, k), np.float32), np.zeros((n, k), np.float32))

    def users(self):
        return self.w.shape[0]

    def items(self):
        return self.h.shape[0]

    def rank(self):
        return self.w.shape[1]

    def w_at(self, i, t):
        return self.w[i, t]

    def h_at(self, j, t):
        return self.h[j, t]

    def __eq__(self, o):
        return isinstance(o, FactorModel) and np.array_equal(self.w, o.w) and np.array_equal(self.h, o.h)


def save_model(path, model: "FactorModel"):
    """model.hpp:233-248 save_model: the reference's PMFB v1 file (float), bit-exact round trip."""
    W = np.ascontiguousarray(model.w, np.float32); H = np.ascontiguousarray(model.h, np.float32)
    _check(lib.pmf_save_model(os.fsencode(path), _ptr(W), _ptr(H), W.shape[0], H.shape[0], W.shape[1]))


def load_model(path) -> "FactorModel":
    """model.hpp:270-295 load_model<float>; DataError like the reference's data_error."""
    m, n, k = C.c_int64(), C.c_int64(), C.c_int64()
    _check(lib.pmf_load_model(os.fsencode(path), C.byref(m), C.byref(n), C.byref(k), None, None))
    W = np.empty((m.value, k.value), np.float32); H = np.empty((n.value, k.value), np.float32)
    _check(lib.pmf_load_model(os.fsencode(path), C.byref(m), C.byref(n), C.byref(k), _ptr(W), _ptr(H)))
    return FactorModel(W, H)


def init_random_items(n: int, k: int, seed: int) -> np.ndarray:
    """H of model.hpp:86-93: mt19937(uint32(seed)), (x+1)/2^32 * 1/sqrt(k), row-major draws."""
    gen = _MT19937(seed & 0xFFFFFFFF)
    raw = gen.draw(n * k).astype(np.float64)
    return ((raw + 1.0) * (1.0 / 4294967296.0) * (1.0 / math.sqrt(k))).astype(np.float32).reshape(n, k)


class _MT19937:
    """std::mt19937 (vectorised tempering) -- host-side init only."""

    def __init__(self, seed):
        mt = np.zeros(624, np.uint64)
        mt[0] = seed
        for i in range(1, 624):
            prev = int(mt[i - 1])
            mt[i] = (1812433253 * (prev ^ (prev >> 30)) + i) & 0xFFFFFFFF
        self.mt = mt.astype(np.uint32)
        self.idx = 624

    def _twist(self):
        mt = self.mt.astype(np.uint64)
        for i in range(624):
            y = (int(mt[i]) & 0x80000000) | (int(mt[(i + 1) % 624]) & 0x7FFFFFFF)
            mt[i] = int(mt[(i + 397) % 624]) ^ (y >> 1) ^ (0x9908B0DF if y & 1 else 0)
        self.mt = mt.astype(np.uint32)
        self.idx = 0

    def draw(self, count):
        out = np.empty(count, np.uint32)
        o = 0
        while o < count:
            if self.idx >= 624:
                self._twist()
            take = min(624 - self.idx, count - o)
            y = self.mt[self.idx:self.idx + take].astype(np.uint32)
            y = y ^ (y >> np.uint32(11))
            y = y ^ ((y << np.uint32(7)) & np.uint32(0x9D2C5680))
            y = y ^ ((y << np.uint32(15)) & np.uint32(0xEFC60000))
            y = y ^ (y >> np.uint32(18))
            out[o:o + take] = y
            o += take
            self.idx += take
        return out


# ---------------------------------------------------------------------------------------------
# configs and reports (ccd.hpp:33-50, als.hpp:26-40, report.hpp:25-70, bench.hpp:21-41)
# ---------------------------------------------------------------------------------------------

@dataclass
class CcdConfig:
    k: int = 5
    lam: float = 0.1
    outer_iters: int = 15
    inner_iters: int = 15
    workers: int = 1          # number of GPUs of this process group (1 = this device)
    seed: int = 0

    def validate(self):
        if self.k < 1:
            raise ValueError("k must be >= 1")
        if self.lam < 0:
            raise ValueError("lambda must be >= 0")
        if self.outer_iters < 1:
            raise ValueError("outer_iters must be >= 1")
        if self.inner_iters < 1:
            raise ValueError("inner_iters must be >= 1")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")

    def _c(self):
        return _CcdConfig(self.k, self.lam, self.outer_iters, self.inner_iters, self.seed, self.workers, 0)


@dataclass
class AlsConfig:
    k: int = 5
    lam: float = 0.1
    outer_iters: int = 15
    workers: int = 1
    seed: int = 0
    weighted_lambda: bool = False   # opt-in lambda*n_i*I; the reference uses plain lambda*I

    def validate(self):
        if self.k < 1:
            raise ValueError("k must be >= 1")
        if not self.lam > 0:
            raise ValueError("als requires lambda > 0")
        if self.outer_iters < 1:
            raise ValueError("outer_iters must be >= 1")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")

    def _c(self):
        return _AlsConfig(self.k, self.lam, self.outer_iters, self.seed, self.workers, 1 if self.weighted_lambda else 0)


@dataclass
class IterationRow:
    iteration: int
    seconds: float
    objective: float
    rmse: float
    train_rmse: float


@dataclass
class TrainReport:
    algorithm: str
    precision: str = "single"
    workers: int = 1
    k: int = 0
    lam: float = 0.0
    outer_iters: int = 0
    inner_iters: int = 0
    seed: int = 0
    users: int = 0
    items: int = 0
    nnz: int = 0
    rows: List[IterationRow] = field(default_factory=list)
    train_seconds: float = 0.0
    wall_seconds: float = 0.0
    setup_seconds: float = 0.0
    final_objective: float = 0.0
    final_rmse: float = float("nan")
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    kernel_launches: int = 0


def _probe_arr(probe):
    if probe is None:
        return np.zeros(0, TRIPLET)
    return _as_triplets(probe)


def _report(alg, cfg, a, rows, tot, inner):
    rep = TrainReport(alg, "single", cfg.workers, cfg.k, float(np.float32(cfg.lam)), cfg.outer_iters, inner, cfg.seed,
                      a.m, a.n, a.nnz())
    rep.rows = [IterationRow(int(r["iteration"]), float(r["seconds"]), float(r["objective"]), float(r["rmse"]),
                             float(r["train_rmse"])) for r in rows]
    rep.train_seconds, rep.wall_seconds, rep.setup_seconds = tot.train_seconds, tot.wall_seconds, tot.setup_seconds
    rep.final_objective, rep.final_rmse = tot.final_objective, tot.final_rmse
    rep.h2d_bytes, rep.d2h_bytes, rep.kernel_launches = tot.h2d_bytes, tot.d2h_bytes, tot.kernel_launches
    return rep


def ccdpp_train(config: CcdConfig, a: RatingsMatrix, probe=None):
    """ccd.hpp:349-404 -> (FactorModel, TrainReport) computed on the B200."""
    config.validate()
    pr = _probe_arr(probe)
    W = np.zeros((a.m, config.k), np.float32); H = np.zeros((a.n, config.k), np.float32)
    rows = np.zeros(config.outer_iters, _ITER); tot = _Totals()
    cfg = config._c()
    _check(lib.pmf_ccdpp_train(C.byref(cfg), a.view(), _ptr(pr), len(pr), _ptr(W), _ptr(H), _ptr(rows),
                               C.byref(tot)))
    return FactorModel(W, H), _report("ccdpp", config, a, rows, tot, config.inner_iters)


def ccd_train(config: CcdConfig, a: RatingsMatrix, probe=None):
    """ccd.hpp:310-344 item/user-wise CCD -> (FactorModel, TrainReport) computed on the B200 (one device;
    inner_iters is ignored, as in the reference)."""
    config.validate()
    pr = _probe_arr(probe)
    W = np.zeros((a.m, config.k), np.float32); H = np.zeros((a.n, config.k), np.float32)
    rows = np.zeros(config.outer_iters, _ITER); tot = _Totals()
    cfg = config._c()
    _check(lib.pmf_ccd_train(C.byref(cfg), a.view(), _ptr(pr), len(pr), _ptr(W), _ptr(H), _ptr(rows), C.byref(tot)))
    return FactorModel(W, H), _report("ccd", config, a, rows, tot, 1)


def als_train(config: AlsConfig, a: RatingsMatrix, probe=None):
    """als.hpp:188-233 -> (FactorModel, TrainReport) computed on the B200."""
    config.validate()
    pr = _probe_arr(probe)
    W = np.zeros((a.m, config.k), np.float32); H = np.zeros((a.n, config.k), np.float32)
    rows = np.zeros(config.outer_iters, _ITER); tot = _Totals()
    cfg = config._c()
    _check(lib.pmf_als_train(C.byref(cfg), a.view(), _ptr(pr), len(pr), _ptr(W), _ptr(H), _ptr(rows), C.byref(tot)))
    return FactorModel(W, H), _report("als", config, a, rows, tot, 1)


class Algorithm(Enum):
    kAls = "als"
    kCcd = "ccd"
    kCcdpp = "ccdpp"


@dataclass
class RunSpec:
    """bench.hpp:32-41 (Precision is always single on the B200 path)."""
    algorithm: Algorithm = Algorithm.kCcdpp
    k: int = 5
    lam: float = 0.1
    outer_iters: int = 15
    inner_iters: int = 15
    workers: int = 1
    seed: int = 0


def run_training(spec: RunSpec, a: RatingsMatrix, probe=None):
    """bench.hpp:44-74 dispatch."""
    if spec.algorithm == Algorithm.kAls:
        return als_train(AlsConfig(spec.k, spec.lam, spec.outer_iters, spec.workers, spec.seed), a, probe)
    if spec.algorithm == Algorithm.kCcdpp:
        return ccdpp_train(CcdConfig(spec.k, spec.lam, spec.outer_iters, spec.inner_iters, spec.workers, spec.seed),
                           a, probe)
    if spec.algorithm == Algorithm.kCcd:
        return ccd_train(CcdConfig(spec.k, spec.lam, spec.outer_iters, spec.inner_iters, spec.workers, spec.seed),
                         a, probe)
    raise ValueError("unknown algorithm")


# ---------------------------------------------------------------------------------------------
# metrics (model.hpp:103-167)
# ---------------------------------------------------------------------------------------------

def rmse(model: FactorModel, probe) -> float:
    pr = _probe_arr(probe)
    if len(pr) == 0:
        raise ValueError("probe set is empty")
    W = np.ascontiguousarray(model.w, np.float32); H = np.ascontiguousarray(model.h, np.float32)
    out = C.c_double()
    _check(lib.pmf_rmse(_ptr(W), _ptr(H), W.shape[0], H.shape[0], W.shape[1], _ptr(pr), len(pr), C.byref(out)))
    return out.value


def objective(model: FactorModel, a: RatingsMatrix, lam: float) -> float:
    if lam < 0:
        raise ValueError("lambda must be >= 0")
    if a.m != model.users() or a.n != model.items():
        raise ValueError("model/matrix dimension mismatch")
    W = np.ascontiguousarray(model.w, np.float32); H = np.ascontiguousarray(model.h, np.float32)
    out = C.c_double()
    _check(lib.pmf_objective(a.view(), _ptr(W), _ptr(H), W.shape[1], float(lam), C.byref(out)))
    return out.value


def predict(model: FactorModel, i: int, j: int) -> float:
    """model.hpp:103-114 (host; FP32 sequential over t, products rounded before the add)."""
    if i < 0 or i >= model.users():
        raise IndexError("user index out of range")
    if j < 0 or j >= model.items():
        raise IndexError("item index out of range")
    s = np.float32(0)
    for t in range(model.rank()):
        s = np.float32(s + np.float32(model.w[i, t] * model.h[j, t]))
    return float(s)


# ---------------------------------------------------------------------------------------------
# stage-level entry points (ccd.hpp:233-271, als.hpp:72-108, dense.hpp:55-131)
# ---------------------------------------------------------------------------------------------

def _f32(x, n=None):
    a = np.ascontiguousarray(np.asarray(x, np.float32))
    if n is not None and a.size != n:
        raise ValueError("vector length does not match the matrix")
    return a


def ccdpp_build_rhat(a: RatingsMatrix, r_row, r_col, u, v):
    """Rhat = R + u v^T over rows with u_i != 0, both layouts (returns new arrays)."""
    rr, rc = _f32(r_row, a.nnz()).copy(), _f32(r_col, a.nnz()).copy()
    _check(lib.pmf_ccdpp_build_rhat(a.view(), _ptr(rr), _ptr(rc), _ptr(_f32(u, a.m)), _ptr(_f32(v, a.n))))
    return rr, rc


def ccdpp_writeback(a: RatingsMatrix, r_row, r_col, u, v):
    """R = Rhat - u v^T in both layouts (the residual half of ccdpp_writeback)."""
    rr, rc = _f32(r_row, a.nnz()).copy(), _f32(r_col, a.nnz()).copy()
    _check(lib.pmf_ccdpp_writeback(a.view(), _ptr(rr), _ptr(rc), _ptr(_f32(u, a.m)), _ptr(_f32(v, a.n))))
    return rr, rc


def ccdpp_update_u(a: RatingsMatrix, rhat_row, v, lam) -> np.ndarray:
    u = np.zeros(a.m, np.float32)
    _check(lib.pmf_ccdpp_update_u(a.view(), _ptr(_f32(rhat_row, a.nnz())), _ptr(u), _ptr(_f32(v, a.n)), float(lam)))
    return u


def ccdpp_update_v(a: RatingsMatrix, rhat_col, u, lam) -> np.ndarray:
    v = np.zeros(a.n, np.float32)
    _check(lib.pmf_ccdpp_update_v(a.view(), _ptr(_f32(rhat_col, a.nnz())), _ptr(_f32(u, a.m)), _ptr(v), float(lam)))
    return v


def solve_user_rows(a: RatingsMatrix, item_factors, k: int, lam: float) -> np.ndarray:
    opp = _f32(item_factors).reshape(a.n, k)
    out = np.zeros((a.m, k), np.float32)
    _check(lib.pmf_als_solve_rows(a.view(), 0, _ptr(opp), k, float(lam), _ptr(out)))
    return out


def solve_item_rows(a: RatingsMatrix, user_factors, k: int, lam: float) -> np.ndarray:
    opp = _f32(user_factors).reshape(a.m, k)
    out = np.zeros((a.n, k), np.float32)
    _check(lib.pmf_als_solve_rows(a.view(), 1, _ptr(opp), k, float(lam), _ptr(out)))
    return out


def cholesky_solve_batched(a, b):
    """(L, x) for a batch of SPD systems a[batch,k,k] x = b[batch,k]."""
    A = np.ascontiguousarray(np.asarray(a, np.float32)).copy()
    if A.ndim == 2:
        A = A[None]
    X = np.ascontiguousarray(np.asarray(b, np.float32)).reshape(A.shape[0], A.shape[1]).copy()
    _check(lib.pmf_cholesky_solve_batched(A.shape[0], A.shape[1], _ptr(A), _ptr(X)))
    return A, X


def partition_balanced(costs: Sequence[int], p: int) -> np.ndarray:
    c = np.ascontiguousarray(costs, np.int64)
    b = np.zeros(max(p, 0) + 1, np.int32)
    _check(lib.pmf_partition_balanced(_ptr(c), len(c), p, _ptr(b)))
    return b


def dist_plan(a: RatingsMatrix, world: int):
    """(row_bounds, col_bounds, block_rows, block_cols) used by multi-GPU contexts."""
    rb = np.zeros(world + 1, np.int32); cb = np.zeros(world + 1, np.int32)
    bm, bn = C.c_int32(), C.c_int32()
    _check(lib.pmf_dist_plan(a.view(), world, _ptr(rb), _ptr(cb), C.byref(bm), C.byref(bn)))
    return rb, cb, bm.value, bn.value


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib.pmf_nccl_unique_id(buf))
    return bytes(buf)


def top_n_batch(model: FactorModel, users, count: int, a: "RatingsMatrix" = None, rated=None):
    """model.hpp:172-209 for a batch of users on the B200 (pmf_top_n): the `count` best unrated items
    of each user, score descending, ties by ascending item; scores bitwise predict()'s.  Exclusions:
    the users' rows of `a` (the matrix overload), or `rated` = one strictly increasing list per user.
    Returns (items [len(users), count] with -1 past the end, scores, counts)."""
    users = np.ascontiguousarray(users, np.int32)
    nu = len(users)
    if count < 1:
        raise ValueError("count must be >= 1")  # model.hpp:175, checked before the user (:176-177)
    if nu and (users.min() < 0 or users.max() >= model.users()):
        raise IndexError("user index out of range")
    if a is not None:
        if rated is not None:
            raise ValueError("pass either a or rated")
        lo = a.row_start[users] if nu else np.zeros(0, np.int64)
        ln = (a.row_start[users + 1] - lo) if nu else np.zeros(0, np.int64)
        ex_start = np.concatenate([[0], np.cumsum(ln)]).astype(np.int64)
        # gather the users' rows in one vectorised index: position p of user u -> lo[u] + (p - ex_start[u])
        pos = np.repeat(lo - ex_start[:-1], ln) + np.arange(int(ex_start[-1]), dtype=np.int64)
        ex = a.col_of[pos]
    else:
        lists = [np.asarray(r, np.int32) for r in (rated if rated is not None else [()] * nu)]
        if len(lists) != nu:
            raise ValueError("one rated list per user")
        ex_start = np.concatenate([[0], np.cumsum([len(r) for r in lists])]).astype(np.int64)
        ex = np.concatenate(lists).astype(np.int32) if lists else np.zeros(0, np.int32)
    ex = np.ascontiguousarray(ex, np.int32) if len(ex) else np.zeros(1, np.int32)
    W = np.ascontiguousarray(model.w, np.float32); H = np.ascontiguousarray(model.h, np.float32)
    c = max(int(count), 1)
    items = np.empty((nu, c), np.int32); scores = np.empty((nu, c), np.float32); counts = np.empty(nu, np.int32)
    _check(lib.pmf_top_n(_ptr(W), _ptr(H), W.shape[0], H.shape[0], W.shape[1], _ptr(users), nu, int(count),
                         _ptr(ex_start), _ptr(ex), _ptr(items), _ptr(scores), _ptr(counts)))
    return items, scores, counts


def top_n(model: FactorModel, *args):
    """The reference's two overloads (model.hpp:172, :203): top_n(model, i, count, rated_sorted) and
    top_n(model, a, i, count) -> [(item, score)], computed on the B200."""
    if args and isinstance(args[0], RatingsMatrix):
        a, i, count = args
        items, scores, counts = top_n_batch(model, [i], count, a=a)
    else:
        i, count = args[0], args[1]
        rated = args[2] if len(args) > 2 else ()
        items, scores, counts = top_n_batch(model, [i], count, rated=[rated])
    return [(int(items[0, x]), float(scores[0, x])) for x in range(counts[0])]


# ---------------------------------------------------------------------------------------------
# resident context
# ---------------------------------------------------------------------------------------------

class _Shape:
    """m, n, nnz() of a context built from triplets (no host matrix)."""

    def __init__(self, m, n, nnz):
        self.m, self.n, self._nnz = m, n, nnz

    def nnz(self):
        return self._nnz


class Context:
    """Matrix resident in HBM (pmf_ctx); CCD++ / ALS state, metrics and model I/O."""

    def __init__(self, a: RatingsMatrix, device: int = -1, rank: int = 0, world: int = 1, nccl_id: bytes = None,
                 gpus: int = 1, devices=None):
        """One device (default), one rank of a multi-process NCCL job (rank / world / nccl_id), or a
        device group of `gpus` ranks driven by this process (pmf_ctx_create_group; `devices` lists
        each rank's device, default rank mod device_count())."""
        self.a = a
        self.h = C.c_void_p()
        if gpus != 1 or devices is not None:
            if gpus < 1:
                raise ValueError("workers must be >= 1")
            dv = None if devices is None else np.ascontiguousarray(devices, np.int32)
            if dv is not None and len(dv) != gpus:
                raise ValueError("devices must list one device per rank")
            _check(lib.pmf_ctx_create_group(a.view(), gpus, _ptr(dv), C.byref(self.h)))
        elif nccl_id is None:
            _check(lib.pmf_ctx_create(a.view(), device, C.byref(self.h)))
        else:
            idb = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
            _check(lib.pmf_ctx_create_dist(a.view(), device, rank, world, idb, C.byref(self.h)))
        self.k = 0

    @classmethod
    def from_triplets(cls, triplets, m: int, n: int, device: int = -1) -> "Context":
        """RatingsMatrix.from_triplets + Context in one step with the matrix built on the device
        (pmf_ctx_create_from_triplets): the CSR / CSC never travel back to the host.  Same errors as
        from_triplets; layouts (and so every result) bitwise those of Context(RatingsMatrix...)."""
        if m < 0 or n < 0:
            raise ValueError("matrix dimensions must be non-negative")
        t = _as_triplets(triplets)
        self = cls.__new__(cls)
        self.a = _Shape(m, n, len(t))
        self.h = C.c_void_p()
        _check(lib.pmf_ctx_create_from_triplets(_ptr(t), len(t), m, n, device, C.byref(self.h)))
        self.k = 0
        return self

    def close(self):
        if self.h:
            lib.pmf_ctx_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def ccdpp_begin(self, config: CcdConfig):
        config.validate()
        cfg = config._c()
        _check(lib.pmf_ctx_ccdpp_begin(self.h, C.byref(cfg)))
        self.k = config.k

    def ccdpp_iterate(self, n: int = 1) -> np.ndarray:
        secs = np.zeros(n)
        _check(lib.pmf_ctx_ccdpp_iterate(self.h, n, _ptr(secs)))
        return secs

    def ccd_begin(self, config: CcdConfig):
        """Item/user-wise CCD (ccd.hpp:52-125) on the resident matrix."""
        config.validate()
        cfg = config._c()
        _check(lib.pmf_ctx_ccd_begin(self.h, C.byref(cfg)))
        self.k = config.k

    def ccd_iterate(self, n: int = 1) -> np.ndarray:
        secs = np.zeros(n)
        _check(lib.pmf_ctx_ccd_iterate(self.h, n, _ptr(secs)))
        return secs

    def als_begin(self, config: AlsConfig):
        config.validate()
        cfg = config._c()
        _check(lib.pmf_ctx_als_begin(self.h, C.byref(cfg)))
        self.k = config.k

    def als_iterate(self, n: int = 1) -> np.ndarray:
        secs = np.zeros(n)
        _check(lib.pmf_ctx_als_iterate(self.h, n, _ptr(secs)))
        return secs

    def set_probe(self, probe):
        self._probe = _probe_arr(probe)
        _check(lib.pmf_ctx_set_probe(self.h, _ptr(self._probe), len(self._probe)))

    def metrics(self):
        o, r, t = C.c_double(), C.c_double(), C.c_double()
        _check(lib.pmf_ctx_metrics(self.h, C.byref(o), C.byref(r), C.byref(t)))
        return o.value, r.value, t.value

    def model(self) -> FactorModel:
        W = np.zeros((self.a.m, self.k), np.float32); H = np.zeros((self.a.n, self.k), np.float32)
        _check(lib.pmf_ctx_get_model(self.h, _ptr(W), _ptr(H)))
        return FactorModel(W, H)

    def set_model(self, model: FactorModel):
        W = np.ascontiguousarray(model.w, np.float32); H = np.ascontiguousarray(model.h, np.float32)
        _check(lib.pmf_ctx_set_model(self.h, _ptr(W), _ptr(H), W.shape[1]))

    def residual(self):
        rr = np.zeros(self.a.nnz(), np.float32); rc = np.zeros(self.a.nnz(), np.float32)
        _check(lib.pmf_ctx_get_residual(self.h, _ptr(rr), _ptr(rc)))
        return rr, rc

    def set_profiling(self, on: bool):
        _check(lib.pmf_ctx_set_profiling(self.h, 1 if on else 0))

    def layout_info(self) -> dict:
        """Device layout of both sides (panels, promote split, units) -- pmf_ctx_layout_info."""
        out = {}
        for side, name in ((0, "csr"), (1, "csc")):
            li = _LayoutInfo()
            _check(lib.pmf_ctx_layout_info(self.h, side, C.byref(li)))
            d = {f: getattr(li, f) for f, _ in li._fields_}
            for f in ("smem", "idx16", "promote_fused"):
                d[f] = bool(d[f])
            out[name] = d
        return out

    def debug_sweep_profile(self, side: int, promote: bool = False):
        n = C.c_int32()
        clk = np.zeros(2 * 1024, np.uint64); st = np.zeros(24 * 1024, np.int64)
        _check(lib.pmf_ctx_debug_sweep_profile(self.h, side, 1 if promote else 0, _ptr(clk), _ptr(st), C.byref(n)))
        c = n.value
        return clk[:2 * c].reshape(c, 2), st[:24 * c].reshape(c, 24)

    def launch_count(self) -> int:
        n = C.c_int64()
        _check(lib.pmf_ctx_launch_count(self.h, C.byref(n)))
        return n.value

    def kernel_stats(self):
        um, vm = C.c_double(), C.c_double()
        un, vn = C.c_int64(), C.c_int64()
        _check(lib.pmf_ctx_kernel_stats(self.h, C.byref(um), C.byref(un), C.byref(vm), C.byref(vn)))
        return {"usweep_ms": um.value, "usweep_launches": un.value, "vsweep_ms": vm.value,
                "vsweep_launches": vn.value}
