"""ctypes bindings for the parity checkers (TEST INFRASTRUCTURE -- never the product path).

* ``Oracle``    -- oracle/build/liborc.so, the C restatement of the reference (pmf_oracle.c).
* ``Reference`` -- oracle/_ref/libparmf_ref.so, the reference headers themselves compiled here
                   (oracle/ref_driver.cpp, oracle/Makefile).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg, ``--impl reference``) may
import this module.  The product package paper_1511_02433_b200 never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_SO = os.path.join(HERE, "build", "liborc.so")
REF_SO = os.path.join(HERE, "_ref", "libparmf_ref.so")

TRIP32 = np.dtype([("user", "<i4"), ("item", "<i4"), ("rating", "<f4")])
TRIP64 = np.dtype([("user", "<i4"), ("item", "<i4"), ("rating", "<f8")])
ITER_ROW = np.dtype([("iteration", "<i4"), ("seconds", "<f8"), ("objective", "<f8"),
                     ("rmse", "<f8"), ("train_rmse", "<f8")], align=True)

P = C.c_void_p
I32, I64, U32, U64, F32, F64 = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_float, C.c_double


def ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def real_of(sfx):
    return (np.float32, F32, TRIP32) if sfx == "_f32" else (np.float64, F64, TRIP64)


class CsrCsc:
    """Host dual-layout matrix (sparse.hpp:64-216 shape) as numpy arrays."""

    def __init__(self, m, n, row_start, col_of, val_row, col_start, row_of, val_col, xlink):
        self.m, self.n = int(m), int(n)
        self.row_start, self.col_of, self.val_row = row_start, col_of, val_row
        self.col_start, self.row_of, self.val_col = col_start, row_of, val_col
        self.xlink = xlink

    @property
    def nnz(self):
        return int(self.row_start[-1])


def _load(path, what):
    if not os.path.exists(path):
        raise RuntimeError(f"{what} not built: {path} (run `make -C oracle`)")
    return C.CDLL(path)


class Oracle:
    def __init__(self):
        self.lib = _load(ORC_SO, "C oracle")
        L = self.lib
        for sfx in ("_f32", "_f64"):
            _, R, _ = real_of(sfx)
            getattr(L, "orc_from_triplets" + sfx).argtypes = [P, I64, I32, I32, P, P, P, P, P, P, P]
            getattr(L, "orc_objective" + sfx).argtypes = [I32, I32, C.c_int, P, P, P, P, P, F64, P]
            getattr(L, "orc_objective" + sfx).restype = F64
            getattr(L, "orc_rmse" + sfx).argtypes = [P, P, C.c_int, P, I64, P]
            getattr(L, "orc_init_random_items" + sfx).argtypes = [P, I64, C.c_int, U64]
            getattr(L, "orc_ccdpp_train" + sfx).argtypes = [C.c_int, R, C.c_int, C.c_int, U64, I32, I32,
                                                            P, P, P, P, P, P, P, P, I64, P, P, P, P, P]
            getattr(L, "orc_als_train" + sfx).argtypes = [C.c_int, R, C.c_int, U64, I32, I32,
                                                          P, P, P, P, P, P, P, I64, P, P, P]
            getattr(L, "orc_ccdpp_update_u" + sfx).argtypes = [I32, P, P, P, P, P, R]
            getattr(L, "orc_ccdpp_update_v" + sfx).argtypes = [I32, P, P, P, P, P, R]
            getattr(L, "orc_ccdpp_build_rhat" + sfx).argtypes = [I32, P, P, P, P, P, P, P]
            getattr(L, "orc_ccdpp_writeback" + sfx).argtypes = [I32, I32, C.c_int, C.c_int, P, P, P,
                                                                P, P, P, P, P, P]
            getattr(L, "orc_als_half" + sfx).argtypes = [I32, P, P, P, P, C.c_int, R, P]
            getattr(L, "orc_cholesky_factor" + sfx).argtypes = [P, C.c_int]
            getattr(L, "orc_cholesky_solve" + sfx).argtypes = [P, P, C.c_int]
            getattr(L, "orc_gram_add_row_upper" + sfx).argtypes = [P, P, C.c_int]
            getattr(L, "orc_gram_finish" + sfx).argtypes = [P, R, C.c_int]
            getattr(L, "orc_top_n" + sfx).argtypes = [P, P, I32, I32, C.c_int, I32, I32, P, I64, P, P]
            getattr(L, "orc_ccd_train" + sfx).argtypes = [C.c_int, R, C.c_int, U64, I32, I32, P, P, P, P, P, P, P,
                                                          P, I64, P, P, P]
        L.orc_random_triplets.argtypes = [I32, I32, I32, U32, F64, F64, P]
        L.orc_random_triplets.restype = I64
        L.orc_planted_full.argtypes = [I32, I32, C.c_int, F64, U32, P]
        L.orc_planted_full.restype = I64
        L.orc_synth_ratings.argtypes = [I32, I32, C.c_int, I64, U32, P]
        L.orc_synth_ratings.restype = I64
        L.orc_carve_probe.argtypes = [P, I64, I64, U32]
        L.orc_partition_balanced.argtypes = [P, I32, C.c_int, P]
        L.orc_mt19937_first.argtypes = [U32, C.c_int]
        L.orc_mt19937_first.restype = U32

    # -- generators (tests/testutil.hpp) ------------------------------------------------------
    def random_triplets(self, m, n, target, seed, lo=1.0, hi=5.0):
        out = np.zeros(target, TRIP64)
        c = self.lib.orc_random_triplets(m, n, target, seed, lo, hi, ptr(out))
        return out[:c]

    def planted_full(self, m, n, k, scale, seed):
        out = np.zeros(m * n, TRIP64)
        self.lib.orc_planted_full(m, n, k, scale, seed, ptr(out))
        return out

    def synth_ratings(self, m, n, rank, target, seed):
        out = np.zeros(target, TRIP64)
        self.lib.orc_synth_ratings(m, n, rank, target, seed, ptr(out))
        return out

    def carve_probe(self, trips, probe_count, seed):
        """returns (train, probe) exactly as testutil.hpp:136-144"""
        t = np.ascontiguousarray(trips.copy())
        self.lib.orc_carve_probe(ptr(t), len(t), probe_count, seed)
        return t[: len(t) - probe_count].copy(), t[len(t) - probe_count:].copy()

    def partition_balanced(self, costs, p):
        costs = np.ascontiguousarray(costs, np.int64)
        b = np.zeros(p + 1, np.int32)
        rc = self.lib.orc_partition_balanced(ptr(costs), len(costs), p, ptr(b))
        if rc:
            raise ValueError("invalid partition arguments")
        return b

    # -- matrix ---------------------------------------------------------------------------------
    def from_triplets(self, trips, m, n, real="_f32"):
        dt, _, td = real_of(real)
        t = np.ascontiguousarray(np.asarray(trips).astype(td))
        nnz = len(t)
        rs = np.zeros(m + 1, np.int64); co = np.zeros(nnz, np.int32); vr = np.zeros(nnz, dt)
        cs = np.zeros(n + 1, np.int64); ro = np.zeros(nnz, np.int32); vc = np.zeros(nnz, dt)
        xl = np.zeros(nnz, np.int64)
        rc = getattr(self.lib, "orc_from_triplets" + real)(ptr(t), nnz, m, n, ptr(rs), ptr(co), ptr(vr),
                                                           ptr(cs), ptr(ro), ptr(vc), ptr(xl))
        if rc == 5:
            raise IndexError("index out of range")
        if rc:
            raise ValueError("invalid triplets (duplicate or non-finite)")
        return CsrCsc(m, n, rs, co, vr, cs, ro, vc, xl)

    def init_random_items(self, n, k, seed, real="_f32"):
        dt, _, _ = real_of(real)
        H = np.zeros(n * k, dt)
        getattr(self.lib, "orc_init_random_items" + real)(ptr(H), n, k, seed)
        return H.reshape(n, k)

    def objective(self, A, W, H, lam, real="_f32"):
        dt, _, _ = real_of(real)
        W = np.ascontiguousarray(W, dt); H = np.ascontiguousarray(H, dt)
        loss = np.zeros(1)
        v = getattr(self.lib, "orc_objective" + real)(A.m, A.n, W.shape[1], ptr(A.row_start),
                                                      ptr(A.col_of), ptr(A.val_row), ptr(W), ptr(H),
                                                      lam, ptr(loss))
        return v, float(loss[0])

    def rmse(self, W, H, probe, real="_f32"):
        dt, _, td = real_of(real)
        W = np.ascontiguousarray(W, dt); H = np.ascontiguousarray(H, dt)
        pr = np.ascontiguousarray(np.asarray(probe).astype(td))
        out = np.zeros(1)
        rc = getattr(self.lib, "orc_rmse" + real)(ptr(W), ptr(H), W.shape[1], ptr(pr), len(pr), ptr(out))
        if rc:
            raise ValueError("probe set is empty")
        return float(out[0])

    def ccd_train(self, A, k, lam, outer, seed, probe=None, real="_f32"):
        """ccd.hpp:310-344 item/user-wise CCD (restated)."""
        dt, _, td = real_of(real)
        pr = np.zeros(0, td) if probe is None else np.ascontiguousarray(np.asarray(probe).astype(td))
        W = np.zeros((A.m, k), dt); H = np.zeros((A.n, k), dt)
        rows = np.zeros(outer, ITER_ROW)
        rc = getattr(self.lib, "orc_ccd_train" + real)(
            k, lam, outer, seed, A.m, A.n, ptr(A.row_start), ptr(A.col_of), ptr(A.val_row),
            ptr(A.col_start), ptr(A.row_of), ptr(A.val_col), ptr(A.xlink), ptr(pr), len(pr),
            ptr(W), ptr(H), ptr(rows))
        if rc:
            raise ValueError("invalid CCD configuration or probe")
        return W, H, rows

    def ccdpp_train(self, A, k, lam, outer, inner, seed, probe=None, real="_f32"):
        dt, _, td = real_of(real)
        pr = np.zeros(0, td) if probe is None else np.ascontiguousarray(np.asarray(probe).astype(td))
        W = np.zeros((A.m, k), dt); H = np.zeros((A.n, k), dt)
        rr = np.zeros(A.nnz, dt); rcl = np.zeros(A.nnz, dt)
        rows = np.zeros(outer, ITER_ROW)
        rc = getattr(self.lib, "orc_ccdpp_train" + real)(
            k, lam, outer, inner, seed, A.m, A.n, ptr(A.row_start), ptr(A.col_of), ptr(A.val_row),
            ptr(A.col_start), ptr(A.row_of), ptr(A.val_col), ptr(A.xlink), ptr(pr), len(pr),
            ptr(W), ptr(H), ptr(rr), ptr(rcl), ptr(rows))
        if rc:
            raise ValueError("invalid CCD++ configuration or probe")
        return W, H, rows, rr, rcl

    def als_train(self, A, k, lam, outer, seed, probe=None, real="_f32"):
        dt, _, td = real_of(real)
        pr = np.zeros(0, td) if probe is None else np.ascontiguousarray(np.asarray(probe).astype(td))
        W = np.zeros((A.m, k), dt); H = np.zeros((A.n, k), dt)
        rows = np.zeros(outer, ITER_ROW)
        rc = getattr(self.lib, "orc_als_train" + real)(
            k, lam, outer, seed, A.m, A.n, ptr(A.row_start), ptr(A.col_of), ptr(A.val_row),
            ptr(A.col_start), ptr(A.row_of), ptr(A.val_col), ptr(pr), len(pr), ptr(W), ptr(H), ptr(rows))
        if rc == 4:
            raise ArithmeticError("not positive definite")
        if rc:
            raise ValueError("invalid ALS configuration or probe")
        return W, H, rows

    def update_u(self, A, rhat_row, v, lam, real="_f32"):
        dt, _, _ = real_of(real)
        u = np.zeros(A.m, dt)
        getattr(self.lib, "orc_ccdpp_update_u" + real)(A.m, ptr(A.row_start), ptr(A.col_of),
                                                       ptr(np.ascontiguousarray(rhat_row, dt)), ptr(u),
                                                       ptr(np.ascontiguousarray(v, dt)), lam)
        return u

    def update_v(self, A, rhat_col, u, lam, real="_f32"):
        dt, _, _ = real_of(real)
        v = np.zeros(A.n, dt)
        getattr(self.lib, "orc_ccdpp_update_v" + real)(A.n, ptr(A.col_start), ptr(A.row_of),
                                                       ptr(np.ascontiguousarray(rhat_col, dt)),
                                                       ptr(np.ascontiguousarray(u, dt)), ptr(v), lam)
        return v

    def build_rhat(self, A, r_row, r_col, u, v, real="_f32"):
        dt, _, _ = real_of(real)
        rr = np.ascontiguousarray(r_row, dt).copy(); rc = np.ascontiguousarray(r_col, dt).copy()
        u = np.ascontiguousarray(u, dt); v = np.ascontiguousarray(v, dt)
        getattr(self.lib, "orc_ccdpp_build_rhat" + real)(A.m, ptr(A.row_start), ptr(A.col_of), ptr(A.xlink),
                                                         ptr(rr), ptr(rc), ptr(u), ptr(v))
        return rr, rc

    def writeback(self, A, r_row, r_col, u, v, k=1, t=0, real="_f32"):
        dt, _, _ = real_of(real)
        rr = np.ascontiguousarray(r_row, dt).copy(); rc = np.ascontiguousarray(r_col, dt).copy()
        u = np.ascontiguousarray(u, dt); v = np.ascontiguousarray(v, dt)
        W = np.zeros((A.m, k), dt); H = np.zeros((A.n, k), dt)
        getattr(self.lib, "orc_ccdpp_writeback" + real)(A.m, A.n, k, t, ptr(A.row_start), ptr(A.col_of),
                                                        ptr(A.xlink), ptr(rr), ptr(rc), ptr(W), ptr(H), ptr(u), ptr(v))
        return rr, rc, W, H

    def als_half(self, A, side, opposing, lam, real="_f32"):
        dt, _, _ = real_of(real)
        k = opposing.shape[1]
        opp = np.ascontiguousarray(opposing, dt)
        if side == 0:
            cnt, st, ix, vals = A.m, A.row_start, A.col_of, A.val_row
        else:
            cnt, st, ix, vals = A.n, A.col_start, A.row_of, A.val_col
        out = np.zeros((cnt, k), dt)
        rc = getattr(self.lib, "orc_als_half" + real)(cnt, ptr(st), ptr(ix), ptr(vals), ptr(opp), k, lam,
                                                      ptr(out))
        if rc == 4:
            raise ArithmeticError("not positive definite")
        return out

    def cholesky_factor(self, a, real="_f64"):
        dt, _, _ = real_of(real)
        a = np.ascontiguousarray(a, dt).copy()
        rc = getattr(self.lib, "orc_cholesky_factor" + real)(ptr(a), a.shape[0])
        if rc == 4:
            raise ArithmeticError("not positive definite")
        return a

    def cholesky_solve(self, l, b, real="_f64"):
        dt, _, _ = real_of(real)
        l = np.ascontiguousarray(l, dt)
        x = np.ascontiguousarray(b, dt).copy()
        rc = getattr(self.lib, "orc_cholesky_solve" + real)(ptr(l), ptr(x), l.shape[0])
        if rc == 6:
            raise ZeroDivisionError("singular triangular factor")
        return x


    def top_n(self, W, H, i, count, rated=(), real="_f32"):
        """model.hpp:172-198; returns [(item, score)] or raises like the reference."""
        npr, R, _ = real_of(real)
        W = np.ascontiguousarray(W, npr); H = np.ascontiguousarray(H, npr)
        m, k = W.shape; n = H.shape[0]
        r = np.ascontiguousarray(rated, np.int32)
        items = np.zeros(max(count, 1), np.int32); scores = np.zeros(max(count, 1), npr)
        kept = getattr(self.lib, "orc_top_n" + real)(ptr(W), ptr(H), m, n, k, i, count, ptr(r), len(r),
                                                      ptr(items), ptr(scores))
        if kept == -1:
            raise ValueError("count must be >= 1")
        if kept == -2:
            raise IndexError("user index out of range")
        return [(int(items[x]), scores[x]) for x in range(kept)]

class Reference:
    """The reference itself (parmf headers compiled in place), through ref_driver.cpp."""

    def __init__(self):
        self.lib = _load(REF_SO, "reference library")
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        for sfx in ("_f32", "_f64"):
            _, R, _ = real_of(sfx)
            f = getattr(L, "ref_matrix_create" + sfx); f.argtypes = [P, I64, I32, I32, P]; f.restype = P
            getattr(L, "ref_matrix_destroy" + sfx).argtypes = [P]
            getattr(L, "ref_matrix_export" + sfx).argtypes = [P] + [P] * 7
            getattr(L, "ref_init_random_items" + sfx).argtypes = [P, I32, C.c_int, U64]
            getattr(L, "ref_objective" + sfx).argtypes = [P, P, P, C.c_int, F64, P]
            getattr(L, "ref_rmse" + sfx).argtypes = [P, P, I32, I32, C.c_int, P, I64, P]
            getattr(L, "ref_ccdpp_train" + sfx).argtypes = [P, C.c_int, R, C.c_int, C.c_int, C.c_int, U64,
                                                            P, I64, P, P, P, P]
            getattr(L, "ref_ccdpp_stage_loop" + sfx).argtypes = [P, C.c_int, R, C.c_int, C.c_int, C.c_int,
                                                                 U64, P, I64, P, P, P, P, P, P, P]
            getattr(L, "ref_als_train" + sfx).argtypes = [P, C.c_int, R, C.c_int, C.c_int, U64, P, I64,
                                                          P, P, P, P]
            getattr(L, "ref_als_epochs" + sfx).argtypes = [P, C.c_int, R, C.c_int, C.c_int, U64, P, I64,
                                                           P, P, P, P, P]
            getattr(L, "ref_ccdpp_update_u" + sfx).argtypes = [P, P, P, P, R]
            getattr(L, "ref_ccdpp_update_v" + sfx).argtypes = [P, P, P, P, R]
            getattr(L, "ref_solve_rows" + sfx).argtypes = [P, C.c_int, P, C.c_int, R, P]
            getattr(L, "ref_cholesky_factor" + sfx).argtypes = [P, C.c_int]
            getattr(L, "ref_cholesky_solve" + sfx).argtypes = [P, P, C.c_int]
            getattr(L, "ref_ccdpp_sample" + sfx).argtypes = [P, C.c_int, R, C.c_int, C.c_int, C.c_int, U64, P]
            getattr(L, "ref_als_sample" + sfx).argtypes = [P, C.c_int, R, C.c_int, C.c_int, U64, P]
            getattr(L, "ref_top_n" + sfx).argtypes = [P, P, I32, I32, C.c_int, I32, I32, P, I64, P, P, P]
            getattr(L, "ref_ccd_train" + sfx).argtypes = [P, C.c_int, R, C.c_int, U64, P, I64, P, P, P]
        L.ref_save_model_f32.argtypes = [C.c_char_p, P, P, I32, I32, C.c_int]
        L.ref_split.argtypes = [P, P, P, I64, F64, U64, P, P, P, P]
        L.ref_load_model_f32.argtypes = [C.c_char_p, P, P, P]
        L.ref_synth_ratings.argtypes = [I32, I32, C.c_int, I64, U32, P]
        L.ref_synth_ratings.restype = I64
        L.ref_random_triplets.argtypes = [I32, I32, C.c_int, U32, F64, F64, P]
        L.ref_random_triplets.restype = I64
        L.ref_planted_full.argtypes = [I32, I32, C.c_int, F64, U32, P]
        L.ref_planted_full.restype = I64
        L.ref_carve_probe.argtypes = [P, I64, I64, U32]
        L.ref_partition_balanced.argtypes = [P, I32, C.c_int, P]

    def _check(self, rc):
        if rc:
            msg = self.lib.ref_last_error().decode()
            if rc == 4:
                raise ArithmeticError(msg)
            if rc == 5:
                raise IndexError(msg)
            if rc == 6:
                raise ZeroDivisionError(msg)
            raise ValueError(msg)

    def split(self, users, items, ratings, ratio, seed):
        """io.hpp:240-285 split_dataset: the probe rows (file order)."""
        u = np.ascontiguousarray(users, np.int64); i = np.ascontiguousarray(items, np.int64)
        r = np.ascontiguousarray(ratings, np.float64)
        pu = np.zeros(max(len(u), 1), np.int64); pi = np.zeros(max(len(u), 1), np.int64)
        pr = np.zeros(max(len(u), 1), np.float64); n = np.zeros(1, np.int64)
        self._check(self.lib.ref_split(ptr(u), ptr(i), ptr(r), len(u), ratio, seed, ptr(pu), ptr(pi), ptr(pr), ptr(n)))
        return pu[:n[0]], pi[:n[0]], pr[:n[0]]

    def save_model(self, path, W, H):
        W = np.ascontiguousarray(W, np.float32); H = np.ascontiguousarray(H, np.float32)
        self._check(self.lib.ref_save_model_f32(os.fsencode(path), ptr(W), ptr(H), W.shape[0], H.shape[0], W.shape[1]))

    def load_model(self, path):
        mnk = np.zeros(3, np.int64)
        self._check(self.lib.ref_load_model_f32(os.fsencode(path), ptr(mnk), None, None))
        W = np.zeros((mnk[0], mnk[2]), np.float32); H = np.zeros((mnk[1], mnk[2]), np.float32)
        self._check(self.lib.ref_load_model_f32(os.fsencode(path), ptr(mnk), ptr(W), ptr(H)))
        return W, H

    def matrix(self, trips, m, n, real="_f32"):
        return RefMatrix(self, trips, m, n, real)

    def synth_ratings(self, m, n, rank, target, seed):
        out = np.zeros(target, TRIP64)
        self.lib.ref_synth_ratings(m, n, rank, target, seed, ptr(out))
        return out

    def random_triplets(self, m, n, target, seed, lo=1.0, hi=5.0):
        out = np.zeros(target, TRIP64)
        c = self.lib.ref_random_triplets(m, n, target, seed, lo, hi, ptr(out))
        return out[:c]

    def planted_full(self, m, n, k, scale, seed):
        out = np.zeros(m * n, TRIP64)
        self.lib.ref_planted_full(m, n, k, scale, seed, ptr(out))
        return out

    def carve_probe(self, trips, probe_count, seed):
        t = np.ascontiguousarray(trips.copy())
        self.lib.ref_carve_probe(ptr(t), len(t), probe_count, seed)
        return t[: len(t) - probe_count].copy(), t[len(t) - probe_count:].copy()

    def partition_balanced(self, costs, p):
        costs = np.ascontiguousarray(costs, np.int64)
        b = np.zeros(p + 1, np.int32)
        self._check(self.lib.ref_partition_balanced(ptr(costs), len(costs), p, ptr(b)))
        return b

    def init_random_items(self, n, k, seed, real="_f32"):
        dt, _, _ = real_of(real)
        H = np.zeros(n * k, dt)
        getattr(self.lib, "ref_init_random_items" + real)(ptr(H), n, k, seed)
        return H.reshape(n, k)

    def rmse(self, W, H, probe, real="_f32"):
        dt, _, td = real_of(real)
        W = np.ascontiguousarray(W, dt); H = np.ascontiguousarray(H, dt)
        pr = np.ascontiguousarray(np.asarray(probe).astype(td))
        out = np.zeros(1)
        self._check(getattr(self.lib, "ref_rmse" + real)(ptr(W), ptr(H), W.shape[0], H.shape[0], W.shape[1],
                                                         ptr(pr), len(pr), ptr(out)))
        return float(out[0])

    def cholesky_factor(self, a, real="_f64"):
        dt, _, _ = real_of(real)
        a = np.ascontiguousarray(a, dt).copy()
        self._check(getattr(self.lib, "ref_cholesky_factor" + real)(ptr(a), a.shape[0]))
        return a

    def cholesky_solve(self, l, b, real="_f64"):
        dt, _, _ = real_of(real)
        l = np.ascontiguousarray(l, dt)
        x = np.ascontiguousarray(b, dt).copy()
        self._check(getattr(self.lib, "ref_cholesky_solve" + real)(ptr(l), ptr(x), l.shape[0]))
        return x


    def top_n(self, W, H, i, count, rated=(), real="_f32"):
        npr, R, _ = real_of(real)
        W = np.ascontiguousarray(W, npr); H = np.ascontiguousarray(H, npr)
        m, k = W.shape; n = H.shape[0]
        r = np.ascontiguousarray(rated, np.int32)
        items = np.zeros(max(count, 1), np.int32); scores = np.zeros(max(count, 1), npr)
        kept = C.c_int32()
        self._check(getattr(self.lib, "ref_top_n" + real)(ptr(W), ptr(H), m, n, k, i, count, ptr(r), len(r),
                                                          ptr(items), ptr(scores), C.byref(kept)))
        return [(int(items[x]), scores[x]) for x in range(kept.value)]

class RefMatrix:
    """parmf::RatingsMatrix<Real> owned by the reference library."""

    def __init__(self, ref, trips, m, n, real):
        self.ref, self.real, self.m, self.n = ref, real, int(m), int(n)
        dt, _, td = real_of(real)
        t = np.ascontiguousarray(np.asarray(trips).astype(td))
        st = C.c_int(0)
        self.h = getattr(ref.lib, "ref_matrix_create" + real)(ptr(t), len(t), m, n, C.byref(st))
        if st.value:
            ref._check(st.value)
        self.nnz = len(t)

    def __del__(self):
        if getattr(self, "h", None):
            getattr(self.ref.lib, "ref_matrix_destroy" + self.real)(self.h)
            self.h = None

    def export(self):
        dt, _, _ = real_of(self.real)
        nnz = self.nnz
        rs = np.zeros(self.m + 1, np.int64); co = np.zeros(nnz, np.int32); vr = np.zeros(nnz, dt)
        cs = np.zeros(self.n + 1, np.int64); ro = np.zeros(nnz, np.int32); vc = np.zeros(nnz, dt)
        xl = np.zeros(nnz, np.int64)
        getattr(self.ref.lib, "ref_matrix_export" + self.real)(self.h, ptr(rs), ptr(co), ptr(vr), ptr(cs),
                                                               ptr(ro), ptr(vc), ptr(xl))
        return CsrCsc(self.m, self.n, rs, co, vr, cs, ro, vc, xl)

    def _probe(self, probe):
        _, _, td = real_of(self.real)
        return np.zeros(0, td) if probe is None else np.ascontiguousarray(np.asarray(probe).astype(td))

    def objective(self, W, H, lam):
        dt, _, _ = real_of(self.real)
        W = np.ascontiguousarray(W, dt); H = np.ascontiguousarray(H, dt)
        out = np.zeros(1)
        self.ref._check(getattr(self.ref.lib, "ref_objective" + self.real)(self.h, ptr(W), ptr(H), W.shape[1],
                                                                           lam, ptr(out)))
        return float(out[0])

    def ccdpp_train(self, k, lam, outer, inner, seed, probe=None, workers=1):
        dt, _, _ = real_of(self.real)
        pr = self._probe(probe)
        W = np.zeros((self.m, k), dt); H = np.zeros((self.n, k), dt)
        rows = np.zeros(outer, ITER_ROW); ts = np.zeros(1)
        self.ref._check(getattr(self.ref.lib, "ref_ccdpp_train" + self.real)(
            self.h, k, lam, outer, inner, workers, seed, ptr(pr), len(pr), ptr(W), ptr(H), ptr(rows), ptr(ts)))
        return W, H, rows

    def ccd_train(self, k, lam, outer, seed, probe=None):
        dt, _, _ = real_of(self.real)
        pr = self._probe(probe)
        W = np.zeros((self.m, k), dt); H = np.zeros((self.n, k), dt)
        rows = np.zeros(outer, ITER_ROW)
        self.ref._check(getattr(self.ref.lib, "ref_ccd_train" + self.real)(
            self.h, k, lam, outer, seed, ptr(pr), len(pr), ptr(W), ptr(H), ptr(rows)))
        return W, H, rows

    def ccdpp_stage_loop(self, k, lam, outer, inner, seed, probe=None, workers=1, history=False):
        """history=True: also the model after every outer iteration, (W_hist, H_hist) [outer, rows, k]."""
        dt, _, _ = real_of(self.real)
        pr = self._probe(probe)
        W = np.zeros((self.m, k), dt); H = np.zeros((self.n, k), dt)
        rr = np.zeros(self.nnz, dt); rc = np.zeros(self.nnz, dt)
        rows = np.zeros(outer, ITER_ROW)
        Wh = np.zeros((outer, self.m, k), dt) if history else None
        Hh = np.zeros((outer, self.n, k), dt) if history else None
        self.ref._check(getattr(self.ref.lib, "ref_ccdpp_stage_loop" + self.real)(
            self.h, k, lam, outer, inner, workers, seed, ptr(pr), len(pr), ptr(W), ptr(H), ptr(rr), ptr(rc),
            ptr(rows), ptr(Wh), ptr(Hh)))
        return (W, H, rows, rr, rc, Wh, Hh) if history else (W, H, rows, rr, rc)

    def als_train(self, k, lam, outer, seed, probe=None, workers=1):
        dt, _, _ = real_of(self.real)
        pr = self._probe(probe)
        W = np.zeros((self.m, k), dt); H = np.zeros((self.n, k), dt)
        rows = np.zeros(outer, ITER_ROW); ts = np.zeros(1)
        self.ref._check(getattr(self.ref.lib, "ref_als_train" + self.real)(
            self.h, k, lam, outer, workers, seed, ptr(pr), len(pr), ptr(W), ptr(H), ptr(rows), ptr(ts)))
        return W, H, rows

    def als_epochs(self, k, lam, outer, seed, probe=None, workers=1, history=False):
        dt, _, _ = real_of(self.real)
        pr = self._probe(probe)
        W = np.zeros((self.m, k), dt); H = np.zeros((self.n, k), dt)
        rows = np.zeros(outer, ITER_ROW)
        Wh = np.zeros((outer, self.m, k), dt) if history else None
        Hh = np.zeros((outer, self.n, k), dt) if history else None
        self.ref._check(getattr(self.ref.lib, "ref_als_epochs" + self.real)(
            self.h, k, lam, outer, workers, seed, ptr(pr), len(pr), ptr(W), ptr(H), ptr(rows), ptr(Wh), ptr(Hh)))
        return (W, H, rows, Wh, Hh) if history else (W, H, rows)

    def update_u(self, rhat_row, v, lam):
        dt, _, _ = real_of(self.real)
        u = np.zeros(self.m, dt)
        self.ref._check(getattr(self.ref.lib, "ref_ccdpp_update_u" + self.real)(
            self.h, ptr(np.ascontiguousarray(rhat_row, dt)), ptr(u), ptr(np.ascontiguousarray(v, dt)), lam))
        return u

    def update_v(self, rhat_col, u, lam):
        dt, _, _ = real_of(self.real)
        v = np.zeros(self.n, dt)
        self.ref._check(getattr(self.ref.lib, "ref_ccdpp_update_v" + self.real)(
            self.h, ptr(np.ascontiguousarray(rhat_col, dt)), ptr(np.ascontiguousarray(u, dt)), ptr(v), lam))
        return v

    def solve_rows(self, side, opposing, lam):
        dt, _, _ = real_of(self.real)
        opp = np.ascontiguousarray(opposing, dt)
        k = opp.shape[1]
        out = np.zeros(((self.m if side == 0 else self.n), k), dt)
        self.ref._check(getattr(self.ref.lib, "ref_solve_rows" + self.real)(self.h, side, ptr(opp), k, lam,
                                                                            ptr(out)))
        return out

    def ccdpp_sample(self, k, lam, inner, workers, steps, seed=1):
        out = np.zeros(1)
        self.ref._check(getattr(self.ref.lib, "ref_ccdpp_sample" + self.real)(
            self.h, k, lam, inner, workers, steps, seed, ptr(out)))
        return float(out[0])

    def als_sample(self, k, lam, workers, epochs, seed=1):
        out = np.zeros(1)
        self.ref._check(getattr(self.ref.lib, "ref_als_sample" + self.real)(
            self.h, k, lam, workers, epochs, seed, ptr(out)))
        return float(out[0])


def have_reference():
    return os.path.exists(REF_SO)
