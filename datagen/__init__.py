"""Synthetic rating corpora (libpmf_synth.so, synth.cpp): the recipe of the reference's
tests/testutil.hpp:91-132 on per-user parallel streams, optionally power-law on users.

Shared by both bench arms and the large-shape tests; it does not load the product library, so the
reference arm of bench.py stays free of it."""
import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpmf_synth.so")
TRIPLET = np.dtype([("user", "<i4"), ("item", "<i4"), ("rating", "<f4")])  # parmf::Triplet<float>

if not os.path.exists(LIB_PATH):
    raise RuntimeError(f"{LIB_PATH} is not built (make -C {HERE})")
_lib = C.CDLL(LIB_PATH)
_lib.dg_synth_ratings.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_int64, C.c_uint32, C.c_double,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
_lib.dg_synth_ratings.restype = C.c_int
_lib.dg_last_error.restype = C.c_char_p


def synth_ratings(m, n, true_rank, n_train, n_probe, seed, user_skew=0.0):
    """(train, probe) Triplet<float> arrays: n_train + n_probe distinct ratings of an m x n matrix,
    the probe carved per user in proportion to its count.  user_skew > 0: per-user counts follow a
    power law with that exponent over a seeded user permutation (capped at n)."""
    tr = np.empty(n_train, TRIPLET)
    pr = np.empty(n_probe, TRIPLET)
    gt, gp = C.c_int64(), C.c_int64()
    rc = _lib.dg_synth_ratings(m, n, true_rank, n_train, n_probe, seed, float(user_skew),
                               tr.ctypes.data_as(C.c_void_p), pr.ctypes.data_as(C.c_void_p), C.byref(gt),
                               C.byref(gp))
    if rc != 0:
        raise ValueError(_lib.dg_last_error().decode())
    return tr[:gt.value], pr[:gp.value]
