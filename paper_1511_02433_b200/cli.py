"""`parmf` command-line front end on the B200 backend (tools/parmf_cli.cpp, io.hpp, report.hpp).

    python -m paper_1511_02433_b200 split --train FILE --split-ratio R [--seed S] [--out DIR]
    python -m paper_1511_02433_b200 train --train FILE [--probe FILE | --split-ratio R] --out DIR
                                          [--algorithm als|ccd|ccdpp] [--k K] [--lambda L]
                                          [--outer-iters N] [--inner-iters N] [--workers W]
                                          [--precision single|double] [--seed S]
    python -m paper_1511_02433_b200 eval MODEL_DIR --probe FILE

Same flags, PARMF_* environment fallbacks (command line wins), rating-file format (whitespace-separated
`user item rating [extra]`, free-form integer ids remapped to dense indices), model directory layout
(model.bin + user_map.txt + item_map.txt), report files (report.jsonl, run.json), printed tables and exit
codes (0 ok, 1 usage / invalid argument, 2 data error, 3 runtime failure) as the reference CLI.  Training
always runs in single precision on the GPU (`--precision double` is accepted and reported as single);
`bench` (worker-count speedup sweeps of the CPU thread pool) has no single-process GPU analogue: use
bench.py.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import re
import sys

import numpy as np

from . import (AlsConfig, Algorithm, CcdConfig, DataError, RatingsMatrix, RunSpec, FactorModel, TRIPLET, lib,
               load_model, run_training, save_model, _check, _ptr)

_INT = re.compile(r"-?[0-9]+\Z")
_SEP = re.compile(rb"[ \t\r]+")
_DBL = re.compile(r"-?([0-9]+\.?[0-9]*|\.[0-9]+)([eE][+-]?[0-9]+)?\Z")


class UsageError(Exception):
    """CLI11::ValidationError / ParseError -> exit code 1."""


# ---- io.hpp ---------------------------------------------------------------------------------------

def read_triplets(path):
    """io.hpp:80-101: (users int64, items int64, ratings float64); data_error naming the line."""
    users, items, ratings = [], [], []
    try:
        fh = open(path, "rb")
    except OSError:
        raise DataError(f"cannot open {path}")
    with fh:
        for lineno, raw in enumerate(fh, 1):
            if raw.endswith(b"\n"):
                raw = raw[:-1]
            fields = [f for f in _SEP.split(raw) if f]  # io.hpp:55-68: ' ', '\t', '\r' separate fields
            if not fields:
                continue
            if len(fields) < 3 or len(fields) > 4:
                raise DataError(f"{path}:{lineno}: expected 'user item rating'")
            try:
                u, i, r = fields[0].decode(), fields[1].decode(), fields[2].decode()
            except UnicodeDecodeError:
                raise DataError(f"{path}:{lineno}: malformed rating line")
            ok = _INT.match(u) and _INT.match(i) and _DBL.match(r)
            if ok:
                uv, iv, rv = int(u), int(i), float(r)
                ok = -(1 << 63) <= uv < (1 << 63) and -(1 << 63) <= iv < (1 << 63) and math.isfinite(rv)
            if not ok:
                raise DataError(f"{path}:{lineno}: malformed rating line")
            users.append(uv)
            items.append(iv)
            ratings.append(rv)
    return np.array(users, np.int64), np.array(items, np.int64), np.array(ratings, np.float64)


def _shortest(x: float) -> str:
    """std::to_chars(double) shortest round-trip form (io.hpp:74-78)."""
    s = repr(float(x))
    if s.endswith(".0"):
        s = s[:-2]
    if "e" in s:
        mant, exp = s.split("e")
        if mant.endswith(".0"):
            mant = mant[:-2]
        sign = "-" if exp.startswith("-") else "+"
        s = f"{mant}e{sign}{exp.lstrip('+-').zfill(2)}"
    return s


def write_triplets(path, users, items, ratings):
    """io.hpp:103-119: one `user item rating` line per entry."""
    try:
        with open(path, "w") as fh:
            fh.write("".join(f"{u} {i} {_shortest(r)}\n" for u, i, r in zip(users.tolist(), items.tolist(),
                                                                          ratings.tolist())))
    except OSError:
        raise DataError(f"cannot open {path} for writing")


class IdMap:
    """io.hpp:123-175: external ids sorted ascending, internal id = position."""

    def __init__(self, ids):
        self.ids = np.asarray(ids, np.int64)

    @staticmethod
    def from_values(values):
        return IdMap(np.unique(np.asarray(values, np.int64)))

    def size(self):
        return len(self.ids)

    def lookup(self, ext):
        """internal ids (int64) of `ext`, -1 where unknown."""
        pos = np.searchsorted(self.ids, ext)
        pos_c = np.minimum(pos, max(len(self.ids) - 1, 0))
        hit = (pos < len(self.ids)) & (self.ids[pos_c] == ext) if len(self.ids) else np.zeros(len(ext), bool)
        return np.where(hit, pos, -1)

    def save(self, path):
        try:
            with open(path, "w") as fh:
                fh.write("".join(f"{v}\n" for v in self.ids.tolist()))
        except OSError:
            raise DataError(f"cannot open {path} for writing")

    @staticmethod
    def load(path):
        try:
            fh = open(path)
        except OSError:
            raise DataError(f"cannot open id map {path}")
        ids = []
        with fh:
            for lineno, line in enumerate(fh, 1):
                line = line.rstrip("\n")
                if not line:
                    continue
                if not _INT.match(line):
                    raise DataError(f"{path}:{lineno}: malformed id")
                ids.append(int(line))
        a = np.array(ids, np.int64)
        if len(a) > 1 and np.any(a[1:] < a[:-1]):
            raise DataError(f"{path}: id map is not sorted")
        return IdMap(a)


def split_dataset(users, items, ratings, ratio, seed):
    """io.hpp:240-285 (the mask comes from pmf_split_mask: std::mt19937, bitwise the reference)."""
    n = len(users)
    mask = np.zeros(max(n, 1), np.uint8)
    got = np.zeros(1, np.int64)
    u = np.ascontiguousarray(users, np.int64)
    _check(lib.pmf_split_mask(_ptr(u), n, float(ratio), int(seed) & ((1 << 64) - 1), _ptr(mask), _ptr(got)))
    m = mask[:n].astype(bool)
    return (users[~m], items[~m], ratings[~m]), (users[m], items[m], ratings[m])


def eval_rmse(model: FactorModel, users: IdMap, items: IdMap, raw):
    """io.hpp:212-230: known pairs predict (Real sum over t), unseen users / items predict 0,
    double accumulation in file order."""
    ru, ri, rr = raw
    if len(ru) == 0:
        raise ValueError("probe set is empty")
    if users.size() != model.users() or items.size() != model.items():
        raise DataError("id maps do not match model dimensions")
    u, i = users.lookup(ru), items.lookup(ri)
    known = (u >= 0) & (i >= 0)
    real = model.w.dtype.type
    pred = np.zeros(len(ru), real)
    w, h = model.w[u[known]], model.h[i[known]]
    acc = np.zeros(int(known.sum()), real)
    for t in range(model.rank()):  # Real, sequential in t, product rounded before the add
        acc = (acc + (w[:, t] * h[:, t]).astype(real)).astype(real)
    pred[known] = acc
    e = rr - pred.astype(np.float64)
    return math.sqrt(float(np.cumsum(e * e)[-1]) / len(ru))  # cumsum: the reference's sequential sum


def _load_model_any(path):
    """model.hpp:251-295: float models through the library, double models read directly."""
    with open(path, "rb") as fh:
        head = fh.read(12)
    if len(head) == 12 and head[:4] == b"PMFB" and int.from_bytes(head[8:12], "little") == 8:
        with open(path, "rb") as fh:
            fh.read(12)
            hdr = fh.read(24)
            if len(hdr) < 24:
                raise DataError(f"model file truncated: {path}")
            m, n, k = (int.from_bytes(hdr[x:x + 8], "little", signed=True) for x in (0, 8, 16))
            if m < 0 or n < 0 or k < 1:
                raise DataError("corrupt model header")
            data = np.frombuffer(fh.read(8 * (m + n) * k), np.float64)
            if len(data) != (m + n) * k:
                raise DataError(f"model file truncated: {path}")
        return FactorModel(data[:m * k].reshape(m, k).copy(), data[m * k:].reshape(n, k).copy())
    return load_model(path)


# ---- report.hpp -----------------------------------------------------------------------------------

def format_report_table(rep):
    """report.hpp:127-144."""
    out = [f"{rep.algorithm} k={rep.k} lambda={_g6(rep.lam)} workers={rep.workers} precision={rep.precision} "
           f"({rep.users} users, {rep.items} items, {rep.nnz} ratings)\n",
           "iter |    seconds |       objective |     rmse\n"]
    for r in rep.rows:
        if math.isnan(r.rmse):
            out.append("%4d | %10.4f | %15.8g |        -\n" % (r.iteration, r.seconds, r.objective))
        else:
            out.append("%4d | %10.4f | %15.8g | %8.6f\n" % (r.iteration, r.seconds, r.objective, r.rmse))
    return "".join(out)


def _g6(x):
    """std::ostream << double (6 significant digits, %g)."""
    return "%g" % x


def _num(x):
    return None if isinstance(x, float) and math.isnan(x) else x


def write_report_jsonl(path, rep):
    """report.hpp:79-93 (nlohmann::json objects: keys sorted, compact)."""
    with open(path, "w") as fh:
        for r in rep.rows:
            fh.write(json.dumps({"iteration": r.iteration, "seconds": r.seconds, "objective": r.objective,
                                 "rmse": _num(r.rmse)}, sort_keys=True, separators=(",", ":")) + "\n")


def write_run_json(path, rep):
    """report.hpp:96-125 (stage totals: the GPU path has none)."""
    doc = {"algorithm": rep.algorithm, "precision": rep.precision, "workers": rep.workers, "k": rep.k,
           "lambda": rep.lam, "outer_iters": rep.outer_iters, "inner_iters": rep.inner_iters, "seed": rep.seed,
           "users": rep.users, "items": rep.items, "nnz": rep.nnz, "train_seconds": rep.train_seconds,
           "wall_seconds": rep.wall_seconds, "final_objective": rep.final_objective,
           "final_rmse": _num(rep.final_rmse), "stages": []}
    with open(path, "w") as fh:
        fh.write(json.dumps(doc, sort_keys=True, indent=2) + "\n")


# ---- parmf_cli.cpp --------------------------------------------------------------------------------

def _env_name(flag):
    return "PARMF_" + flag.upper().replace("-", "_")


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        raise UsageError(message)


def _add(p, flag, env=True, **kw):
    dest = flag.lstrip("-").replace("-", "_")
    if env and _env_name(flag.lstrip("-")) in os.environ:
        kw["default"] = kw.get("type", str)(os.environ[_env_name(flag.lstrip("-"))])
        kw.pop("required", None)
    p.add_argument(flag, dest=dest, **kw)


def _parser():
    ap = _Parser(prog="parmf", description="parmf: parallel matrix factorization for recommender systems "
                                          "(B200 backend)")
    sub = ap.add_subparsers(dest="cmd")
    sp = sub.add_parser("split", help="Split a rating file into train/probe")
    _add(sp, "--train", required=True)
    _add(sp, "--split-ratio", type=float, required=True)
    _add(sp, "--seed", type=int, default=0)
    _add(sp, "--out", default="")
    for name in ("train", "bench"):
        tp = sub.add_parser(name, help="Train a model" if name == "train" else "Speedup sweep (use bench.py)")
        _add(tp, "--train", required=True)
        _add(tp, "--probe", default="")
        _add(tp, "--split-ratio", type=float, default=0.0)
        _add(tp, "--out", required=name == "train", default="")
        _add(tp, "--algorithm", default="ccdpp", choices=["als", "ccd", "ccdpp"])
        _add(tp, "--k", type=int, default=5)
        _add(tp, "--lambda", type=float, default=0.1)
        _add(tp, "--outer-iters", type=int, default=15)
        _add(tp, "--inner-iters", type=int, default=15)
        _add(tp, "--workers", default="")
        _add(tp, "--precision", default="double", choices=["single", "double"])
        _add(tp, "--seed", type=int, default=0)
    ev = sub.add_parser("eval", help="Evaluate a model directory on a probe file")
    ev.add_argument("model_dir")
    _add(ev, "--probe", required=True)
    return ap


def _load_train_probe(o):
    """parmf_cli.cpp:125-141."""
    tu, ti, tr = read_triplets(o.train)
    if len(tu) == 0:
        raise DataError(f"{o.train}: no ratings")
    if o.probe:
        return (tu, ti, tr), read_triplets(o.probe)
    if o.split_ratio != 0.0:
        return split_dataset(tu, ti, tr, o.split_ratio, o.seed)
    return (tu, ti, tr), (np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0))


def _spec(o):
    """parmf_cli.cpp:101-117."""
    algo = {"als": Algorithm.kAls, "ccd": Algorithm.kCcd, "ccdpp": Algorithm.kCcdpp}[o.algorithm]
    if o.k < 1:
        raise UsageError("--k: k must be >= 1")
    if o.__dict__["lambda"] < 0:
        raise UsageError("--lambda: lambda must be >= 0")
    if algo == Algorithm.kAls and not o.__dict__["lambda"] > 0:
        raise UsageError("--lambda: als requires lambda > 0")
    if o.outer_iters < 1 or o.inner_iters < 1:
        raise UsageError("--outer-iters: iteration counts must be >= 1")
    workers = [w for w in (o.workers or "1").split(",") if w]
    if not workers or not all(re.fullmatch(r"[0-9]+", w) and int(w) >= 1 for w in workers):
        raise UsageError("--workers: bad worker count")
    if len(workers) != 1:
        raise UsageError("--workers: train takes a single worker count")
    # --workers W -> W GPU ranks (a device group, ccd.hpp:39 / als.hpp:30; ranks share devices round-robin
    # when W exceeds the device count); item/user-wise CCD always runs one (ccd.hpp:306-309)
    w = int(workers[0]) if algo != Algorithm.kCcd else 1
    return RunSpec(algo, o.k, o.__dict__["lambda"], o.outer_iters, o.inner_iters, w, o.seed)


def run_train(o):
    spec = _spec(o)
    if o.precision == "double":
        # parmf_cli's default is double (parmf_cli.cpp:43); the B200 path computes in FP32 only
        print("warning: --precision double requested; the B200 path trains in single precision "
              "(model.bin holds float32 factors, run.json reports precision=single)", file=sys.stderr)
    (tu, ti, tr), (pu, pi, pr) = _load_train_probe(o)
    users, items = IdMap.from_values(tu), IdMap.from_values(ti)
    t = np.empty(len(tu), TRIPLET)
    t["user"], t["item"], t["rating"] = users.lookup(tu), items.lookup(ti), tr.astype(np.float32)
    qu, qi = users.lookup(pu), items.lookup(pi)
    known = (qu >= 0) & (qi >= 0)
    if (~known).sum():
        print(f"warning: {int((~known).sum())} probe entries reference users/items unseen in training; "
              "eval scores them with prediction 0", file=sys.stderr)
    probe = np.empty(int(known.sum()), TRIPLET)
    probe["user"], probe["item"], probe["rating"] = qu[known], qi[known], pr[known].astype(np.float32)
    a = RatingsMatrix.from_triplets(t, users.size(), items.size())
    model, rep = run_training(spec, a, probe)
    if o.out:
        os.makedirs(o.out, exist_ok=True)
        save_model(os.path.join(o.out, "model.bin"), model)
        users.save(os.path.join(o.out, "user_map.txt"))
        items.save(os.path.join(o.out, "item_map.txt"))
        write_report_jsonl(os.path.join(o.out, "report.jsonl"), rep)
        write_run_json(os.path.join(o.out, "run.json"), rep)
    sys.stdout.write(format_report_table(rep))
    if not math.isnan(rep.final_rmse):
        print("final RMSE %.6f" % rep.final_rmse)
    print("train seconds %.4f (wall %.4f)" % (rep.train_seconds, rep.wall_seconds))
    return 0


def run_split(o):
    """parmf_cli.cpp:177-193."""
    if not 0.0 < o.split_ratio < 1.0:
        raise UsageError("--split-ratio: ratio must be in (0, 1)")
    tu, ti, tr = read_triplets(o.train)
    (au, ai, ar), (bu, bi, br) = split_dataset(tu, ti, tr, o.split_ratio, o.seed)
    out = o.out or "."
    os.makedirs(out, exist_ok=True)
    write_triplets(os.path.join(out, "train.txt"), au, ai, ar)
    write_triplets(os.path.join(out, "probe.txt"), bu, bi, br)
    print(f"train {len(au)} probe {len(bu)} -> {os.path.join(out, 'train.txt')}, {os.path.join(out, 'probe.txt')}")
    return 0


def run_eval(model_dir, probe_path):
    """parmf_cli.cpp:195-211."""
    raw = read_triplets(probe_path)
    if len(raw[0]) == 0:
        raise DataError(f"{probe_path}: no ratings")
    users = IdMap.load(os.path.join(model_dir, "user_map.txt"))
    items = IdMap.load(os.path.join(model_dir, "item_map.txt"))
    model = _load_model_any(os.path.join(model_dir, "model.bin"))
    print("%.6f" % eval_rmse(model, users, items, raw))
    return 0


def main(argv=None):
    try:
        o = _parser().parse_args(argv)
        if not o.cmd:
            raise UsageError("a subcommand is required")
    except UsageError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    except SystemExit as e:  # --help
        return 0 if not e.code else 1
    try:
        if o.cmd == "split":
            return run_split(o)
        if o.cmd == "eval":
            return run_eval(o.model_dir, o.probe)
        if o.probe and o.split_ratio != 0.0:
            raise UsageError("--probe: give either --probe or --split-ratio")
        if o.split_ratio != 0.0 and not 0.0 < o.split_ratio < 1.0:
            raise UsageError("--split-ratio: ratio must be in (0, 1)")
        if o.cmd == "bench":
            raise UsageError("bench: worker-count sweeps are a CPU thread-pool measurement; use bench.py "
                             "for the B200 backend")
        return run_train(o)
    except (UsageError, ValueError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    except DataError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    except IndexError as e:  # out_of_range from the library: a data problem in the files
        print(f"error: {e}", file=sys.stderr)
        return 3
    except MemoryError:
        print("error: out of memory (input too large for this host)", file=sys.stderr)
        return 3
    except Exception as e:  # noqa: BLE001
        print(f"error: {e}", file=sys.stderr)
        return 3


if __name__ == "__main__":
    sys.exit(main())
