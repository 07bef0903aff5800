"""Multi-rank CPU tests (gloo, world_size 2) of the multi-GPU decomposition used by
pmf_ctx_create_dist: the library's own plan (pmf_dist_plan: partition_balanced row / column blocks,
runtime.hpp:91-136, and the padded index space for equal-count all-gathers) drives a distributed
CCD++ schedule in which every rank updates only its CSR row block and CSC column block and the only
exchange is an all-gather of u after each u-sweep and of v after each v-sweep.  The per-block math is
the oracle's (test infrastructure), so the result must equal the single-process reference run
bit-for-bit -- this pins the claim that residual updates never cross ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as td
import torch.multiprocessing as mp


class _Blk:
    """CSR (or CSC) restricted to a contiguous block of outputs, as the oracle stage calls expect."""

    def __init__(self, start, idx, count):
        self.row_start = self.col_start = start
        self.col_of = self.row_of = idx
        self.m = self.n = count


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _allgather_padded(local, block, bounds, world):
    """ncclAllGather of equal-count padded blocks, then unpadding (the library's padded space)."""
    buf = np.zeros(block, np.float32)
    buf[:len(local)] = local
    out = [torch.zeros(block, dtype=torch.float32) for _ in range(world)]
    td.all_gather(out, torch.from_numpy(buf))
    return np.concatenate([out[r].numpy()[:bounds[r + 1] - bounds[r]] for r in range(world)])


def _worker(rank, world, port, payload, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, payload["root"])
        from oracle.pyoracle import Oracle
        O = Oracle()
        A = payload["A"]
        k, lam, outer, inner, seed = payload["cfg"]
        rb, cb, Bm, Bn = payload["plan"]
        r0, r1, c0, c1 = rb[rank], rb[rank + 1], cb[rank], cb[rank + 1]
        f32 = np.float32
        # local CSR row block / CSC column block (the only residual copies this rank owns)
        rs = A.row_start[r0:r1 + 1] - A.row_start[r0]
        co = A.col_of[A.row_start[r0]:A.row_start[r1]].copy()
        Rr = A.val_row[A.row_start[r0]:A.row_start[r1]].copy()
        rows_of_entry = np.repeat(np.arange(r0, r1), np.diff(rs))
        cs = A.col_start[c0:c1 + 1] - A.col_start[c0]
        ro = A.row_of[A.col_start[c0]:A.col_start[c1]].copy()
        Rc = A.val_col[A.col_start[c0]:A.col_start[c1]].copy()
        cols_of_entry = np.repeat(np.arange(c0, c1), np.diff(cs))
        csr, csc = _Blk(rs, co, r1 - r0), _Blk(cs, ro, c1 - c0)
        W = np.zeros((A.m, k), f32)
        H = O.init_random_items(A.n, k, seed)
        for _ in range(outer):
            for t in range(k):
                u, v = W[:, t].copy(), H[:, t].copy()
                # build-rhat on both local layouts, identical arithmetic (ccd.hpp:142-147)
                ur, uc = u[rows_of_entry], u[ro]
                Rr = np.where(ur != 0, Rr + (ur * v[co]).astype(f32), Rr).astype(f32)
                Rc = np.where(uc != 0, Rc + (uc * v[cols_of_entry]).astype(f32), Rc).astype(f32)
                for _s in range(inner):
                    u = _allgather_padded(O.update_u(csr, Rr, v, lam), Bm, rb, world)
                    v = _allgather_padded(O.update_v(csc, Rc, u, lam), Bn, cb, world)
                W[:, t], H[:, t] = u, v
                # writeback R = Rhat - u v^T (ccd.hpp:213-214), no skip
                Rr = (Rr - (u[rows_of_entry] * v[co]).astype(f32)).astype(f32)
                Rc = (Rc - (u[ro] * v[cols_of_entry]).astype(f32)).astype(f32)
        # distributed metric: local squared-error sum over the CSR block, all-reduced
        _, loss = O.objective(type("M", (), {"m": r1 - r0, "n": A.n, "row_start": rs, "col_of": co,
                                             "val_row": A.val_row[A.row_start[r0]:A.row_start[r1]]})(),
                              W[r0:r1], H, 0.0)
        tot = torch.tensor([loss], dtype=torch.float64)
        td.all_reduce(tot)
        if rank == 0:
            q.put((W, H, Rr, float(tot.item())))
    finally:
        td.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_distributed_ccdpp_schedule_matches_reference(oracle, pmf, world):
    t = oracle.synth_ratings(300, 200, 3, 8000, 11)
    A = oracle.from_triplets(t, 300, 200)
    Ap = pmf.RatingsMatrix.from_triplets(t, 300, 200)
    rb, cb, Bm, Bn = pmf.dist_plan(Ap, world)
    assert rb[0] == 0 and rb[-1] == 300 and cb[-1] == 200
    assert Bm == max(np.diff(rb)) and Bn == max(np.diff(cb))
    # the plan is the reference's partition_balanced over 4|Omega| costs
    assert np.array_equal(rb, oracle.partition_balanced(4 * np.diff(A.row_start), world))
    assert np.array_equal(cb, oracle.partition_balanced(4 * np.diff(A.col_start), world))
    cfg = (3, 0.05, 2, 3, 7)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    payload = {"A": A, "cfg": cfg, "plan": (rb, cb, Bm, Bn), "root": root}
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, payload, q)) for r in range(world)]
    for p in procs:
        p.start()
    W, H, _, loss = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    Wr, Hr, rows, _, _ = oracle.ccdpp_train(A, 3, 0.05, 2, 3, 7)
    assert np.array_equal(W, Wr) and np.array_equal(H, Hr)   # bit-identical to the single-process run
    _, loss_ref = oracle.objective(A, Wr, Hr, 0.0)
    assert abs(loss - loss_ref) <= 1e-12 * loss_ref


def test_dist_plan_edge_cases(pmf):
    A = pmf.RatingsMatrix.from_triplets([(0, 0, 1.0), (3, 2, 2.0)], 5, 4)
    rb, cb, Bm, Bn = pmf.dist_plan(A, 8)          # more ranks than work: empty blocks allowed
    assert len(rb) == 9 and rb[-1] == 5 and cb[-1] == 4 and np.all(np.diff(rb) >= 0)
    rb1, cb1, Bm1, Bn1 = pmf.dist_plan(A, 1)
    assert list(rb1) == [0, 5] and Bm1 == 5 and Bn1 == 4
    with pytest.raises(ValueError):
        pmf.dist_plan(A, 0)


def test_bench_relaunches_ranks_for_the_reference_arm():
    """bench.py --gpus 2 outside torchrun relaunches itself as 2 ranks (torch.distributed.run, 127.0.0.1);
    the reference arm runs on rank 0 only and prints exactly one JSON line (CPU, gloo)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--config", "ml100k-ccdpp", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 0
