"""The parmf CLI on the B200 backend (paper_1511_02433_b200/cli.py; tools/parmf_cli.cpp, io.hpp,
report.hpp): split pinned to the reference's split_dataset, rating-file errors, eval known answers
(tests/cli_test.cpp:146-175), exit codes (:222-251).  Host-only; training runs in test_gpu_cli.py."""
import os
import struct
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def cli(args, cwd, env=None):
    e = dict(os.environ, PYTHONPATH=ROOT)
    e.update(env or {})
    r = subprocess.run([sys.executable, "-m", "paper_1511_02433_b200"] + args, cwd=cwd, env=e,
                       capture_output=True, text=True, timeout=300)
    return r.returncode, r.stdout, r.stderr


def fixture(path, m, n, count, seed):
    rng = np.random.default_rng(seed)
    seen = set()
    with open(path, "w") as fh:
        while len(seen) < count:
            u, i = int(rng.integers(1, m + 1)) * 7, int(rng.integers(1, n + 1)) * 3  # sparse external ids
            if (u, i) in seen:
                continue
            seen.add((u, i))
            fh.write(f"{u} {i} {int(rng.integers(1, 6))}\n")


def test_split_matches_reference(reference, tmp_path):
    from paper_1511_02433_b200 import cli as C
    fixture(tmp_path / "all.txt", 30, 20, 200, 3)
    u, i, r = C.read_triplets(tmp_path / "all.txt")
    for ratio, seed in [(0.2, 0), (0.5, 7), (0.9, 123456789012)]:
        (tu, ti, tr), (pu, pi, pr) = C.split_dataset(u, i, r, ratio, seed)
        eu, ei, er = reference.split(u, i, r, ratio, seed)
        assert np.array_equal(pu, eu) and np.array_equal(pi, ei) and np.array_equal(pr, er)
        assert len(tu) + len(pu) == len(u)
    code, out, _ = cli(["split", "--train", "all.txt", "--split-ratio", "0.3", "--seed", "5", "--out", "s"],
                       tmp_path)
    assert code == 0 and out.startswith("train ")
    code2, _, _ = cli(["split", "--train", "all.txt", "--split-ratio", "0.3", "--seed", "5", "--out", "s2"],
                      tmp_path)
    assert (tmp_path / "s" / "probe.txt").read_text() == (tmp_path / "s2" / "probe.txt").read_text()


def test_rating_file_errors(tmp_path):
    from paper_1511_02433_b200 import cli as C
    (tmp_path / "ok.txt").write_text("1 2 3\n\n4\t5 2.5 99\r\n")
    u, i, r = C.read_triplets(tmp_path / "ok.txt")
    assert list(u) == [1, 4] and list(i) == [2, 5] and list(r) == [3.0, 2.5]
    for body, msg in [("1 2 3\nbroken\n", ":2: expected"), ("1 2 x\n", ":1: malformed"),
                      ("1 2 inf\n", ":1: malformed"), ("+1 2 3\n", ":1: malformed"), ("1 2 3 4 5\n", ":1: expected")]:
        (tmp_path / "b.txt").write_text(body)
        with pytest.raises(C.DataError, match=msg):
            C.read_triplets(tmp_path / "b.txt")


def _double_model_dir(d, W, H, users, items):
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, "model.bin"), "wb") as fh:
        fh.write(b"PMFB" + struct.pack("<II", 1, 8) + struct.pack("<qqq", W.shape[0], H.shape[0], W.shape[1]))
        fh.write(np.ascontiguousarray(W, np.float64).tobytes() + np.ascontiguousarray(H, np.float64).tobytes())
    for name, ids in (("user_map.txt", users), ("item_map.txt", items)):
        with open(os.path.join(d, name), "w") as fh:
            fh.write("".join(f"{v}\n" for v in ids))


def test_eval_known_answers(tmp_path):
    _double_model_dir(tmp_path / "m", np.array([[1.0], [1.0]]), np.array([[4.0], [2.0]]), [1, 2], [1, 2])
    (tmp_path / "exact.txt").write_text("1 1 4\n2 1 4\n")
    assert cli(["eval", "m", "--probe", "exact.txt"], tmp_path)[:2] == (0, "0.000000\n")
    (tmp_path / "off.txt").write_text("1 2 4\n")       # prediction 2, rating 4
    assert cli(["eval", "m", "--probe", "off.txt"], tmp_path)[:2] == (0, "2.000000\n")
    (tmp_path / "unseen.txt").write_text("9 9 3\n")    # unseen ids predict 0
    assert cli(["eval", "m", "--probe", "unseen.txt"], tmp_path)[:2] == (0, "3.000000\n")


def test_exit_codes(tmp_path):
    fixture(tmp_path / "all.txt", 10, 8, 40, 4)
    out = ["--out", "u"]
    assert cli(["train", "--train", "all.txt", "--algorithm", "sgd"] + out, tmp_path)[0] == 1
    assert cli(["split", "--train", "all.txt", "--split-ratio", "1.5"], tmp_path)[0] == 1
    assert cli(["train", "--train", "all.txt", "--k", "0"] + out, tmp_path)[0] == 1
    assert cli(["bench", "--train", "all.txt", "--workers", "2,4"], tmp_path)[0] == 1
    assert cli(["train", "--train", "all.txt", "--probe", "all.txt", "--split-ratio", "0.2"] + out, tmp_path)[0] == 1
    assert cli(["train", "--train", "all.txt"], tmp_path)[0] == 1       # --out missing
    assert cli([], tmp_path)[0] == 1
    assert cli(["train", "--train", "nope.txt", "--out", "m"], tmp_path)[0] == 2
    (tmp_path / "bad.txt").write_text("1 2 3\nbroken\n")
    code, _, err = cli(["train", "--train", "bad.txt", "--out", "m"], tmp_path)
    assert code == 2 and ":2:" in err
