"""parmf CLI train on the GPU (parmf_cli.cpp:143-175): split -> train -> eval end to end; the model
directory, report.jsonl and run.json it writes; eval's RMSE of the saved model agrees with the
training report's final RMSE (tests/cli_test.cpp:177-220)."""
import json
import os
import re

import pytest

from test_cli import cli, fixture

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("algo", ["ccdpp", "als", "ccd"])
def test_split_train_eval(tmp_path, algo):
    fixture(tmp_path / "all.txt", 60, 40, 900, 11)
    code, _, err = cli(["split", "--train", "all.txt", "--split-ratio", "0.2", "--seed", "3", "--out", "s"], tmp_path)
    assert code == 0, err
    code, out, err = cli(["train", "--train", "s/train.txt", "--probe", "s/probe.txt", "--algorithm", algo,
                          "--k", "6", "--lambda", "0.5", "--outer-iters", "4", "--inner-iters", "2", "--out", "m"],
                         tmp_path)
    assert code == 0, err
    assert out.splitlines()[1] == "iter |    seconds |       objective |     rmse"
    final = float(re.search(r"final RMSE ([0-9.]+)", out).group(1))
    for f in ("model.bin", "user_map.txt", "item_map.txt", "report.jsonl", "run.json"):
        assert (tmp_path / "m" / f).exists()
    rows = [json.loads(x) for x in (tmp_path / "m" / "report.jsonl").read_text().splitlines()]
    assert [r["iteration"] for r in rows] == [1, 2, 3, 4]
    assert all(set(r) == {"iteration", "seconds", "objective", "rmse"} for r in rows)
    run = json.loads((tmp_path / "m" / "run.json").read_text())
    assert run["algorithm"] == algo and run["k"] == 6 and run["outer_iters"] == 4
    assert run["final_rmse"] == pytest.approx(rows[-1]["rmse"])
    code, out, err = cli(["eval", "m", "--probe", "s/probe.txt"], tmp_path)
    assert code == 0, err
    assert float(out) == pytest.approx(final, abs=2e-6)


def test_split_ratio_train(tmp_path):
    fixture(tmp_path / "all.txt", 50, 30, 600, 12)
    code, out, err = cli(["train", "--train", "all.txt", "--split-ratio", "0.25", "--k", "4", "--outer-iters", "2",
                          "--out", "m"], tmp_path, env={"PARMF_INNER_ITERS": "3"})
    assert code == 0, err
    assert json.loads((tmp_path / "m" / "run.json").read_text())["inner_iters"] == 3
    assert "final RMSE" in out
