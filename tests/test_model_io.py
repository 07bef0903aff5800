"""PMFB model files (model.hpp:211-295): files written by this package load in the
reference and vice versa, bit-exact; the reference's data_error cases (not a model file, truncated,
wrong precision) raise DataError.  Host-only (no GPU)."""
import numpy as np
import pytest


def test_model_roundtrip_with_reference(pmf, reference, tmp_path):
    rng = np.random.default_rng(4)
    model = pmf.FactorModel(rng.normal(0, 1, (13, 5)).astype(np.float32), rng.normal(0, 1, (7, 5)).astype(np.float32))
    ours = tmp_path / "ours.pmfb"
    pmf.save_model(ours, model)
    W, H = reference.load_model(ours)
    assert W.tobytes() == model.w.tobytes() and H.tobytes() == model.h.tobytes()
    theirs = tmp_path / "theirs.pmfb"
    reference.save_model(theirs, model.w, model.h)
    assert theirs.read_bytes() == ours.read_bytes()
    assert pmf.load_model(theirs) == model


def test_model_file_errors(pmf, tmp_path):
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"XXXX" + b"\0" * 40)
    with pytest.raises(pmf.DataError, match="not a model file"):
        pmf.load_model(bad)
    good = tmp_path / "m.pmfb"
    pmf.save_model(good, pmf.FactorModel.zeros(3, 4, 2))
    (tmp_path / "trunc.pmfb").write_bytes(good.read_bytes()[:-4])
    with pytest.raises(pmf.DataError, match="truncated"):
        pmf.load_model(tmp_path / "trunc.pmfb")
    dbl = bytearray(good.read_bytes()); dbl[8] = 8   # scalar width 8: a double model
    (tmp_path / "dbl.pmfb").write_bytes(bytes(dbl))
    with pytest.raises(pmf.DataError, match="precision"):
        pmf.load_model(tmp_path / "dbl.pmfb")
    with pytest.raises(pmf.DataError):
        pmf.load_model(tmp_path / "missing.pmfb")
