"""Model files in the reference format (reference model_io.hpp:124-283), CPU only.

The forest (trees identical to the reference's, from the oracle) is written by
paper_2603_00326_b200.model_io and must be byte-identical to the reference's own save_model output
for the same training run; the reference's validating loader must accept our file, and our loader
must round-trip it and reject corrupted files like the reference does."""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle_lib
import paper_2603_00326_b200 as sofg
from paper_2603_00326_b200 import model_io

pytestmark = pytest.mark.skipif(not oracle_lib.have_reference(), reason="needs the reference build (oracle/_ref)")


def _forest(flat, k, d):
    return sofg.Forest(flat.tree_off, flat.left, flat.right, flat.pred, flat.thr, flat.term_off, flat.feat,
                       flat.weight, flat.breakeven, k, d)


@pytest.mark.parametrize("mode,breakeven,max_depth", [("dynamic", 256, None), ("histogram", None, 6),
                                                      ("exact", None, None)])
def test_save_model_byte_identical_to_reference(tmp_path, mode, breakeven, max_depth):
    ref = oracle_lib.get("reference")
    X, y = ref.generate_trunk(2500, 12, 3)
    kw = dict(n_trees=3, mode=mode, breakeven=breakeven, seed=9, max_depth=max_depth, n_workers=1)
    ref_path = str(tmp_path / "ref.model")
    ref.train_save_model(X, y, 2, oracle_lib.make_config(**kw), ref_path)
    flat = oracle_lib.get("port").train_forest(X, y, 2, oracle_lib.make_config(**kw))
    ours = str(tmp_path / "ours.model")
    model_io.save_model(_forest(flat, 2, 12), sofg.TrainConfig(**kw), ours)
    assert open(ours, "rb").read() == open(ref_path, "rb").read()
    assert ref.load_model_summary(ours) == (3, len(flat.left))


def test_load_model_round_trip_and_validation(tmp_path):
    ref = oracle_lib.get("reference")
    X, y = ref.generate_trunk(1500, 8, 4)
    kw = dict(n_trees=2, mode="dynamic", breakeven=300, seed=1, n_workers=1)
    path = str(tmp_path / "ref.model")
    ref.train_save_model(X, y, 2, oracle_lib.make_config(**kw), path)
    f, cfg, names = model_io.load_model(path)
    assert names == ["0", "1"] and cfg.breakeven == 300 and cfg.mode == "dynamic" and f.n_trees == 2
    again = str(tmp_path / "again.model")
    model_io.save_model(f, cfg, again, label_names=names)
    assert open(again, "rb").read() == open(path, "rb").read()
    blob = bytearray(open(path, "rb").read())
    blob[40] ^= 0xFF
    bad = str(tmp_path / "bad.model")
    open(bad, "wb").write(bytes(blob))
    with pytest.raises(RuntimeError, match="checksum"):
        model_io.load_model(bad)
    with pytest.raises(RuntimeError):
        ref.load_model_summary(bad)


def test_calibration_record_read_by_reference_loader(tmp_path):
    """A calibrated GPU forest stores Forest::calibration (model_io.hpp:155-157); the reference's
    validating loader reads the record back (here a synthetic record on an oracle forest)."""
    ref = oracle_lib.get("reference")
    X, y = ref.generate_trunk(1200, 8, 2)
    kw = dict(n_trees=2, mode="dynamic", breakeven=700, seed=4, n_workers=1)
    flat = oracle_lib.get("port").train_forest(X, y, 2, oracle_lib.make_config(**kw))
    f = _forest(flat, 2, 8)
    f.calibration = model_io.Calibration(breakeven=700, elapsed_seconds=0.0123, fallback=False,
                                         samples=[(64, 1e-6, 3e-6), (700, 5e-6, 6e-6), (65536, 9e-4, 2e-4)])
    cfg = sofg.TrainConfig(n_trees=2, mode="dynamic", seed=4, n_workers=1)  # breakeven absent: calibrated
    path = str(tmp_path / "cal.model")
    model_io.save_model(f, cfg, path)
    assert ref.load_model_calibration(path) == (700, True, 700, 3, False)
    f2, cfg2, _ = model_io.load_model(path)
    assert f2.calibration.samples == [(64, 1e-6, 3e-6), (700, 5e-6, 6e-6), (65536, 9e-4, 2e-4)]
    assert cfg2.breakeven is None and cfg2.calibration.n_max == 65536
    assert model_io.model_bytes(f2, cfg2) == open(path, "rb").read()
