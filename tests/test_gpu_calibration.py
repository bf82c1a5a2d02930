"""Dynamic-switch calibration and training instrumentation on the GPU.

* train_forest in Dynamic mode with no breakeven calibrates (forest.hpp:285-293): the record is the
  reference's CrossoverCalibration (calibrate.hpp:34-41) produced by the reference's search
  (calibrate.hpp:51-112) over GPU probes; the trees are the reference's trees at the calibrated
  breakeven; save_model writes the record and the reference's validating loader reads it back.
* TrainInstrumentation (timing.hpp:39-79): per-depth node and sample counts equal the reference's
  for the same forest (they depend only on the trees), and the phase / depth seconds are positive
  device times.
"""
import numpy as np
import pytest

import oracle_lib

pytestmark = pytest.mark.gpu


def _bad_trees(g, o):
    ff = oracle_lib.FlatForest(g.tree_off, g.left, g.right, g.pred, g.thr, g.term_off, g.feat, g.weight)
    return [t for t in range(o.n_trees) if not ff.tree_equal(o, t)]


def test_train_forest_calibrates_when_breakeven_absent(gpu_ctx, oracle, tmp_path):
    import paper_2603_00326_b200 as sofg
    from paper_2603_00326_b200 import model_io

    X, y = oracle.generate_trunk(20000, 64, 5)
    gpu_ctx.upload(X, y, 2)
    cfg = sofg.TrainConfig(n_trees=4, mode="dynamic", seed=3, n_workers=8)
    g = gpu_ctx.train_forest(cfg)
    cal = g.calibration
    assert cal is not None
    assert not cal.fallback or cal.breakeven == 1024
    assert g.breakeven == cal.breakeven
    assert 64 <= cal.breakeven <= 65537
    ns = [s[0] for s in cal.samples]
    assert ns == sorted(ns) and ns[0] == 64
    if len(ns) == 1:  # the histogram probe already won at n_min (calibrate.hpp:84)
        assert cal.breakeven == 64
    assert all(e > 0 and h > 0 for _, e, h in cal.samples)
    assert cal.elapsed_seconds > 0
    # the trees are the reference's at the calibrated breakeven
    o = oracle.train_forest(X, y, 2, oracle_lib.make_config(n_trees=4, mode="dynamic", breakeven=g.breakeven,
                                                            seed=3, n_workers=8))
    assert _bad_trees(g, o) == []
    # Forest::calibration is serialized (model_io.hpp:155-157) and the reference loader accepts it
    if oracle_lib.have_reference():
        path = str(tmp_path / "cal.model")
        model_io.save_model(g, cfg, path)
        ref = oracle_lib.get("reference")
        be, has_cal, cal_be, n_samp, fb = ref.load_model_calibration(path)
        assert (be, has_cal, cal_be, n_samp, fb) == (g.breakeven, True, cal.breakeven, len(cal.samples),
                                                     cal.fallback)
        f2, cfg2, _ = model_io.load_model(path)
        assert f2.calibration.breakeven == cal.breakeven and cfg2.breakeven is None


def test_calibrate_options_and_errors(gpu_ctx, oracle):
    import paper_2603_00326_b200 as sofg
    from paper_2603_00326_b200.model_io import CalibrationOptions

    X, y = oracle.generate_trunk(8000, 32, 2)
    gpu_ctx.upload(X, y, 2)
    opts = CalibrationOptions(n_min=16, n_max=4096, budget_seconds=0.05, repetitions=3)
    cal = gpu_ctx.calibrate(sofg.TrainConfig(calibration=opts))
    assert 16 <= cal.breakeven <= 4097
    assert [s[0] for s in cal.samples][0] == 16
    with pytest.raises(ValueError, match="n_min"):
        gpu_ctx.calibrate(sofg.TrainConfig(calibration=CalibrationOptions(n_min=100, n_max=100)))
    with pytest.raises(ValueError, match="repetitions"):
        gpu_ctx.calibrate(sofg.TrainConfig(calibration=CalibrationOptions(repetitions=0)))
    # an explicit breakeven is used as is: no calibration record (forest.hpp:286-287)
    g = gpu_ctx.train_forest(sofg.TrainConfig(n_trees=2, mode="dynamic", breakeven=300, seed=1))
    assert g.calibration is None and g.breakeven == 300
    # non-dynamic modes neither calibrate nor store a breakeven (forest.hpp:285)
    g = gpu_ctx.train_forest(sofg.TrainConfig(n_trees=2, mode="histogram", seed=1))
    assert g.calibration is None and g.breakeven == 0


@pytest.mark.parametrize("mode,breakeven,max_depth", [("dynamic", 256, None), ("exact", None, None),
                                                      ("histogram", None, 7)])
def test_instrumentation_depth_counts_match_reference(gpu_ctx, oracle, mode, breakeven, max_depth):
    import paper_2603_00326_b200 as sofg

    if not oracle_lib.have_reference():
        pytest.skip("needs the reference build (oracle/_ref)")
    ref = oracle_lib.get("reference")
    X, y = ref.generate_trunk(6000, 24, 7)
    gpu_ctx.upload(X, y, 2)
    kw = dict(n_trees=5, mode=mode, breakeven=breakeven, seed=11, max_depth=max_depth, n_workers=4)
    g = gpu_ctx.train_forest(sofg.TrainConfig(instrument=True, **kw))
    ins = g.instrumentation
    assert ins is not None
    nodes, samples = ref.train_forest_depths(X, y, 2, oracle_lib.make_config(**kw))
    assert ins.nodes == nodes
    assert ins.samples == samples
    assert sum(ins.nodes) == len(g.left)
    # a depth's seconds are its waves' device time; the deepest depths hold only leaves (no wave)
    assert ins.seconds[0] > 0 and all(s >= 0 for s in ins.seconds)
    split_total = sum(sum(b.values()) for b in ins.phases)
    assert abs(split_total - ins.split_seconds) < 1e-9 + 1e-6 * split_total
    assert ins.split_seconds <= ins.total_seconds
    for b in ins.phases:
        assert all(v >= 0 for v in b.values())
    # histogram time only where histogram nodes exist
    if mode == "exact":
        assert all(b["build_histograms"] == 0 for b in ins.phases)
    else:
        assert ins.phases[0]["build_histograms"] > 0
