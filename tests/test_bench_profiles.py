"""bench.hpp CSV schema (bench.hpp:36-40,126-153): the Python harness writes the reference's
headers and numbers formatted exactly as std::to_chars (checked against the reference build)."""
import io

import numpy as np
import pytest

import oracle_lib
from paper_2603_00326_b200 import bench_profiles as bp


@pytest.mark.skipif(not oracle_lib.have_reference(), reason="needs the reference build (oracle/_ref)")
def test_csv_number_matches_std_to_chars():
    ref = oracle_lib.get("reference")
    rng = np.random.default_rng(5)
    vals = [0.0, -0.0, 1.0, 0.5, 0.1, 2.0 / 3.0, 1e-5, 1.5e-5, 123456789.0, 1e15, 1e16, 1e22, 1.25e21, 5e-324,
            1.7976931348623157e308, 100.0, 1000000.0, 1e7, 0.001, 0.0001, 12345.678, -3.25, 1e100, 2.5e-8,
            float("inf"), float("-inf")]
    vals += list(rng.standard_normal(300) * 10.0 ** rng.integers(-12, 12, 300))
    vals += list(rng.integers(0, 10**9, 100).astype(float))
    for v in vals:
        assert bp.csv_number(v) == ref.csv_number(v), v


def test_write_csv_headers_and_rows():
    s = io.StringIO()
    bp.write_csv([bp.DepthProfileRow(0, "exact", 0.25, 1, 632)], s)
    assert s.getvalue() == "depth,mode,seconds,nodes,samples\n0,exact,0.25,1,632\n"
    s = io.StringIO()
    bp.write_csv([bp.PhaseProfileRow("sample_projections", "0-4", 1e-5)], s)
    assert s.getvalue() == "phase,depth_bucket,seconds\nsample_projections,0-4,1e-05\n"
    s = io.StringIO()
    bp.write_csv([bp.ModeComparisonRow("exact", 2.0, 1.0)], s)
    assert s.getvalue() == "mode,seconds,normalized\nexact,2,1\n"
    s = io.StringIO()
    bp.write_csv([], s, kind=bp.PhaseProfileRow)
    assert s.getvalue() == "phase,depth_bucket,seconds\n"


@pytest.mark.gpu
def test_gpu_depth_profile_rows_match_reference(gpu_ctx):
    import paper_2603_00326_b200 as sofg

    if not oracle_lib.have_reference():
        pytest.skip("needs the reference build (oracle/_ref)")
    ref = oracle_lib.get("reference")
    X, y = ref.generate_trunk(4000, 16, 9)
    gpu_ctx.upload(X, y, 2)
    base = sofg.TrainConfig(n_trees=3, mode="dynamic", breakeven=300, seed=2, n_workers=4)
    rows = bp.bench_depth_profile(gpu_ctx, base)
    for mode in ("exact", "histogram", "dynamic"):
        nodes, samples = ref.train_forest_depths(X, y, 2, oracle_lib.make_config(
            n_trees=3, mode=mode, breakeven=300, seed=2, n_workers=4))
        mine = [r for r in rows if r.mode == mode]
        assert [r.depth for r in mine] == list(range(len(nodes)))
        assert [r.nodes for r in mine] == nodes and [r.samples for r in mine] == samples
    phases = bp.bench_phase_profile(gpu_ctx, base)
    assert [(r.phase, r.depth_bucket) for r in phases[:4]] == [
        ("sample_projections", "0-4"), ("apply_projections", "0-4"), ("build_histograms", "0-4"),
        ("evaluate_splits", "0-4")]
    assert len(phases) == 16 and all(r.seconds >= 0 for r in phases)
    modes = bp.bench_mode_comparison(gpu_ctx, base)
    assert [m.mode for m in modes] == ["exact", "histogram", "dynamic_scalar", "dynamic_two_level"]
    assert modes[0].normalized == 1.0
