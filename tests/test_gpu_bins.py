"""Histograms of more than 1024 bins (the reference takes any bin_count, histogram.hpp:37-61):
boundaries by the CTA sampler (k_hist_boundaries_cta), counts by wide.cu; forests and single
splits against the reference build."""
import numpy as np
import pytest

from test_gpu_parity import _cfg, _forest_equal, _split_eq

pytestmark = pytest.mark.gpu


def _data(n, d, k, seed):
    rng = np.random.default_rng(seed)
    y = rng.integers(0, k, n).astype(np.int32)
    X = (rng.standard_normal((d, n)) + 0.7 * (y[None, :] % d == np.arange(d)[:, None])).astype(np.float32)
    return X, y


@pytest.mark.parametrize("bins", [1500, 2048, 4096, 8192])
@pytest.mark.parametrize("k", [2, 5, 12])
def test_large_bin_forest(gpu_ctx, oracle, bins, k):
    X, y = _data(20000, 10, k, bins + k)
    gpu_ctx.upload(X, y, k)
    if 12 * bins + 2 * bins * k + 8 * k + 8 > 226 * 1024:  # wide.cu's shared-memory counters
        import paper_2603_00326_b200 as sofg
        with pytest.raises(ValueError):
            gpu_ctx.train_forest(sofg.TrainConfig(n_trees=1, bin_count=bins))
        return
    for mode, breakeven in (("histogram", None), ("dynamic", 600)):
        gc, oc = _cfg(n_trees=2, mode=mode, breakeven=breakeven, seed=3, bin_count=bins, max_depth=8)
        assert _forest_equal(gpu_ctx.train_forest(gc), oracle.train_forest(X, y, k, oc)) == [], (mode, bins, k)


@pytest.mark.parametrize("bins", [2048, 4096, 8192])
def test_large_bin_find_node_split(gpu_ctx, oracle, bins):
    X, y = _data(9000, 12, 3, bins)
    gpu_ctx.upload(X, y, 3)
    rng = np.random.default_rng(bins)
    for m in (3000, 6000, 9000):  # more, about as many and fewer samples than bins
        active = np.sort(rng.choice(9000, m, replace=False)).astype(np.uint32)
        seed = int(rng.integers(1, 1 << 62))
        rp, feat, w, used = oracle.sample_projection(12, 6, 0.3, seed, 0)
        g = gpu_ctx.find_node_split(active, rp, feat, w, "histogram", bins, seed, used)
        o, oused, _ = oracle.find_node_split(X, y, 3, active, rp, feat, w, "histogram", bins, seed, used)
        _split_eq(g, o)
        assert int(g.consumed) == oused


def test_bin_count_limits(gpu_ctx):
    X, y = _data(100, 4, 2, 1)
    gpu_ctx.upload(X, y, 2)
    import paper_2603_00326_b200 as sofg
    with pytest.raises(Exception):
        gpu_ctx.train_forest(sofg.TrainConfig(n_trees=1, bin_count=8193))
