"""More than 8 classes (wide.cu; the reference bounds class_count only by its label table,
dataset.hpp:36-44): whole forests against the reference build in all three modes, with
multi-chunk histogram nodes, device-sorted exact nodes, ties, predict and train_tree."""
import numpy as np
import pytest

import oracle_lib
from test_gpu_parity import _cfg, _forest_equal

pytestmark = pytest.mark.gpu


def _data(n, d, k, seed, quantize=False):
    rng = np.random.default_rng(seed)
    y = (rng.integers(0, k, n)).astype(np.int32)
    X = (rng.standard_normal((d, n)) + 0.8 * (y[None, :] % d == np.arange(d)[:, None])).astype(np.float32)
    if quantize:
        X = (np.round(X * 4) / 4).astype(np.float32)
    return X, y


@pytest.mark.parametrize("k", [9, 23, 64])
@pytest.mark.parametrize("mode,breakeven", [("dynamic", 400), ("histogram", None), ("exact", None)])
def test_wide_class_forest(gpu_ctx, oracle, k, mode, breakeven):
    X, y = _data(5000, 12, k, k)
    gpu_ctx.upload(X, y, k)
    gc, oc = _cfg(n_trees=3, mode=mode, breakeven=breakeven, seed=k + 1)
    g = gpu_ctx.train_forest(gc)
    o = oracle.train_forest(X, y, k, oc)
    assert _forest_equal(g, o) == []


def test_wide_class_multichunk_and_ties(gpu_ctx, oracle):
    # root nodes above 65535 samples: histogram counting in several chunks merged in global counters
    X, y = _data(110000, 6, 12, 5, quantize=True)
    gpu_ctx.upload(X, y, 12)
    gc, oc = _cfg(n_trees=2, mode="dynamic", breakeven=3000, seed=9, max_depth=6)
    assert _forest_equal(gpu_ctx.train_forest(gc), oracle.train_forest(X, y, 12, oc)) == []


def test_wide_class_bins_and_predict(gpu_ctx, oracle):
    X, y = _data(6000, 10, 17, 3)
    gpu_ctx.upload(X, y, 17)
    gc, oc = _cfg(n_trees=4, mode="dynamic", breakeven=300, seed=4, bin_count=1024)
    Xt, _ = _data(3000, 10, 17, 99)
    rows = np.ascontiguousarray(Xt.T)
    g = gpu_ctx.train_forest(gc)
    o, (olab, ovotes) = oracle.train_forest(X, y, 17, oc, predict_rows=rows)
    assert _forest_equal(g, o) == []
    lab, votes = gpu_ctx.predict(g, rows)
    assert np.array_equal(lab, olab)
    assert np.array_equal(votes, ovotes)


def test_wide_class_train_tree(gpu_ctx, oracle):
    X, y = _data(2500, 8, 30, 8)
    gpu_ctx.upload(X, y, 30)
    gc, oc = _cfg(n_trees=1, mode="dynamic", breakeven=200, seed=13)
    ts = oracle.derive_seed(13, 1)
    boot = oracle.bootstrap(2500, 0.632, oracle.derive_seed(ts, 0))
    t = gpu_ctx.train_tree(boot, gc, oracle.derive_seed(ts, 1))
    o = oracle.train_tree(X, y, 30, boot, oc, oracle.derive_seed(ts, 1))
    assert _forest_equal(t, o) == []


def test_class_count_limit(gpu_ctx):
    X, y = _data(100, 4, 65, 1)
    with pytest.raises(Exception):
        gpu_ctx.upload(X, y, 65)
