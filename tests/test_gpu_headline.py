"""GPU parity on the kernel variants and batch shapes the headline bench actually runs.

The small-shape suite (test_gpu_parity.py) trains at most ~20 trees per batch, so the projection
sweep runs its 128-thread variant. The bench trains 100 trees per batch at 1M x 4096, which selects
the 256-thread sweep with two samples per CTA step (sweep.cu: sweep_threads / sweep_k). These tests
train full 100-tree batches and compare every tree with the reference compiled as-is (oracle/_ref):
  * 100 trees at 20K x 64 (16-bit term entries) and 4K x 9000 (32-bit term entries);
  * BASELINE config 2 (100K x 512, 50 trees) in all three split modes at breakeven 512, plus
    identical hold-out labels;
  * BASELINE config 3 (1M x 4096): trees 500, 557 and 599 of the batch [500, 600) — not the first
    batch a context trains — against the reference's train_tree on each tree's derived stream
    (forest_test.cpp:172-185).
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle_lib

pytestmark = pytest.mark.gpu


def _cfg(**kw):
    import paper_2603_00326_b200 as sofg

    ref_kw = {k: v for k, v in kw.items() if k not in ("batch_trees", "tree_begin", "tree_end")}
    return sofg.TrainConfig(**kw), oracle_lib.make_config(**ref_kw)


def _flat(g):
    return oracle_lib.FlatForest(g.tree_off, g.left, g.right, g.pred, g.thr, g.term_off, g.feat, g.weight)


def _bad_trees(g, o):
    ff = _flat(g)
    return [t for t in range(o.n_trees) if not ff.tree_equal(o, t)]


@pytest.mark.parametrize("n,d,entry_bytes", [(20000, 64, 2), (4000, 9000, 4)])
def test_batch100_wide_sweep_variant(gpu_ctx, oracle, n, d, entry_bytes):
    X, y = oracle.generate_trunk(n, d, 3)
    gpu_ctx.upload(X, y, 2)
    gc, oc = _cfg(n_trees=100, mode="dynamic", breakeven=512, seed=7, n_workers=16)
    gpu_ctx.reset_stats()
    g = gpu_ctx.train_forest(gc)
    st = gpu_ctx.stats()
    # the shipped variant: 256-thread CTAs, 16- or 32-bit term entries
    assert st["sweep_waves"] > 0
    assert st["sweep_cta_threads"] == 256
    assert st["sweep_entry_bytes"] == entry_bytes
    o = oracle.train_forest(X, y, 2, oc)
    assert g.n_trees == 100
    assert _bad_trees(g, o) == []


@pytest.mark.parametrize("mode", ["exact", "histogram", "dynamic"])
def test_config2_three_modes(gpu_ctx, oracle, mode):
    """BASELINE config 2: 100K x 512, 2-class, 50 trees; the sort / histogram / dynamic comparison."""
    X, y = oracle.generate_trunk(100_000, 512, 1)
    Xt, yt = oracle.generate_trunk(5_000, 512, 2)
    gpu_ctx.upload(X, y, 2)
    gc, oc = _cfg(n_trees=50, mode=mode, breakeven=512, seed=7, n_workers=16)
    g = gpu_ctx.train_forest(gc)
    rows = np.ascontiguousarray(Xt.T)
    o, (olab, _) = oracle.train_forest(X, y, 2, oc, predict_rows=rows)
    assert _bad_trees(g, o) == []
    lab, _ = gpu_ctx.predict(g, rows)
    assert np.array_equal(lab, olab)
    assert (lab == yt).mean() > 0.8


def test_config3_subset_of_a_later_batch(gpu_ctx, oracle):
    """1M x 4096: the context trains the batch of trees [500, 600) of a 600-tree forest after a
    warm-up batch, and trees 500, 557, 599 must equal the reference's train_tree on their derived
    streams (tree t: seed derive_seed(cfg.seed, t+1), bootstrap derive_seed(ts, 0), root
    derive_seed(ts, 1); forest.hpp:153-154,305)."""
    n, d, seed, be = 1_000_000, 4096, 7, 512
    gpu_ctx.generate_trunk(n, d, 2, seed=1)
    warm, _ = _cfg(n_trees=600, mode="dynamic", breakeven=be, seed=seed, n_workers=16, tree_begin=0, tree_end=100)
    gpu_ctx.train_forest(warm)
    gc, oc = _cfg(n_trees=600, mode="dynamic", breakeven=be, seed=seed, n_workers=16, tree_begin=500, tree_end=600)
    gpu_ctx.reset_stats()
    g = gpu_ctx.train_forest(gc)
    st = gpu_ctx.stats()
    assert g.n_trees == 100
    assert st["sweep_cta_threads"] == 256 and st["sweep_entry_bytes"] == 2
    X = np.empty((d, n), np.float32)
    y = np.empty(n, np.int32)
    gpu_ctx.download(X, y)
    ds = oracle.dataset(X, y, 2)
    del X
    try:
        picks = (500, 557, 599)

        def ref_tree(t):
            ts = oracle.derive_seed(seed, t + 1)
            boot = oracle.bootstrap(n, 0.632, oracle.derive_seed(ts, 0))
            return oracle.train_tree_ds(ds, boot, oc, oracle.derive_seed(ts, 1))

        with ThreadPoolExecutor(len(picks)) as ex:
            refs = list(ex.map(ref_tree, picks))
    finally:
        oracle.dataset_free(ds)
    ff = _flat(g)
    for t, o in zip(picks, refs):
        assert ff.tree_equal(o, t - 500, 0), t
