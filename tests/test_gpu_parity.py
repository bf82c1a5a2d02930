"""GPU parity: every CUDA path against the CPU oracle on identical inputs and seeds.

The oracle is the reference compiled as-is (oracle/_ref) when present, else the restated port;
both are pinned to each other in tests/test_oracle.py. Integer/byte/index results and floats
produced by identical IEEE operation sequences are compared bit-for-bit.
"""
import numpy as np
import pytest

import oracle_lib

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


@pytest.mark.parametrize("d", [4, 8, 64, 512, 4096])
def test_sample_projection_matches_oracle(gpu_ctx, oracle, d):
    R, _, dens = oracle.projection_config(d)
    seeds = np.array([oracle.derive_seed(7, i) for i in range(300)], np.uint64)
    skips = np.array([(i * 13) % 700 for i in range(300)], np.uint64)
    rp, feat, w, used = gpu_ctx.sample_projection(d, R, dens, seeds, skips)
    for i in range(len(seeds)):
        orp, ofeat, ow, oused = oracle.sample_projection(d, R, dens, int(seeds[i]), int(skips[i]))
        assert np.array_equal(rp[i], orp), i
        z = int(orp[-1])
        assert np.array_equal(feat[i, :z], ofeat), i
        assert np.array_equal(_bits(w[i, :z]), _bits(ow)), i
        assert int(used[i]) == oused, i


def test_sample_projection_dense_density(gpu_ctx, oracle):
    # extension knob: denser matrices exercise long Floyd runs and collisions
    d, R = 64, 12
    for dens in (0.05, 0.3, 0.9):
        seeds = np.arange(40, dtype=np.uint64) * 977 + 5
        rp, feat, w, used = gpu_ctx.sample_projection(d, R, dens, seeds, cap=1024)
        for i in range(len(seeds)):
            orp, ofeat, ow, oused = oracle.sample_projection(d, R, dens, int(seeds[i]), 0)
            assert np.array_equal(rp[i], orp)
            z = int(orp[-1])
            assert np.array_equal(feat[i, :z], ofeat)
            assert np.array_equal(_bits(w[i, :z]), _bits(ow))
            assert int(used[i]) == oused


def test_apply_projection_goldens(gpu_ctx):
    # projection_test.cpp:138-156
    X = np.array([[1, 2, 3, 4], [10, 20, 30, 40], [100, 200, 300, 400]], np.float32)
    gpu_ctx.upload(X, np.array([0, 1, 0, 1]), 2)
    out = gpu_ctx.apply_projection([0, 2], [1, -1], [0, 1, 2, 3])
    assert out.tolist() == [-99, -198, -297, -396]
    assert gpu_ctx.apply_projection([0, 2], [1, -1], [3, 1]).tolist() == [-396, -198]
    assert gpu_ctx.apply_projection([], [], [3, 1]).tolist() == [0, 0]
    assert gpu_ctx.apply_projection([1], [-1], [0, 1, 2, 3]).tolist() == [-10, -20, -30, -40]


def test_apply_projection_random(gpu_ctx, oracle):
    rng = np.random.default_rng(3)
    n, d = 5000, 50
    X = (rng.standard_normal((d, n)) * rng.choice([1e-3, 1, 1e3], size=(d, 1))).astype(np.float32)
    gpu_ctx.upload(X, rng.integers(0, 2, n), 2)
    for it in range(30):
        nt = int(rng.integers(0, 8))
        feat = np.sort(rng.choice(d, nt, replace=False)).astype(np.uint32)
        w = rng.choice([-1.0, 1.0], nt).astype(np.float32)
        act = np.sort(rng.choice(n, int(rng.integers(1, n)), replace=False)).astype(np.uint32)
        assert np.array_equal(_bits(gpu_ctx.apply_projection(feat, w, act)),
                              _bits(oracle.apply_projection(X, feat, w, act)))


def _split_eq(g, o):
    assert bool(g.found) == bool(o.found)
    if not o.found:
        return
    assert g.projection_index == o.projection_index
    assert _bits(g.threshold) == _bits(o.threshold)
    assert g.gain == o.gain
    assert g.n_left == o.n_left


@pytest.mark.parametrize("method,bins", [("exact", 256), ("histogram", 1024), ("histogram", 256),
                                         ("histogram", 64), ("histogram", 8)])
def test_find_node_split_trunk400(gpu_ctx, oracle, method, bins):
    # FindNodeSplitTest fixture (split_test.cpp:231-240): generate_trunk(400, 8, 123), all rows
    X, y = oracle.generate_trunk(400, 8, 123)
    gpu_ctx.upload(X, y, 2)
    R, _, dens = oracle.projection_config(8)
    active = np.arange(400, dtype=np.uint32)
    for seed in range(12):
        rp, feat, w, used = oracle.sample_projection(8, R, dens, seed, 0)
        g = gpu_ctx.find_node_split(active, rp, feat, w, method, bins, seed, used)
        o, oused, _ = oracle.find_node_split(X, y, 2, active, rp, feat, w, method, bins, seed, used)
        _split_eq(g, o)
        assert int(g.consumed) == oused


@pytest.mark.parametrize("n,method,bins", [(2, "exact", 256), (3, "exact", 256), (31, "exact", 256),
                                           (32, "exact", 256), (33, "exact", 256), (64, "exact", 256),
                                           (65, "exact", 256), (128, "exact", 256), (255, "exact", 256),
                                           (512, "exact", 256), (700, "exact", 256), (1024, "exact", 256),
                                           (1025, "exact", 256), (2048, "exact", 256),
                                           (300, "histogram", 256), (5000, "histogram", 256),
                                           (20000, "histogram", 256), (9000, "histogram", 32),
                                           (257, "histogram", 256), (3000, "histogram", 1024),
                                           (1500, "histogram", 512), (40, "histogram", 64),
                                           (200, "histogram", 128), (129, "histogram", 128)])
def test_find_node_split_subsets(gpu_ctx, oracle, n, method, bins):
    X, y = oracle.generate_trunk(30000, 16, 5)
    gpu_ctx.upload(X, y, 2)
    R, _, dens = oracle.projection_config(16)
    rng = np.random.default_rng(n)
    for it in range(4):
        active = np.sort(rng.choice(30000, n, replace=False)).astype(np.uint32)
        seed = int(rng.integers(1 << 60))
        rp, feat, w, used = oracle.sample_projection(16, R, dens, seed, 0)
        g = gpu_ctx.find_node_split(active, rp, feat, w, method, bins, seed, used)
        o, oused, vals = oracle.find_node_split(X, y, 2, active, rp, feat, w, method, bins, seed, used)
        _split_eq(g, o)
        assert int(g.consumed) == oused
        if o.found:
            assert g.n_left_partition == int((vals <= o.threshold).sum())


def test_find_node_split_quantized_ties(gpu_ctx, oracle):
    # many equal projected values: grouping, signed zeros, first-max tie breaks
    rng = np.random.default_rng(11)
    n, d = 4000, 6
    X = np.round(rng.standard_normal((d, n)) * 2).astype(np.float32) / 2
    X[0, ::7] = -0.0
    y = rng.integers(0, 3, n).astype(np.int32)
    gpu_ctx.upload(X, y, 3)
    R, _, dens = oracle.projection_config(d)
    for it in range(20):
        m = int(rng.integers(2, 1500))
        active = np.sort(rng.choice(n, m, replace=False)).astype(np.uint32)
        seed = it * 101 + 3
        rp, feat, w, used = oracle.sample_projection(d, R, dens, seed, 0)
        for method in ("exact", "histogram"):
            if method == "exact" and m > 2048:
                continue
            g = gpu_ctx.find_node_split(active, rp, feat, w, method, 64, seed, used)
            o, oused, _ = oracle.find_node_split(X, y, 3, active, rp, feat, w, method, 64, seed, used)
            _split_eq(g, o)


def _cfg(**kw):
    import paper_2603_00326_b200 as sofg

    return sofg.TrainConfig(**kw), oracle_lib.make_config(**{k: v for k, v in kw.items()
                                                             if k not in ("batch_trees", "tree_begin", "tree_end")})


def _forest_equal(g, o, t_g=None):
    ff = oracle_lib.FlatForest(g.tree_off, g.left, g.right, g.pred, g.thr, g.term_off, g.feat, g.weight)
    bad = [t for t in range(o.n_trees) if not ff.tree_equal(o, t)]
    return bad


@pytest.mark.parametrize("mode,breakeven", [("dynamic", 300), ("histogram", None), ("dynamic", 2048)])
def test_train_forest_small(gpu_ctx, oracle, mode, breakeven):
    X, y = oracle.generate_trunk(3000, 10, 21)
    gpu_ctx.upload(X, y, 2)
    gc, oc = _cfg(n_trees=6, mode=mode, breakeven=breakeven, seed=5, n_workers=4)
    g = gpu_ctx.train_forest(gc)
    o = oracle.train_forest(X, y, 2, oc)
    assert g.n_trees == o.n_trees
    assert _forest_equal(g, o) == []
    assert g.breakeven == o.breakeven


def test_train_forest_config1_10k_x_64(gpu_ctx, oracle):
    # BASELINE config 1: 10K x 64, 10 trees to purity (dynamic, fixed breakeven)
    X, y = oracle.generate_trunk(10000, 64, 1)
    gpu_ctx.upload(X, y, 2)
    gc, oc = _cfg(n_trees=10, mode="dynamic", breakeven=1024, seed=7, n_workers=8)
    g = gpu_ctx.train_forest(gc)
    o = oracle.train_forest(X, y, 2, oc)
    assert _forest_equal(g, o) == []


def test_train_tree_matches_forest_stream(gpu_ctx, oracle):
    # forest_test.cpp:172-185: tree t equals train_tree on its derived stream
    X, y = oracle.generate_trunk(600, 6, 13)
    gpu_ctx.upload(X, y, 2)
    gc, oc = _cfg(n_trees=1, mode="dynamic", breakeven=128, seed=77)
    f = gpu_ctx.train_forest(gc)
    ts = oracle.derive_seed(77, 1)
    boot = oracle.bootstrap(600, 0.632, oracle.derive_seed(ts, 0))
    t = gpu_ctx.train_tree(boot, gc, oracle.derive_seed(ts, 1))
    o = oracle.train_tree(X, y, 2, boot, oc, oracle.derive_seed(ts, 1))
    assert _forest_equal(t, o) == []
    assert _forest_equal(f, o) == []


def test_max_depth_and_min_samples(gpu_ctx, oracle):
    X, y = oracle.generate_trunk(2000, 8, 3)
    gpu_ctx.upload(X, y, 2)
    for kw in (dict(max_depth=0), dict(max_depth=3), dict(min_samples_split=50), dict(max_split_retries=0)):
        gc, oc = _cfg(n_trees=3, mode="dynamic", breakeven=200, seed=11, **kw)
        assert _forest_equal(gpu_ctx.train_forest(gc), oracle.train_forest(X, y, 2, oc)) == [], kw


def test_multiclass_forest(gpu_ctx, oracle):
    rng = np.random.default_rng(1)
    n, d, k = 4000, 12, 4
    y = (np.arange(n) % k).astype(np.int32)
    X = (rng.standard_normal((d, n)) + 0.6 * (y[None, :] == (np.arange(d) % k)[:, None])).astype(np.float32)
    gpu_ctx.upload(X, y, k)
    gc, oc = _cfg(n_trees=4, mode="dynamic", breakeven=256, seed=2)
    assert _forest_equal(gpu_ctx.train_forest(gc), oracle.train_forest(X, y, k, oc)) == []


def test_predict_matches_oracle(gpu_ctx, oracle):
    X, y = oracle.generate_trunk(3000, 10, 4)
    Xt, yt = oracle.generate_trunk(500, 10, 99)
    gpu_ctx.upload(X, y, 2)
    gc, oc = _cfg(n_trees=8, mode="dynamic", breakeven=256, seed=1)
    g = gpu_ctx.train_forest(gc)
    o, (olab, ovotes) = oracle.train_forest(X, y, 2, oc, predict_rows=Xt.T.copy())
    lab, votes = gpu_ctx.predict(g, Xt.T.copy())
    assert np.array_equal(lab, olab)
    assert np.array_equal(votes, ovotes)


@pytest.mark.parametrize("batch", [0, 7])
def test_train_forest_two_groups_and_batches(gpu_ctx, oracle, batch):
    """>= 16 trees per batch runs two tree groups concurrently (own streams, shared table);
    batch_trees splits the forest into several batches. Trees must not depend on either."""
    X, y = oracle.generate_trunk(4000, 24, 9)
    gpu_ctx.upload(X, y, 2)
    gc, oc = _cfg(n_trees=21, mode="dynamic", breakeven=256, seed=3, n_workers=4, batch_trees=batch)
    g = gpu_ctx.train_forest(gc)
    o = oracle.train_forest(X, y, 2, oc)
    assert g.n_trees == 21
    assert _forest_equal(g, o) == []


def test_tree_range_shards_concatenate(gpu_ctx, oracle):
    """tree_begin/tree_end blocks (the multi-GPU shards) reproduce the whole forest."""
    from paper_2603_00326_b200.shard import concat_forests, shard_range

    X, y = oracle.generate_trunk(3000, 16, 4)
    gpu_ctx.upload(X, y, 2)
    parts = []
    for r in range(3):
        b, e = shard_range(11, r, 3)
        gc, _ = _cfg(n_trees=11, mode="dynamic", breakeven=300, seed=8, tree_begin=b, tree_end=e)
        parts.append(gpu_ctx.train_forest(gc))
    g = concat_forests(parts)
    _, oc = _cfg(n_trees=11, mode="dynamic", breakeven=300, seed=8)
    assert _forest_equal(g, oracle.train_forest(X, y, 2, oc)) == []


@pytest.mark.parametrize("density,d", [(0.05, 256), (0.6, 64)])
def test_dense_multiclass_forest_config5_style(gpu_ctx, oracle, density, d):
    """BASELINE config 5 in miniature: 4 classes, dense projections (the SURVEY D3 density knob),
    so rows carry many terms (winning rows longer than NodeRes holds inline) and z is large."""
    rng = np.random.default_rng(5)
    n, k = 3000, 4
    y = (np.arange(n) % k).astype(np.int32)
    X = (rng.standard_normal((d, n)) + 0.5 * (y[None, :] == (np.arange(d) % k)[:, None])).astype(np.float32)
    gpu_ctx.upload(X, y, k)
    gc, oc = _cfg(n_trees=3, mode="dynamic", breakeven=400, seed=13, cell_density=density)
    assert _forest_equal(gpu_ctx.train_forest(gc), oracle.train_forest(X, y, k, oc)) == []


def test_wide_table_sweep_u32_terms(gpu_ctx, oracle):
    """d >= 8192 switches the sweep's term lists to 32-bit entries (feature index > 13 bits)."""
    X, y = oracle.generate_trunk(600, 9000, 3)
    gpu_ctx.upload(X, y, 2)
    gc, oc = _cfg(n_trees=2, mode="dynamic", breakeven=128, seed=4)
    assert _forest_equal(gpu_ctx.train_forest(gc), oracle.train_forest(X, y, 2, oc)) == []


def test_sample_projection_very_dense_global_scratch(gpu_ctx, oracle):
    """z ~ 20K cells per matrix: the Floyd cell sets no longer fit in shared memory."""
    d, R, dens = 4096, 96, 0.05
    seeds = np.array([3, 77, 1234], dtype=np.uint64)
    rp, feat, w, used = gpu_ctx.sample_projection(d, R, dens, seeds, cap=24000)
    for i in range(len(seeds)):
        orp, ofeat, ow, oused = oracle.sample_projection(d, R, dens, int(seeds[i]), 0, cap=1 << 16)
        z = int(orp[-1])
        assert z > 16000
        assert np.array_equal(rp[i], orp) and np.array_equal(feat[i, :z], ofeat)
        assert np.array_equal(_bits(w[i, :z]), _bits(ow)) and int(used[i]) == oused


@pytest.mark.parametrize("mode,breakeven", [("exact", None), ("dynamic", 5000)])
def test_exact_large_nodes_segmented_sort(gpu_ctx, oracle, mode, breakeven):
    """Exact splits of nodes above the shared-memory splitter (n > 2048): ExactOnly mode (the
    'sort' arm of BASELINE config 2) and a breakeven above 2048 use the device-wide segmented sort."""
    X, y = oracle.generate_trunk(9000, 20, 6)
    Xq = np.round(X * 8) / 8  # plus heavy ties
    for data in (X, Xq):
        gpu_ctx.upload(data, y, 2)
        gc, oc = _cfg(n_trees=3, mode=mode, breakeven=breakeven, seed=21)
        assert _forest_equal(gpu_ctx.train_forest(gc), oracle.train_forest(data, y, 2, oc)) == []


@pytest.mark.parametrize("with_inf,mode,breakeven", [(False, "dynamic", 300), (True, "dynamic", 300),
                                                     (False, "exact", None), (True, "histogram", None)])
def test_sweep_special_values(gpu_ctx, oracle, with_inf, mode, breakeven):
    """Signed zeros, subnormals and infinities through both projection producers (sweep and
    gather: float -> double widening, FP64 accumulation, one rounding) and both splitters; one
    infinite feature makes projections +-inf (never NaN: a row holds a feature at most once)."""
    X, y = oracle.generate_trunk(3000, 24, 8)
    X = X.copy()
    rng = np.random.default_rng(8)
    m = rng.random(X.shape)
    X[m < 0.05] = 0.0
    X[(m >= 0.05) & (m < 0.1)] = -0.0
    X[(m >= 0.1) & (m < 0.15)] *= np.float32(1e-40)  # subnormal
    X[3, (m[3] > 0.9)] = np.float32(1e-45)  # smallest subnormal
    if with_inf:
        X[5, ::97] = np.inf  # one infinite feature: projections are +-inf, never NaN
    X = X.astype(np.float32)
    gpu_ctx.upload(X, y, 2)
    gc, oc = _cfg(n_trees=3, mode=mode, breakeven=breakeven, seed=17)
    assert _forest_equal(gpu_ctx.train_forest(gc), oracle.train_forest(X, y, 2, oc)) == []


def test_reupload_same_shape_alternating(gpu_ctx, oracle):
    """Back-to-back uploads of different tables of one shape: the row table and label buffers are
    reused, and each upload must have landed before the next training reads it (pageable copies
    run on the legacy stream; the engine stream does not order against it)."""
    X, y = oracle.generate_trunk(6000, 24, 11)
    variants = [X, np.round(X * 4) / 4, -X, X * np.float32(3.0)]
    for rep in range(2):
        for data in variants:
            data = np.ascontiguousarray(data, np.float32)
            gpu_ctx.upload(data, y, 2)
            gc, oc = _cfg(n_trees=3, mode="dynamic", breakeven=400, seed=5 + rep)
            assert _forest_equal(gpu_ctx.train_forest(gc), oracle.train_forest(data, y, 2, oc)) == []


def test_pinned_upload_in_flight(gpu_ctx, oracle):
    """Uploads from page-locked memory (sofg_host_alloc) stay in flight on the engine stream while
    training starts on the host; rewriting the same page-locked buffer between steps must still
    give each step's own trees."""
    import ctypes as C

    X, y = oracle.generate_trunk(8000, 32, 13)
    d, n = X.shape
    L = gpu_ctx.L
    ptr = L.sofg_host_alloc(n * d * 4)
    assert ptr
    try:
        H = np.ctypeslib.as_array((C.c_float * (n * d)).from_address(ptr)).reshape(d, n)
        for rep, data in enumerate((X, -X, np.round(X * 2) / 2)):
            H[...] = data
            gpu_ctx.upload_ptr(ptr, y, n, d, 2)
            gc, oc = _cfg(n_trees=3, mode="dynamic", breakeven=400, seed=31 + rep)
            assert _forest_equal(gpu_ctx.train_forest(gc), oracle.train_forest(H.copy(), y, 2, oc)) == []
    finally:
        L.sofg_host_free(ptr)


def test_two_contexts_pipelined_pinned_uploads(gpu_ctx, oracle):
    """The bench's end-to-end pipeline on small tables: two contexts on one GPU, each table
    uploaded from its own page-locked buffer in several 32 MB slices while the other context
    trains (one slice in flight), or while the other's call waits for its own table (paused), or
    with nothing else running (two in flight); every training must see its own table."""
    import ctypes as C

    import paper_2603_00326_b200 as sofg

    base, y = oracle.generate_trunk(100_000, 256, 23)  # 102 MB: four slices
    d, n = base.shape
    L = gpu_ctx.L
    ptrs = [L.sofg_host_alloc(n * d * 4) for _ in range(2)]
    assert all(ptrs)
    other = sofg.Context(0)
    try:
        H = [np.ctypeslib.as_array((C.c_float * (n * d)).from_address(p)).reshape(d, n) for p in ptrs]
        ctxs = [gpu_ctx, other]
        tables = [base, -base, np.round(base * 2) / 2, base * np.float32(3.0)]
        H[0][...] = tables[0]
        H[1][...] = tables[1]
        ctxs[0].upload_ptr(ptrs[0], y, n, d, 2)
        ctxs[1].upload_ptr(ptrs[1], y, n, d, 2)  # both in flight; context 0's call waits first
        for j, data in enumerate(tables):
            cur = ctxs[j % 2]
            gc, oc = _cfg(n_trees=2, mode="dynamic", breakeven=400, seed=41 + j)
            f = cur.train_forest(gc)  # joins this context's upload
            if j + 2 < len(tables):  # the buffer this step read, refilled for the step after next
                H[j % 2][...] = tables[j + 2]
                cur.upload_ptr(ptrs[j % 2], y, n, d, 2)  # in flight while the other context trains
            assert _forest_equal(f, oracle.train_forest(np.ascontiguousarray(data, np.float32), y, 2, oc)) == [], j
    finally:
        other.close()
        for p in ptrs:
            L.sofg_host_free(p)


def test_dense_projection_collision_resolution(gpu_ctx, oracle):
    """Matrices with thousands of cells (z ~ 10K of 49K cells): Floyd collisions are the rule, and
    are resolved by the parallel fixpoint (smallest index per sorted value, then the J0 + j chain)."""
    X, y = oracle.generate_trunk(2500, 1024, 17)
    gpu_ctx.upload(X, y, 2)
    gc, oc = _cfg(n_trees=2, mode="dynamic", breakeven=300, seed=9, cell_density=0.2)
    assert _forest_equal(gpu_ctx.train_forest(gc), oracle.train_forest(X, y, 2, oc)) == []


def test_train_tree_repeated_active_longer_than_n(gpu_ctx, oracle):
    # train_tree takes any active list (forest.hpp:250-262 checks only empty / out of range):
    # repeated samples, more entries than the dataset has rows (xlogx tables grow with the list)
    X, y = oracle.generate_trunk(700, 6, 17)
    gpu_ctx.upload(X, y, 2)
    rng = np.random.default_rng(5)
    active = np.sort(rng.integers(0, 700, 1900)).astype(np.uint32)
    for mode, breakeven in (("dynamic", 300), ("histogram", None), ("exact", None)):
        gc, oc = _cfg(n_trees=1, mode=mode, breakeven=breakeven, seed=31)
        t = gpu_ctx.train_tree(active, gc, 1234)
        o = oracle.train_tree(X, y, 2, active, oc, 1234)
        assert _forest_equal(t, o) == [], mode
