"""Tree-wise sharding host logic on CPU: world_size 2 over gloo (no GPU).

Each rank trains its block of trees (here with the CPU oracle standing in for a GPU context, via
train_tree on each tree's derived stream exactly as the reference's forest_test.cpp:172-185
does), blocks are gathered with all_gather_object, and the concatenation must equal the
single-process forest tree for tree (the reference's 1-vs-N-worker determinism, acceptance C8).
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_lib
from paper_2603_00326_b200.shard import concat_forests, shard_range, train_forest_distributed

N_TREES = 7


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _train_range(orc, X, y, b, e):
    """Trees [b, e) of the forest: tree t = train_tree(bootstrap(derive_seed(ts,0)), derive_seed(ts,1)),
    ts = derive_seed(cfg.seed, t+1) (forest.hpp:151-157,305)."""
    cfg = oracle_lib.make_config(n_trees=N_TREES, mode="dynamic", breakeven=200, seed=7)
    parts = []
    for t in range(b, e):
        ts = orc.derive_seed(7, t + 1)
        act = orc.bootstrap(X.shape[1], 0.632, orc.derive_seed(ts, 0))
        parts.append(orc.train_tree(X, y, 2, act, cfg, orc.derive_seed(ts, 1)))
    return concat_forests(parts)


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = oracle_lib.get("port")
        X, y = orc.generate_trunk(1500, 12, 3)
        f = train_forest_distributed(lambda b, e: _train_range(orc, X, y, b, e), N_TREES)
        if rank == 0:
            np.savez(out_path, **{k: getattr(f, k) for k in ("tree_off", "left", "right", "pred", "thr",
                                                              "term_off", "feat", "weight")})
    finally:
        dist.destroy_process_group()


def test_shard_range_partitions():
    for n in (0, 1, 7, 100, 801):
        for w in (1, 2, 3, 8):
            rs = [shard_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
            assert max(e - b for b, e in rs) - min(e - b for b, e in rs) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_world2_gloo_sharded_forest_equals_single_process(tmp_path):
    out = str(tmp_path / "f.npz")
    mp.start_processes(_worker, args=(2, _port(), out), nprocs=2, join=True, start_method="spawn")
    got = oracle_lib.FlatForest(**dict(np.load(out)))
    orc = oracle_lib.get("port")
    X, y = orc.generate_trunk(1500, 12, 3)
    want = orc.train_forest(X, y, 2, oracle_lib.make_config(n_trees=N_TREES, mode="dynamic", breakeven=200, seed=7))
    assert got.n_trees == N_TREES
    assert all(got.tree_equal(want, t) for t in range(N_TREES))
