"""Tree-wise sharding of a forest across GPUs.

Tree t of a forest is a pure function of (data, cfg, t) (reference forest.hpp:264-266, tested by
forest_test.cpp:172-204), so a forest shards into independent tree ranges with no collective on
the data path. Each rank (one process per GPU under torchrun, or one host thread per GPU context
in a single process) trains the contiguous block ``shard_range(n_trees, rank, world)`` through
``TrainConfig.tree_begin/tree_end``; the blocks are gathered on the host afterwards and
concatenated in tree order, which reproduces the single-device forest exactly.
"""
from __future__ import annotations

import threading
from typing import Callable, Sequence

import numpy as np

__all__ = ["shard_range", "concat_forests", "train_forest_distributed", "train_forest_devices"]


def shard_range(n_trees: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous balanced block of trees for `rank` (the first n_trees % world ranks get one more)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    base, extra = divmod(n_trees, world)
    b = rank * base + min(rank, extra)
    return b, b + base + (1 if rank < extra else 0)


def concat_forests(parts: Sequence):
    """Concatenates flat forests (tree order = list order). Works for any object with the flat
    forest fields (paper_2603_00326_b200.Forest, tests' oracle FlatForest)."""
    parts = [p for p in parts if p is not None]
    if not parts:
        raise ValueError("no forests to concatenate")
    node_base = np.cumsum([0] + [len(p.left) for p in parts])
    term_base = np.cumsum([0] + [len(p.feat) for p in parts])
    tree_off = [np.zeros(1, np.int64)] + [p.tree_off[1:] + node_base[i] for i, p in enumerate(parts)]
    term_off = [np.zeros(1, np.int64)] + [p.term_off[1:] + term_base[i] for i, p in enumerate(parts)]
    out = type(parts[0]).__new__(type(parts[0]))
    fields = dict(tree_off=np.concatenate(tree_off).astype(np.int64),
                  term_off=np.concatenate(term_off).astype(np.int64))
    for k in ("left", "right", "pred", "thr", "feat", "weight"):
        fields[k] = np.concatenate([getattr(p, k) for p in parts])
    for k, v in vars(parts[0]).items():
        if k not in fields:
            fields[k] = v
    out.__dict__.update(fields)
    return out


def train_forest_distributed(train_range: Callable[[int, int], object], n_trees: int, group=None):
    """Each rank of the torch.distributed group trains its block through ``train_range(begin, end)``
    (e.g. ``lambda b, e: ctx.train_forest(replace(cfg, tree_begin=b, tree_end=e))``); the blocks are
    gathered host-side with ``all_gather_object`` (gloo or nccl — the gather is off the hot path)
    and every rank returns the whole forest in tree order."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    b, e = shard_range(n_trees, rank, world)
    mine = train_range(b, e) if e > b else None
    parts = [None] * world
    dist.all_gather_object(parts, mine, group=group)
    return concat_forests(parts)


def train_forest_devices(contexts: Sequence, cfg, n_trees: int | None = None):
    """Single-process multi-GPU train_forest: one host thread per device context (the C ABI's
    contexts are independent, one host thread each), trees sharded in contiguous blocks — the
    analogue of the reference's worker threads (parallel.hpp:15-40) with GPUs as workers."""
    from dataclasses import replace

    n = cfg.n_trees if n_trees is None else n_trees
    parts = [None] * len(contexts)
    errors = []

    def run(i):
        try:
            b, e = shard_range(n, i, len(contexts))
            if e > b:
                parts[i] = contexts[i].train_forest(replace(cfg, n_trees=n, tree_begin=b, tree_end=e))
        except BaseException as ex:  # rethrow the first failure, like parallel_for (parallel.hpp:26-39)
            errors.append(ex)

    threads = [threading.Thread(target=run, args=(i,)) for i in range(len(contexts))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    return concat_forests(parts)
