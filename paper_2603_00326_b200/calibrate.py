"""B200 crossover calibration for the dynamic split switch.

The reference calibrates `breakeven` on the CPU by timing exact vs histogram splits of one
synthetic node (calibrate.hpp:51-112, 135-196) and stores it in `Forest::breakeven`
(forest.hpp:80, 285-293). On the GPU the split methods run as batched waves, so the per-node
crossover is not what matters: the breakeven that minimises whole-forest training time is. This
calibrates that directly — train the same forest with each candidate threshold on the resident
table, time it on the device, return the fastest. The chosen value is a model parameter: pass the
same breakeven to the CPU reference for parity runs (exact and histogram give different trees).
"""
from __future__ import annotations

import time
from dataclasses import replace

__all__ = ["calibrate_breakeven"]

DEFAULT_CANDIDATES = (256, 512, 768, 1024, 1536, 2048)


def calibrate_breakeven(ctx, cfg, candidates=DEFAULT_CANDIDATES, trees: int = 20, repeats: int = 1):
    """Returns (best_breakeven, {candidate: seconds}) for `ctx`'s resident dataset.

    cfg: a TrainConfig (seed, bins, ...); its mode is forced to dynamic and n_trees/tree range to
    `trees` trees. Each candidate is timed `repeats` times after one warm-up run (device-synchronised
    wall clock around train_forest, which synchronises its own stream)."""
    import torch

    times = {}
    base = replace(cfg, mode="dynamic", n_trees=trees, tree_begin=0, tree_end=trees)
    ctx.train_forest(replace(base, breakeven=int(candidates[0])))  # warm-up (allocations)
    for be in candidates:
        best = float("inf")
        for _ in range(repeats):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ctx.train_forest(replace(base, breakeven=int(be)))
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        times[int(be)] = best
    return min(times, key=times.get), times
