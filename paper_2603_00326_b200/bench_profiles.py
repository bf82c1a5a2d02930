"""The reference's profiling harness (proj/include/soforest/bench.hpp:53-153) on the GPU trainer.

Same rows and the same CSV files as bench_depth_profile / bench_phase_profile /
bench_mode_comparison + write_csv, so tools that read the reference's CSVs read these unchanged.
Depth seconds and phase seconds are device times of the level-wise waves (CUDA events; see
Forest.instrumentation); node and sample counts per depth equal the reference's for the same trees.
The C++ counterpart on the reference's own types is soforest::gpu::bench_* in
include/sofg/soforest_gpu.hpp.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, replace
from decimal import Decimal

__all__ = ["DepthProfileRow", "PhaseProfileRow", "ModeComparisonRow", "bench_depth_profile",
           "bench_phase_profile", "bench_mode_comparison", "write_csv", "csv_number"]

_DEPTH_BUCKETS = ("0-4", "5-9", "10-14", "15+")  # timing.hpp:50-56
_PHASES = ("sample_projections", "apply_projections", "build_histograms", "evaluate_splits")


@dataclass
class DepthProfileRow:  # bench.hpp:14-20
    depth: int
    mode: str
    seconds: float
    nodes: int
    samples: int


@dataclass
class PhaseProfileRow:  # bench.hpp:22-26
    phase: str
    depth_bucket: str
    seconds: float


@dataclass
class ModeComparisonRow:  # bench.hpp:28-32
    mode: str
    seconds: float
    normalized: float


def _resolved(ctx, base):
    """bench.hpp:45-51: Dynamic runs of one harness call share one calibration."""
    if base.breakeven is None:
        return replace(base, breakeven=ctx.calibrate(base).breakeven)
    return base


def bench_depth_profile(ctx, base) -> list[DepthProfileRow]:
    """bench.hpp:53-72 on the resident dataset of `ctx`."""
    cfg = _resolved(ctx, base)
    rows = []
    for mode in ("exact", "histogram", "dynamic"):
        ins = ctx.train_forest(replace(cfg, mode=mode, instrument=True)).instrumentation
        for d, (s, n, m) in enumerate(zip(ins.seconds, ins.nodes, ins.samples)):
            rows.append(DepthProfileRow(d, mode, s, n, m))
    return rows


def bench_phase_profile(ctx, base) -> list[PhaseProfileRow]:
    """bench.hpp:74-93."""
    ins = ctx.train_forest(replace(_resolved(ctx, base), instrument=True)).instrumentation
    return [PhaseProfileRow(p, _DEPTH_BUCKETS[b], ins.phases[b][p]) for b in range(4) for p in _PHASES]


def bench_mode_comparison(ctx, base) -> list[ModeComparisonRow]:
    """bench.hpp:95-123 (wall clock of each whole training call)."""
    cfg = _resolved(ctx, base)
    runs = (("exact", "exact", True), ("histogram", "histogram", True), ("dynamic_scalar", "dynamic", False),
            ("dynamic_two_level", "dynamic", True))
    rows = []
    for name, mode, two_level in runs:
        t0 = time.perf_counter()
        ctx.train_forest(replace(cfg, mode=mode, two_level_binning=two_level))
        rows.append(ModeComparisonRow(name, time.perf_counter() - t0, 0.0))
    for r in rows:
        r.normalized = r.seconds / rows[0].seconds
    return rows


def csv_number(v: float) -> str:
    """std::to_chars(double) (bench.hpp:36-40): the shortest round-trip digits, printed in fixed or
    scientific notation (printf %f / %e style, exponent of at least two digits), whichever is
    shorter, fixed on a tie."""
    v = float(v)
    if v != v:
        return "nan" if str(v)[0] != "-" else "-nan"
    if v in (float("inf"), float("-inf")):
        return "inf" if v > 0 else "-inf"
    if v == 0.0:
        return "-0" if str(v).startswith("-") else "0"
    sign, digits, exp = Decimal(repr(v)).normalize().as_tuple()
    ds = "".join(map(str, digits))
    e10 = exp + len(ds) - 1  # decimal exponent of the leading digit
    neg = "-" if sign else ""
    # fixed
    if exp >= 0:
        fixed = ds + "0" * exp
    elif -exp < len(ds):
        fixed = ds[:exp] + "." + ds[exp:]
    else:
        fixed = "0." + "0" * (-exp - len(ds)) + ds
    # scientific
    mant = ds[0] + ("." + ds[1:] if len(ds) > 1 else "")
    sci = f"{mant}e{'-' if e10 < 0 else '+'}{abs(e10):02d}"
    return neg + (fixed if len(fixed) <= len(sci) else sci)


def write_csv(rows, out, kind=None) -> None:
    """bench.hpp:126-153: header line, then one line per row (`out` is a text stream; `kind` names
    the row type when `rows` is empty)."""
    kind = kind or (type(rows[0]) if rows else None)
    if kind is DepthProfileRow:
        out.write("depth,mode,seconds,nodes,samples\n")
        for r in rows:
            out.write(f"{r.depth},{r.mode},{csv_number(r.seconds)},{r.nodes},{r.samples}\n")
    elif kind is PhaseProfileRow:
        out.write("phase,depth_bucket,seconds\n")
        for r in rows:
            out.write(f"{r.phase},{r.depth_bucket},{csv_number(r.seconds)}\n")
    elif kind is ModeComparisonRow:
        out.write("mode,seconds,normalized\n")
        for r in rows:
            out.write(f"{r.mode},{csv_number(r.seconds)},{csv_number(r.normalized)}\n")
    else:
        raise TypeError("write_csv needs DepthProfileRow, PhaseProfileRow or ModeComparisonRow rows")
