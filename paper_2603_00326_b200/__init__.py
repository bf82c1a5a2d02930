"""B200-native sparse-oblique split finding for the soforest learner (arXiv 2603.00326).

Python host mirror of the reference's train/predict API (reference
proj/include/soforest/forest.hpp): ``train_forest``, ``train_tree``, ``predict``, plus the
per-function entry points the parity tests use (``find_node_split``, ``sample_projection``,
``apply_projection``). Everything calls ``lib/libsofg.so`` (hand-written sm_100a CUDA behind the
C ABI of ``include/sofg.h``). There is no CPU fallback: if the library or a GPU is missing, calls
raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

__all__ = ["TrainConfig", "Forest", "Context", "lib_path", "load", "SofgError"]

_HERE = os.path.dirname(os.path.abspath(__file__))


def lib_path() -> str:
    return os.path.join(_HERE, "lib", os.environ.get("SOFG_LIB", "libsofg.so"))


class SofgError(RuntimeError):
    pass


class _CalOpts(C.Structure):
    _fields_ = [("n_min", C.c_uint64), ("n_max", C.c_uint64), ("budget_seconds", C.c_double),
                ("bin_count", C.c_uint64), ("two_level", C.c_int32), ("_pad", C.c_int32),
                ("repetitions", C.c_uint64), ("seed", C.c_uint64)]


class _CalSample(C.Structure):
    _fields_ = [("n", C.c_uint64), ("exact_seconds", C.c_double), ("histogram_seconds", C.c_double)]


class _Cal(C.Structure):
    _fields_ = [("breakeven", C.c_uint64), ("elapsed_seconds", C.c_double), ("fallback", C.c_int32),
                ("_pad", C.c_int32), ("n_samples", C.c_uint64), ("samples", _CalSample * 64)]


class _Phases(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("sample_projections", "apply_projections", "build_histograms",
                                          "evaluate_splits")]


class _Cfg(C.Structure):
    _fields_ = [
        ("n_trees", C.c_uint64), ("mode", C.c_int32), ("two_level_binning", C.c_int32),
        ("bin_count", C.c_uint64), ("has_breakeven", C.c_int32), ("has_max_depth", C.c_int32),
        ("breakeven", C.c_uint64), ("max_depth", C.c_uint64), ("bootstrap_fraction", C.c_double),
        ("min_samples_split", C.c_uint64), ("max_split_retries", C.c_uint64),
        ("n_workers", C.c_uint64), ("seed", C.c_uint64), ("num_projections", C.c_uint64),
        ("cell_density", C.c_double), ("batch_trees", C.c_uint64), ("tree_begin", C.c_uint64),
        ("tree_end", C.c_uint64), ("calibration", _CalOpts), ("instrument", C.c_int32), ("_pad2", C.c_int32),
    ]


class _Split(C.Structure):
    _fields_ = [("found", C.c_int32), ("projection_index", C.c_int32), ("threshold", C.c_float),
                ("n_left", C.c_uint32), ("n_right", C.c_uint32), ("n_left_partition", C.c_uint32),
                ("gain", C.c_double), ("consumed", C.c_uint64)]


class _Stats(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("ms_sample", "ms_hist_rng", "ms_hist_count", "ms_exact",
                                           "ms_partition", "ms_waves_total", "ms_host_binomial",
                                           "ms_host_bootstrap", "ms_train_total")] + \
               [(n, C.c_uint64) for n in ("waves", "nodes", "hist_nodes", "exact_nodes", "kernel_launches",
                                           "levels", "hist_count_launches", "exact_launches")] + \
               [(n, C.c_double) for n in ("hist_strict_bytes", "exact_strict_bytes", "hist_sector_bytes",
                                          "exact_sector_bytes", "ms_host_roots", "ms_host_prep", "ms_host_submit",
                                          "ms_host_spec", "ms_host_wait", "ms_host_post", "ms_host_final")] + \
               [(n, C.c_uint64) for n in ("sweep_waves", "gather_waves")] + [("sweep_alg_bytes", C.c_double)] + \
               [("sweep_cta_threads", C.c_uint32), ("sweep_entry_bytes", C.c_uint32)]


_MODES = {"exact": 0, "histogram": 1, "dynamic": 2}
_lib = None


def load():
    """Loads libsofg.so (raises if it is missing — the product path has no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    path = lib_path()
    if not os.path.exists(path):
        raise SofgError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(path)
    vp, u64, i32, f64 = C.c_void_p, C.c_uint64, C.c_int32, C.c_double
    P = C.POINTER
    L.sofg_last_error.restype = C.c_char_p
    L.sofg_version.restype = C.c_char_p
    L.sofg_default_config.argtypes = [P(_Cfg)]
    L.sofg_create.argtypes = [C.c_int, P(vp)]
    L.sofg_destroy.argtypes = [vp]
    L.sofg_upload_dataset.argtypes = [vp, vp, u64, u64, vp, i32]
    L.sofg_upload_columns.argtypes = [vp, vp, u64, u64, vp, i32]
    L.sofg_generate_trunk.argtypes = [vp, u64, u64, i32, u64]
    L.sofg_download_dataset.argtypes = [vp, vp, vp]
    L.sofg_train_forest.argtypes = [vp, P(_Cfg), P(vp)]
    L.sofg_train_tree.argtypes = [vp, vp, u64, P(_Cfg), u64, u64, P(vp)]
    L.sofg_calibrate.argtypes = [vp, P(_Cfg), P(_Cal)]
    L.sofg_forest_calibration.argtypes = [vp, P(_Cal)]
    L.sofg_forest_instrumentation.restype = u64
    L.sofg_forest_instrumentation.argtypes = [vp, vp, vp, vp, u64, P(_Phases), P(f64), P(f64)]
    for fn in ("sofg_forest_num_trees", "sofg_forest_num_nodes", "sofg_forest_num_terms",
               "sofg_forest_breakeven"):
        getattr(L, fn).restype = u64
        getattr(L, fn).argtypes = [vp]
    L.sofg_forest_export.argtypes = [vp] * 9
    L.sofg_forest_arrays.argtypes = [vp, vp]
    L.sofg_forest_import.argtypes = [u64, u64, i32] + [vp] * 8 + [P(vp)]
    L.sofg_forest_free.argtypes = [vp]
    L.sofg_predict.argtypes = [vp, vp, vp, u64, u64, vp, vp]
    L.sofg_apply_projection.argtypes = [vp, vp, vp, u64, vp, u64, vp]
    L.sofg_sample_projection.argtypes = [vp, u64, u64, f64, vp, vp, u64, vp, vp, vp, u64, vp]
    L.sofg_bootstrap_sample.argtypes = [u64, f64, u64, vp, P(u64)]
    L.sofg_find_node_split.argtypes = [vp, vp, u64, vp, u64, vp, vp, i32, u64, u64, u64, P(_Split)]
    L.sofg_stream.restype = vp
    L.sofg_stream.argtypes = [vp]
    L.sofg_host_alloc.restype = vp
    L.sofg_host_alloc.argtypes = [u64]
    L.sofg_host_free.argtypes = [vp]
    L.sofg_set_stats.argtypes = [vp, C.c_int]
    L.sofg_get_stats.argtypes = [vp, P(_Stats)]
    L.sofg_reset_stats.argtypes = [vp]
    L.sofg_stats_kernels.argtypes = [vp]
    L.sofg_stats_kernel.argtypes = [vp, C.c_int, P(C.c_char_p), P(C.c_double), P(u64)]
    _lib = L
    return L


def _check(rc: int, what: str):
    if rc == 0:
        return
    msg = load().sofg_last_error().decode()
    if rc == 1:
        raise ValueError(f"{what}: {msg}")
    if rc == 2:
        raise IndexError(f"{what}: {msg}")
    raise SofgError(f"{what}: {msg}")


@dataclass
class TrainConfig:
    """soforest::TrainConfig (forest.hpp:38-53) plus GPU extensions."""

    n_trees: int = 100
    mode: str = "dynamic"
    bin_count: int = 256
    two_level_binning: bool = True
    breakeven: int | None = None
    bootstrap_fraction: float = 0.632
    max_depth: int | None = None
    min_samples_split: int = 2
    max_split_retries: int = 1
    n_workers: int = 0
    seed: int = 0
    num_projections: int = 0
    cell_density: float = 0.0
    batch_trees: int = 0
    tree_begin: int = 0
    tree_end: int = 0
    calibration: "CalibrationOptions | None" = None  # soforest::CalibrationOptions; None = defaults
    instrument: bool = False  # record soforest::TrainInstrumentation (Forest.instrumentation)

    def to_c(self) -> _Cfg:
        c = _Cfg()
        load().sofg_default_config(C.byref(c))
        c.n_trees = self.n_trees
        c.mode = _MODES[self.mode] if isinstance(self.mode, str) else int(self.mode)
        c.two_level_binning = int(self.two_level_binning)
        c.bin_count = self.bin_count
        c.has_breakeven = int(self.breakeven is not None)
        c.breakeven = self.breakeven or 0
        c.has_max_depth = int(self.max_depth is not None)
        c.max_depth = self.max_depth or 0
        c.bootstrap_fraction = self.bootstrap_fraction
        c.min_samples_split = self.min_samples_split
        c.max_split_retries = self.max_split_retries
        c.n_workers = self.n_workers
        c.seed = self.seed
        c.num_projections = self.num_projections
        c.cell_density = self.cell_density
        c.batch_trees = self.batch_trees
        c.tree_begin = self.tree_begin
        c.tree_end = self.tree_end
        if self.calibration is not None:
            co = self.calibration
            c.calibration.n_min, c.calibration.n_max = co.n_min, co.n_max
            c.calibration.budget_seconds, c.calibration.bin_count = co.budget_seconds, co.bin_count
            c.calibration.two_level, c.calibration.repetitions = int(co.two_level), co.repetitions
            c.calibration.seed = co.seed
        c.instrument = int(self.instrument)
        return c


@dataclass
class Forest:
    """Flat forest; node ids follow the reference's depth-first split order."""

    tree_off: np.ndarray
    left: np.ndarray
    right: np.ndarray
    pred: np.ndarray
    thr: np.ndarray
    term_off: np.ndarray
    feat: np.ndarray
    weight: np.ndarray
    breakeven: int = 0
    class_count: int = 0
    n_features: int = 0
    calibration: "Calibration | None" = None          # Forest::calibration (forest.hpp:81)
    instrumentation: "Instrumentation | None" = None  # TrainInstrumentation of the run

    @property
    def n_trees(self) -> int:
        return len(self.tree_off) - 1

    def tree_nodes(self, t: int) -> int:
        return int(self.tree_off[t + 1] - self.tree_off[t])


def _export(h) -> Forest:
    """Copy of a library forest (the handle stays with the caller)."""
    L = load()
    T, N, Q = L.sofg_forest_num_trees(h), L.sofg_forest_num_nodes(h), L.sofg_forest_num_terms(h)
    f = Forest(np.empty(T + 1, np.int64), np.empty(N, np.int32), np.empty(N, np.int32), np.empty(N, np.int32),
               np.empty(N, np.float32), np.empty(N + 1, np.int64), np.empty(Q, np.uint32), np.empty(Q, np.float32),
               int(L.sofg_forest_breakeven(h)))
    L.sofg_forest_export(h, *(a.ctypes.data for a in (f.tree_off, f.left, f.right, f.pred, f.thr, f.term_off,
                                                       f.feat, f.weight)))
    return f


@dataclass
class Instrumentation:
    """soforest::TrainInstrumentation (timing.hpp:39-79): per-depth device seconds, node and
    sample counts; split phases per depth bucket ("0-4", "5-9", "10-14", "15+")."""

    seconds: list
    nodes: list
    samples: list
    phases: list  # 4 buckets x dict(sample_projections, apply_projections, build_histograms, evaluate_splits)
    split_seconds: float
    total_seconds: float


def _cal_from_c(c: "_Cal"):
    from .model_io import Calibration

    return Calibration(breakeven=int(c.breakeven),
                       samples=[(int(c.samples[i].n), float(c.samples[i].exact_seconds),
                                 float(c.samples[i].histogram_seconds)) for i in range(int(c.n_samples))],
                       elapsed_seconds=float(c.elapsed_seconds), fallback=bool(c.fallback))


def _records(h, f: "Forest") -> "Forest":
    """Attach the calibration record and instrumentation of library forest `h` to `f`."""
    L = load()
    cal = _Cal()
    if L.sofg_forest_calibration(h, C.byref(cal)):
        f.calibration = _cal_from_c(cal)
    nd = L.sofg_forest_instrumentation(h, None, None, None, 0, None, None, None)
    if nd:
        sec, nodes, samp = np.zeros(nd), np.zeros(nd, np.uint64), np.zeros(nd, np.uint64)
        ph = (_Phases * 4)()
        split_s, total_s = C.c_double(), C.c_double()
        L.sofg_forest_instrumentation(h, sec.ctypes.data, nodes.ctypes.data, samp.ctypes.data, nd, ph,
                                      C.byref(split_s), C.byref(total_s))
        f.instrumentation = Instrumentation(
            sec.tolist(), [int(x) for x in nodes], [int(x) for x in samp],
            [{n: getattr(ph[b], n) for n, _ in _Phases._fields_} for b in range(4)], split_s.value, total_s.value)
    return f


class _ForestOwner:
    """Keeps a library forest alive while numpy views of its arrays exist."""

    def __init__(self, h):
        self.h = h

    def __del__(self):
        if self.h:
            try:
                load().sofg_forest_free(self.h)
            except Exception:  # interpreter shutdown
                pass
            self.h = None


def _adopt(h) -> Forest:
    """Zero-copy Forest over the library's arrays; the handle is freed with the last view."""
    L = load()
    T, N, Q = L.sofg_forest_num_trees(h), L.sofg_forest_num_nodes(h), L.sofg_forest_num_terms(h)
    ptrs = (C.c_void_p * 8)()
    L.sofg_forest_arrays(h, ptrs)
    owner = _ForestOwner(h)

    # numpy arrays cannot carry attributes: a subclass holds the owner reference instead
    def own(i, count, ctype, dtype):
        if count == 0 or not ptrs[i]:
            return np.empty(0, dtype)
        a = _Owned(np.ctypeslib.as_array((ctype * count).from_address(ptrs[i])).view(dtype))
        a._owner = owner
        return a

    f = Forest(own(0, T + 1, C.c_int64, np.int64), own(1, N, C.c_int32, np.int32), own(2, N, C.c_int32, np.int32),
               own(3, N, C.c_int32, np.int32), own(4, N, C.c_float, np.float32), own(5, N + 1, C.c_int64, np.int64),
               own(6, Q, C.c_uint32, np.uint32), own(7, Q, C.c_float, np.float32), int(L.sofg_forest_breakeven(h)))
    return f


class _Owned(np.ndarray):
    """ndarray view that keeps its memory owner alive (attribute `_owner`)."""

    def __new__(cls, a):
        return np.asarray(a).view(cls)

    def __array_finalize__(self, obj):
        self._owner = getattr(obj, "_owner", None)


class Context:
    """One GPU with a resident dataset (column-major float32 table + labels)."""

    def __init__(self, device: int = 0):
        self.L = load()
        self.h = C.c_void_p()
        _check(self.L.sofg_create(device, C.byref(self.h)), "sofg_create")
        self.n_samples = 0
        self.n_features = 0
        self.class_count = 0

    def close(self):
        if self.h:
            self.L.sofg_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- dataset ---------------------------------------------------------------------------------
    def upload(self, X: np.ndarray, y: np.ndarray, class_count: int):
        """X column-major [n_features][n_samples] float32 (the reference's column layout)."""
        X = np.ascontiguousarray(X, np.float32)
        y = np.ascontiguousarray(y, np.int32)
        d, n = X.shape
        _check(self.L.sofg_upload_dataset(self.h, X.ctypes.data, n, d, y.ctypes.data, class_count), "upload")
        self.n_samples, self.n_features, self.class_count = n, d, class_count

    def generate_trunk(self, n: int, d: int, class_count: int = 2, seed: int = 1):
        _check(self.L.sofg_generate_trunk(self.h, n, d, class_count, seed), "generate_trunk")
        self.n_samples, self.n_features, self.class_count = n, d, class_count

    def download(self, X: np.ndarray | None = None, y: np.ndarray | None = None):
        _check(self.L.sofg_download_dataset(self.h, X.ctypes.data if X is not None else None,
                                            y.ctypes.data if y is not None else None), "download")

    # -- training --------------------------------------------------------------------------------
    def train_forest(self, cfg: TrainConfig) -> Forest:
        c = cfg.to_c()
        h = C.c_void_p()
        _check(self.L.sofg_train_forest(self.h, C.byref(c), C.byref(h)), "train_forest")
        if os.environ.get("SOFG_COPY_EXPORT"):
            try:
                f = _records(h, _export(h))
            finally:
                self.L.sofg_forest_free(h)
        else:
            f = _records(h, _adopt(h))  # zero-copy; the library forest is freed with the arrays
        f.class_count, f.n_features = self.class_count, self.n_features
        return f

    def calibrate(self, cfg: TrainConfig | None = None):
        """soforest::calibrate_crossover (calibrate.hpp:51-196) with GPU probes on the resident table;
        returns a model_io.Calibration record."""
        c = (cfg or TrainConfig()).to_c()
        out = _Cal()
        _check(self.L.sofg_calibrate(self.h, C.byref(c), C.byref(out)), "calibrate")
        return _cal_from_c(out)

    def train_tree(self, active, cfg: TrainConfig, seed: int, depth: int = 0) -> Forest:
        a = np.ascontiguousarray(active, np.uint32)
        c = cfg.to_c()
        h = C.c_void_p()
        _check(self.L.sofg_train_tree(self.h, a.ctypes.data, len(a), C.byref(c), seed, depth, C.byref(h)),
               "train_tree")
        try:
            f = _records(h, _export(h))
        finally:
            self.L.sofg_forest_free(h)
        f.class_count, f.n_features = self.class_count, self.n_features
        return f

    def predict(self, forest: Forest, rows: np.ndarray):
        rows = np.ascontiguousarray(rows, np.float32)
        n, d = rows.shape
        h = C.c_void_p()
        _check(self.L.sofg_forest_import(forest.n_trees, d, forest.class_count,
                                         *(a.ctypes.data for a in (forest.tree_off, forest.left, forest.right,
                                                                   forest.pred, forest.thr, forest.term_off,
                                                                   forest.feat, forest.weight)), C.byref(h)),
               "forest_import")
        labels = np.zeros(n, np.int32)
        votes = np.zeros((n, forest.class_count), np.float64)
        try:
            _check(self.L.sofg_predict(self.h, h, rows.ctypes.data, n, d, labels.ctypes.data, votes.ctypes.data),
                   "predict")
        finally:
            self.L.sofg_forest_free(h)
        return labels, votes

    # -- per-function entry points ---------------------------------------------------------------
    def apply_projection(self, feat, weight, active):
        feat = np.ascontiguousarray(feat, np.uint32)
        weight = np.ascontiguousarray(weight, np.float32)
        active = np.ascontiguousarray(active, np.uint32)
        out = np.zeros(len(active), np.float32)
        _check(self.L.sofg_apply_projection(self.h, feat.ctypes.data, weight.ctypes.data, len(feat),
                                            active.ctypes.data, len(active), out.ctypes.data), "apply_projection")
        return out

    def sample_projection(self, d, R, density, seeds, skips=None, cap=4096):
        seeds = np.ascontiguousarray(seeds, np.uint64)
        skips = np.zeros_like(seeds) if skips is None else np.ascontiguousarray(skips, np.uint64)
        n = len(seeds)
        row_ptr = np.zeros((n, R + 1), np.uint32)
        feat = np.zeros((n, cap), np.uint32)
        w = np.zeros((n, cap), np.float32)
        used = np.zeros(n, np.uint64)
        _check(self.L.sofg_sample_projection(self.h, d, R, density, seeds.ctypes.data, skips.ctypes.data, n,
                                             row_ptr.ctypes.data, feat.ctypes.data, w.ctypes.data, cap,
                                             used.ctypes.data), "sample_projection")
        return row_ptr, feat, w, used

    def find_node_split(self, active, row_ptr, feat, weight, method, bin_count, seed, skip=0):
        a = np.ascontiguousarray(active, np.uint32)
        rp = np.ascontiguousarray(row_ptr, np.uint32)
        f = np.ascontiguousarray(feat, np.uint32)
        w = np.ascontiguousarray(weight, np.float32)
        s = _Split()
        m = _MODES[method] if isinstance(method, str) else int(method)
        _check(self.L.sofg_find_node_split(self.h, a.ctypes.data, len(a), rp.ctypes.data, len(rp) - 1, f.ctypes.data,
                                           w.ctypes.data, m, bin_count, seed, skip, C.byref(s)), "find_node_split")
        return s

    def stream_ptr(self) -> int:
        return int(self.L.sofg_stream(self.h) or 0)

    def upload_ptr(self, x_ptr: int, y: np.ndarray, n: int, d: int, class_count: int):
        """Upload from a raw (e.g. page-locked) column-major host pointer."""
        y = np.ascontiguousarray(y, np.int32)
        _check(self.L.sofg_upload_dataset(self.h, x_ptr, n, d, y.ctypes.data, class_count), "upload")
        self.n_samples, self.n_features, self.class_count = n, d, class_count

    # -- instrumentation -------------------------------------------------------------------------
    def set_stats(self, mode: int = 1):
        _check(self.L.sofg_set_stats(self.h, mode), "set_stats")

    def reset_stats(self):
        _check(self.L.sofg_reset_stats(self.h), "reset_stats")

    def stats(self) -> dict:
        s = _Stats()
        _check(self.L.sofg_get_stats(self.h, C.byref(s)), "get_stats")
        out = {name: getattr(s, name) for name, _ in _Stats._fields_}
        kern = {}
        for i in range(self.L.sofg_stats_kernels(self.h)):
            nm, ms, la = C.c_char_p(), C.c_double(), C.c_uint64()
            _check(self.L.sofg_stats_kernel(self.h, i, C.byref(nm), C.byref(ms), C.byref(la)), "stats_kernel")
            kern[nm.value.decode()] = {"ms": round(ms.value, 2), "launches": la.value}
        out["kernels"] = kern
        return out


def bootstrap_sample(n: int, fraction: float, seed: int) -> np.ndarray:
    """soforest::bootstrap_sample (dataset.hpp:332-349) -> sorted uint32 row indices. Host-side."""
    L = load()
    out = np.empty(max(int(n), 1), np.uint32)
    cnt = C.c_uint64()
    _check(L.sofg_bootstrap_sample(int(n), float(fraction), int(seed) % 2**64, out.ctypes.data, C.byref(cnt)),
           "bootstrap_sample")
    return out[:cnt.value].copy()


def train_forest(X, y, class_count, cfg: TrainConfig, device: int = 0) -> Forest:
    """soforest::train_forest (forest.hpp:267) on one GPU."""
    with Context(device) as ctx:
        ctx.upload(X, y, class_count)
        return ctx.train_forest(cfg)


def train_tree(X, y, class_count, active, cfg: TrainConfig, seed: int, depth: int = 0, device: int = 0) -> Forest:
    """soforest::train_tree (forest.hpp:250)."""
    with Context(device) as ctx:
        ctx.upload(X, y, class_count)
        return ctx.train_tree(active, cfg, seed, depth)
