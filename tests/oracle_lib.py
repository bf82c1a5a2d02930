"""ctypes view of the CPU oracle (test infrastructure only).

Two builds share oracle/oracle_capi.h:
  * "port"      oracle/liboracle_port.so         — C++ restatement of the reference algorithm
  * "reference" oracle/_ref/libsoforest_ref.so   — the reference headers compiled as-is

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE = os.path.join(ROOT, "oracle")


class OrcConfig(C.Structure):
    _fields_ = [
        ("n_trees", C.c_uint64),
        ("mode", C.c_int32),
        ("two_level_binning", C.c_int32),
        ("bin_count", C.c_uint64),
        ("has_breakeven", C.c_int32),
        ("has_max_depth", C.c_int32),
        ("breakeven", C.c_uint64),
        ("max_depth", C.c_uint64),
        ("bootstrap_fraction", C.c_double),
        ("min_samples_split", C.c_uint64),
        ("max_split_retries", C.c_uint64),
        ("n_workers", C.c_uint64),
        ("seed", C.c_uint64),
        ("num_projections", C.c_uint64),
        ("cell_density", C.c_double),
    ]


class OrcSplit(C.Structure):
    _fields_ = [
        ("found", C.c_int32),
        ("projection_index", C.c_int32),
        ("threshold", C.c_float),
        ("n_left", C.c_uint32),
        ("n_right", C.c_uint32),
        ("_pad", C.c_uint32),
        ("gain", C.c_double),
    ]


MODES = {"exact": 0, "histogram": 1, "dynamic": 2}


def make_config(n_trees=100, mode="dynamic", bin_count=256, breakeven=None, bootstrap_fraction=0.632,
                max_depth=None, min_samples_split=2, max_split_retries=1, n_workers=1, seed=0,
                two_level_binning=True, num_projections=0, cell_density=0.0) -> OrcConfig:
    c = OrcConfig()
    c.n_trees = n_trees
    c.mode = MODES[mode] if isinstance(mode, str) else int(mode)
    c.two_level_binning = int(bool(two_level_binning))
    c.bin_count = bin_count
    c.has_breakeven = int(breakeven is not None)
    c.breakeven = breakeven or 0
    c.has_max_depth = int(max_depth is not None)
    c.max_depth = max_depth or 0
    c.bootstrap_fraction = bootstrap_fraction
    c.min_samples_split = min_samples_split
    c.max_split_retries = max_split_retries
    c.n_workers = n_workers
    c.seed = seed
    c.num_projections = num_projections
    c.cell_density = cell_density
    return c


@dataclass
class FlatForest:
    """Forest as flat arrays; identical layout for oracle and GPU exports."""

    tree_off: np.ndarray
    left: np.ndarray
    right: np.ndarray
    pred: np.ndarray
    thr: np.ndarray
    term_off: np.ndarray
    feat: np.ndarray
    weight: np.ndarray
    breakeven: int = 0

    @property
    def n_trees(self) -> int:
        return len(self.tree_off) - 1

    def head(self, m: int) -> "FlatForest":
        """The first m trees."""
        e = int(self.tree_off[m])
        q = int(self.term_off[e])
        return FlatForest(self.tree_off[:m + 1].copy(), self.left[:e], self.right[:e], self.pred[:e], self.thr[:e],
                          self.term_off[:e + 1].copy(), self.feat[:q], self.weight[:q], self.breakeven)

    @staticmethod
    def concat(parts: "list[FlatForest]") -> "FlatForest":
        to, so = [np.zeros(1, np.int64)], [np.zeros(1, np.int64)]
        nb = qb = 0
        for p in parts:
            to.append(p.tree_off[1:] + nb)
            so.append(p.term_off[1:] + qb)
            nb += len(p.left)
            qb += len(p.feat)
        cat = lambda name: np.concatenate([getattr(p, name) for p in parts])
        return FlatForest(np.concatenate(to), cat("left"), cat("right"), cat("pred"), cat("thr"), np.concatenate(so),
                          cat("feat"), cat("weight"), parts[0].breakeven if parts else 0)

    def tree(self, t: int) -> "FlatForest":
        a, b = int(self.tree_off[t]), int(self.tree_off[t + 1])
        ta, tb = int(self.term_off[a]), int(self.term_off[b])
        return FlatForest(np.array([0, b - a], np.int64), self.left[a:b], self.right[a:b], self.pred[a:b],
                          self.thr[a:b], self.term_off[a:b + 1] - ta, self.feat[ta:tb], self.weight[ta:tb])

    def tree_equal(self, other: "FlatForest", t: int, u: int | None = None) -> bool:
        """Tree::operator== (forest.hpp:67-71): every node field, thresholds bitwise."""
        x, y = self.tree(t), other.tree(t if u is None else u)
        return (len(x.left) == len(y.left)
                and np.array_equal(x.left, y.left) and np.array_equal(x.right, y.right)
                and np.array_equal(x.pred, y.pred)
                and np.array_equal(x.thr.view(np.uint32), y.thr.view(np.uint32))
                and np.array_equal(x.term_off, y.term_off) and np.array_equal(x.feat, y.feat)
                and np.array_equal(x.weight.view(np.uint32), y.weight.view(np.uint32)))


class Oracle:
    def __init__(self, kind: str = "port"):
        if kind == "port":
            path = os.path.join(ORACLE, "liboracle_port.so")
        elif kind == "reference":
            path = os.path.join(ORACLE, "_ref", "libsoforest_ref.so")
            if not _cpu_has_avx512():
                path = os.path.join(ORACLE, "_ref", "libsoforest_ref_v3.so")
        else:
            raise ValueError(kind)
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run make -C oracle)")
        self.kind = kind
        self.lib = L = C.CDLL(path)
        p = C.POINTER
        u64, i64, i32, u32, f32, f64 = C.c_uint64, C.c_int64, C.c_int32, C.c_uint32, C.c_float, C.c_double
        vp = C.c_void_p
        L.orc_last_error.restype = C.c_char_p
        L.orc_impl_name.restype = C.c_char_p
        L.orc_train_forest.argtypes = [vp, vp, u64, u64, i32, p(OrcConfig), p(vp)]
        L.orc_dataset_create.argtypes = [vp, vp, u64, u64, i32, p(vp)]
        L.orc_dataset_free.argtypes = [vp]
        L.orc_train_forest_ds.argtypes = [vp, p(OrcConfig), p(vp)]
        L.orc_train_tree.argtypes = [vp, vp, u64, u64, i32, vp, u64, p(OrcConfig), u64, u64, p(vp)]
        L.orc_forest_import.argtypes = [u64, u64, i32] + [vp] * 9
        L.orc_train_tree_ds.argtypes = [vp, vp, u64, p(OrcConfig), u64, u64, p(vp)]
        for fn in ("orc_forest_num_trees", "orc_forest_num_nodes", "orc_forest_num_terms", "orc_forest_breakeven"):
            getattr(L, fn).restype = u64
            getattr(L, fn).argtypes = [vp]
        L.orc_forest_export.argtypes = [vp] * 9
        L.orc_forest_free.argtypes = [vp]
        L.orc_predict.argtypes = [vp, vp, u64, u64, vp, vp]
        L.orc_split_mix64.restype = u64
        L.orc_split_mix64.argtypes = [u64]
        L.orc_derive_seed.restype = u64
        L.orc_derive_seed.argtypes = [u64, u64]
        L.orc_rng_outputs.argtypes = [u64, u64, u64, vp]
        L.orc_generate_trunk.argtypes = [u64, u64, u64, vp, vp]
        L.orc_bootstrap.restype = u64
        L.orc_bootstrap.argtypes = [u64, f64, u64, vp]
        L.orc_projection_config.argtypes = [u64, p(u64), p(u64), p(f64)]
        L.orc_sample_projection.restype = i64
        L.orc_sample_projection.argtypes = [u64, u64, f64, u64, u64, vp, vp, vp, u64, p(u64)]
        L.orc_binomial_draw.restype = u64
        L.orc_binomial_draw.argtypes = [u64, f64, u64, u64, p(u64)]
        L.orc_apply_projection.argtypes = [vp, u64, vp, vp, u64, vp, u64, vp]
        L.orc_sample_boundaries.restype = u64
        L.orc_sample_boundaries.argtypes = [vp, u64, u64, u64, u64, vp, p(u64)]
        L.orc_build_histogram.argtypes = [vp, vp, u64, vp, u64, i32, vp]
        L.orc_entropy.restype = f64
        L.orc_entropy.argtypes = [vp, i32]
        L.orc_best_split_exact.restype = OrcSplit
        L.orc_best_split_exact.argtypes = [vp, vp, u64, i32]
        L.orc_best_split_histogram.restype = OrcSplit
        L.orc_best_split_histogram.argtypes = [vp, u64, vp, i32]
        if kind == "reference":
            L.orc_train_save_model.argtypes = [vp, vp, u64, u64, i32, p(OrcConfig), C.c_char_p]
            L.orc_load_model_summary.argtypes = [C.c_char_p, p(u64), p(u64)]
            L.orc_csv_number.restype = u64
            L.orc_csv_number.argtypes = [C.c_double, C.c_char_p, u64]
            L.orc_train_forest_depths.argtypes = [vp, vp, u64, u64, i32, p(OrcConfig), vp, vp, u64, p(u64)]
            L.orc_load_model_calibration.argtypes = [C.c_char_p, p(u64), p(i32), p(u64), p(u64), p(i32)]
        L.orc_find_node_split.restype = OrcSplit
        L.orc_find_node_split.argtypes = [vp, vp, u64, i32, vp, u64, vp, u64, vp, vp, i32, u64, u64, u64,
                                          p(u64), vp]

    # -- helpers -----------------------------------------------------------------------------
    def _err(self, rc: int, what: str):
        if rc != 0:
            msg = self.lib.orc_last_error().decode()
            if msg.startswith("invalid_argument"):
                raise ValueError(f"{what}: {msg}")
            if msg.startswith("out_of_range"):
                raise IndexError(f"{what}: {msg}")
            raise RuntimeError(f"{what}: {msg}")

    def _export(self, h) -> FlatForest:
        L = self.lib
        T, N, Q = L.orc_forest_num_trees(h), L.orc_forest_num_nodes(h), L.orc_forest_num_terms(h)
        f = FlatForest(np.zeros(T + 1, np.int64), np.zeros(N, np.int32), np.zeros(N, np.int32),
                       np.zeros(N, np.int32), np.zeros(N, np.float32), np.zeros(N + 1, np.int64),
                       np.zeros(Q, np.uint32), np.zeros(Q, np.float32), int(L.orc_forest_breakeven(h)))
        L.orc_forest_export(h, *(a.ctypes.data for a in (f.tree_off, f.left, f.right, f.pred, f.thr,
                                                          f.term_off, f.feat, f.weight)))
        return f

    # -- training ----------------------------------------------------------------------------
    def train_forest(self, X: np.ndarray, y: np.ndarray, k: int, cfg: OrcConfig, predict_rows=None):
        X = np.ascontiguousarray(X, np.float32)  # [d][n]
        y = np.ascontiguousarray(y, np.int32)
        d, n = X.shape
        h = C.c_void_p()
        self._err(self.lib.orc_train_forest(X.ctypes.data, y.ctypes.data, n, d, k, C.byref(cfg), C.byref(h)),
                  "train_forest")
        try:
            f = self._export(h)
            if predict_rows is not None:
                return f, self._predict(h, predict_rows, d, k)
            return f
        finally:
            self.lib.orc_forest_free(h)

    def dataset(self, X: np.ndarray, y: np.ndarray, k: int):
        """Converts the table once into the implementation's own dataset type."""
        X = np.ascontiguousarray(X, np.float32)
        y = np.ascontiguousarray(y, np.int32)
        d, n = X.shape
        h = C.c_void_p()
        self._err(self.lib.orc_dataset_create(X.ctypes.data, y.ctypes.data, n, d, k, C.byref(h)), "dataset")
        return h

    def dataset_free(self, h):
        self.lib.orc_dataset_free(h)

    def train_forest_ds(self, ds, cfg: OrcConfig, predict_rows=None, d=None, k=2, timing=None):
        import time as _time

        h = C.c_void_p()
        t0 = _time.perf_counter()
        self._err(self.lib.orc_train_forest_ds(ds, C.byref(cfg), C.byref(h)), "train_forest")
        if timing is not None:
            timing["train_s"] = _time.perf_counter() - t0
        try:
            f = self._export(h)
            if predict_rows is not None:
                return f, self._predict(h, predict_rows, d, k)
            return f
        finally:
            self.lib.orc_forest_free(h)

    def train_tree(self, X, y, k, active, cfg, seed, depth=0) -> FlatForest:
        X = np.ascontiguousarray(X, np.float32)
        y = np.ascontiguousarray(y, np.int32)
        a = np.ascontiguousarray(active, np.uint32)
        d, n = X.shape
        h = C.c_void_p()
        self._err(self.lib.orc_train_tree(X.ctypes.data, y.ctypes.data, n, d, k, a.ctypes.data, len(a),
                                          C.byref(cfg), seed, depth, C.byref(h)), "train_tree")
        try:
            return self._export(h)
        finally:
            self.lib.orc_forest_free(h)

    def train_tree_ds(self, ds, active, cfg, seed, depth=0) -> FlatForest:
        """train_tree on a dataset handle (dataset()); releases the GIL, so threads run in parallel."""
        a = np.ascontiguousarray(active, np.uint32)
        h = C.c_void_p()
        self._err(self.lib.orc_train_tree_ds(ds, a.ctypes.data, len(a), C.byref(cfg), seed, depth, C.byref(h)),
                  "train_tree")
        try:
            return self._export(h)
        finally:
            self.lib.orc_forest_free(h)

    def predict_flat(self, f: FlatForest, rows, d, k):
        """predict (forest.hpp:110-121) with this oracle on a flat forest (e.g. assembled trees)."""
        h = C.c_void_p()
        arrs = [np.ascontiguousarray(a) for a in (f.tree_off, f.left, f.right, f.pred, f.thr, f.term_off, f.feat,
                                                  f.weight)]
        self._err(self.lib.orc_forest_import(f.n_trees, d, k, *(a.ctypes.data for a in arrs), C.byref(h)),
                  "forest_import")
        try:
            return self._predict(h, rows, d, k)
        finally:
            self.lib.orc_forest_free(h)

    def _predict(self, h, rows, d, k):
        rows = np.ascontiguousarray(rows, np.float32)
        out = np.zeros(rows.shape[0], np.int32)
        votes = np.zeros((rows.shape[0], k), np.float64)
        self._err(self.lib.orc_predict(h, rows.ctypes.data, rows.shape[0], d, out.ctypes.data, votes.ctypes.data),
                  "predict")
        return out, votes

    # -- model I/O (reference build) ---------------------------------------------------------
    def train_save_model(self, X, y, k, cfg, path: str):
        X = np.ascontiguousarray(X, np.float32)
        y = np.ascontiguousarray(y, np.int32)
        d, n = X.shape
        self._err(self.lib.orc_train_save_model(X.ctypes.data, y.ctypes.data, n, d, k, C.byref(cfg),
                                                path.encode()), "train_save_model")

    def load_model_summary(self, path: str):
        t, nn = C.c_uint64(), C.c_uint64()
        self._err(self.lib.orc_load_model_summary(path.encode(), C.byref(t), C.byref(nn)), "load_model")
        return t.value, nn.value

    def csv_number(self, v: float) -> str:
        buf = C.create_string_buffer(64)
        self.lib.orc_csv_number(float(v), buf, 64)
        return buf.value.decode()

    def train_forest_depths(self, X: np.ndarray, y: np.ndarray, k: int, cfg: OrcConfig):
        """TrainInstrumentation::by_depth (nodes, samples) of the reference's train_forest."""
        X = np.ascontiguousarray(X, np.float32)
        y = np.ascontiguousarray(y, np.int32)
        d, n = X.shape
        cap = 4096
        nodes, samples, nd = np.zeros(cap, np.uint64), np.zeros(cap, np.uint64), C.c_uint64()
        self._err(self.lib.orc_train_forest_depths(X.ctypes.data, y.ctypes.data, n, d, k, C.byref(cfg),
                                                   nodes.ctypes.data, samples.ctypes.data, cap, C.byref(nd)),
                  "train_forest_depths")
        return [int(v) for v in nodes[:nd.value]], [int(v) for v in samples[:nd.value]]

    def load_model_calibration(self, path: str):
        """(forest.breakeven, has_calibration, calibration.breakeven, n_samples, fallback) as the
        reference's load_model reads them."""
        be, hc, cb, ns, fb = C.c_uint64(), C.c_int32(), C.c_uint64(), C.c_uint64(), C.c_int32()
        self._err(self.lib.orc_load_model_calibration(path.encode(), C.byref(be), C.byref(hc), C.byref(cb),
                                                      C.byref(ns), C.byref(fb)), "load_model")
        return be.value, bool(hc.value), cb.value, ns.value, bool(fb.value)

    # -- primitives --------------------------------------------------------------------------
    def split_mix64(self, x):
        return self.lib.orc_split_mix64(x)

    def derive_seed(self, s, k):
        return self.lib.orc_derive_seed(s, k)

    def rng_outputs(self, seed, skip, count):
        out = np.zeros(count, np.uint64)
        self.lib.orc_rng_outputs(seed, skip, count, out.ctypes.data)
        return out

    def generate_trunk(self, n, d, seed):
        X = np.zeros((d, n), np.float32)
        y = np.zeros(n, np.int32)
        self._err(self.lib.orc_generate_trunk(n, d, seed, X.ctypes.data, y.ctypes.data), "generate_trunk")
        return X, y

    def bootstrap(self, n, fraction, seed):
        out = np.zeros(n, np.uint32)
        m = self.lib.orc_bootstrap(n, fraction, seed, out.ctypes.data)
        return out[:m]

    def projection_config(self, d):
        R, e, dens = C.c_uint64(), C.c_uint64(), C.c_double()
        self.lib.orc_projection_config(d, C.byref(R), C.byref(e), C.byref(dens))
        return R.value, e.value, dens.value

    def sample_projection(self, d, R, density, seed, skip=0, cap=1 << 16):
        row_ptr = np.zeros(R + 1, np.uint32)
        feat = np.zeros(cap, np.uint32)
        w = np.zeros(cap, np.float32)
        used = C.c_uint64()
        nnz = self.lib.orc_sample_projection(d, R, density, seed, skip, row_ptr.ctypes.data, feat.ctypes.data,
                                             w.ctypes.data, cap, C.byref(used))
        assert nnz >= 0
        return row_ptr, feat[:nnz].copy(), w[:nnz].copy(), used.value

    def binomial_draw(self, cells, density, seed, skip=0):
        used = C.c_uint64()
        z = self.lib.orc_binomial_draw(cells, density, seed, skip, C.byref(used))
        return z, used.value

    def apply_projection(self, X, feat, weight, active):
        X = np.ascontiguousarray(X, np.float32)
        feat = np.ascontiguousarray(feat, np.uint32)
        weight = np.ascontiguousarray(weight, np.float32)
        active = np.ascontiguousarray(active, np.uint32)
        out = np.zeros(len(active), np.float32)
        self.lib.orc_apply_projection(X.ctypes.data, X.shape[1], feat.ctypes.data, weight.ctypes.data, len(feat),
                                      active.ctypes.data, len(active), out.ctypes.data)
        return out

    def sample_boundaries(self, values, bin_count, seed, skip=0):
        v = np.ascontiguousarray(values, np.float32)
        out = np.zeros(max(bin_count - 1, 1), np.float32)
        used = C.c_uint64()
        nb = self.lib.orc_sample_boundaries(v.ctypes.data, len(v), bin_count, seed, skip, out.ctypes.data,
                                            C.byref(used))
        return out[:nb].copy(), used.value

    def build_histogram(self, values, labels, boundaries, k):
        v = np.ascontiguousarray(values, np.float32)
        y = np.ascontiguousarray(labels, np.int32)
        b = np.ascontiguousarray(boundaries, np.float32)
        counts = np.zeros((len(b) + 1) * k, np.uint32)
        self.lib.orc_build_histogram(v.ctypes.data, y.ctypes.data, len(v), b.ctypes.data, len(b), k,
                                     counts.ctypes.data)
        return counts

    def entropy(self, counts):
        c = np.ascontiguousarray(counts, np.uint32)
        return self.lib.orc_entropy(c.ctypes.data, len(c))

    def best_split_exact(self, values, labels, k):
        v = np.ascontiguousarray(values, np.float32)
        y = np.ascontiguousarray(labels, np.int32)
        return self.lib.orc_best_split_exact(v.ctypes.data, y.ctypes.data, len(v), k)

    def best_split_histogram(self, boundaries, counts, k):
        b = np.ascontiguousarray(boundaries, np.float32)
        c = np.ascontiguousarray(counts, np.uint32)
        return self.lib.orc_best_split_histogram(b.ctypes.data, len(b), c.ctypes.data, k)

    def find_node_split(self, X, y, k, active, row_ptr, feat, weight, method, bin_count, seed, skip=0):
        X = np.ascontiguousarray(X, np.float32)
        y = np.ascontiguousarray(y, np.int32)
        a = np.ascontiguousarray(active, np.uint32)
        rp = np.ascontiguousarray(row_ptr, np.uint32)
        f = np.ascontiguousarray(feat, np.uint32)
        w = np.ascontiguousarray(weight, np.float32)
        used = C.c_uint64()
        vals = np.zeros(len(a), np.float32)
        s = self.lib.orc_find_node_split(X.ctypes.data, y.ctypes.data, X.shape[1], k, a.ctypes.data, len(a),
                                         rp.ctypes.data, len(rp) - 1, f.ctypes.data, w.ctypes.data,
                                         MODES[method] if isinstance(method, str) else method, bin_count, seed,
                                         skip, C.byref(used), vals.ctypes.data)
        return s, used.value, vals


def _cpu_has_avx512() -> bool:
    try:
        with open("/proc/cpuinfo") as fh:
            flags = fh.read()
        return all(f in flags for f in ("avx512f", "avx512bw", "avx512vl", "avx512dq"))
    except OSError:
        return False


_cache: dict[str, Oracle] = {}


def get(kind: str = "port") -> Oracle:
    if kind not in _cache:
        _cache[kind] = Oracle(kind)
    return _cache[kind]


def have_reference() -> bool:
    return os.path.exists(os.path.join(ORACLE, "_ref", "libsoforest_ref.so"))
