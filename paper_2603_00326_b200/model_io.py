"""Model files in the reference's format (reference model_io.hpp:124-283), so GPU-trained forests drop
into the reference CLI / load_model unchanged.

File: magic "soforest" (8 bytes), u32 version 1, payload, u32 CRC-32 (zlib) of the payload.
Payload (little-endian): u8 sizeof(T)=4; u32 n_features; i32 class_count; u32 #labels + strings
(u32 length + bytes); the TrainConfig (model_io.hpp:133-155, including CalibrationOptions with the
reference defaults, calibrate.hpp:22-32); u64 forest.breakeven; u8 has_calibration (+ record);
u64 #trees; per tree u64 #nodes; per node u32 #terms, (u32 feature, f32 weight)*, f32 threshold,
i32 left, i32 right, i32 predicted_class.

`save_model(forest, cfg, path)` writes byte-identical files to the reference's save_model for the
same trees and config (tested against the reference build, tests/test_model_io.py).
"""
from __future__ import annotations

import struct
import zlib
from dataclasses import dataclass, field

import numpy as np

__all__ = ["save_model", "load_model", "model_bytes", "CalibrationOptions"]

MAGIC = b"soforest"
VERSION = 1
_MODES = {"exact": 0, "histogram": 1, "dynamic": 2}
_MODE_NAMES = {v: k for k, v in _MODES.items()}


@dataclass
class CalibrationOptions:
    """soforest::CalibrationOptions (calibrate.hpp:22-32) with the reference defaults."""

    n_min: int = 64
    n_max: int = 65536
    budget_seconds: float = 0.1
    bin_count: int = 256
    two_level: bool = True
    repetitions: int = 5
    seed: int = 0xCA11B8A7E5EED


@dataclass
class Calibration:
    """soforest::CrossoverCalibration (calibrate.hpp:34-41)."""

    breakeven: int = 1024
    elapsed_seconds: float = 0.0
    fallback: bool = False
    samples: list = field(default_factory=list)  # (n, exact_seconds, histogram_seconds)


def _mode_id(mode) -> int:
    return _MODES[mode] if isinstance(mode, str) else int(mode)


def model_bytes(forest, cfg, label_names=None, calibration_options: CalibrationOptions | None = None,
                calibration: Calibration | None = None, breakeven: int | None = None) -> bytes:
    """The complete file contents save_model would write (model_io.hpp:124-184)."""
    k = int(forest.class_count)
    names = [str(c) for c in range(k)] if label_names is None else list(label_names)
    co = calibration_options or getattr(cfg, "calibration", None) or CalibrationOptions()
    if calibration is None:
        calibration = getattr(forest, "calibration", None)  # Forest::calibration of a calibrated run
    out = bytearray()
    out += struct.pack("<BIi", 4, int(forest.n_features), k)
    out += struct.pack("<I", len(names))
    for nm in names:
        b = nm.encode()
        out += struct.pack("<I", len(b)) + b
    be = cfg.breakeven
    md = cfg.max_depth
    out += struct.pack("<QBQBBQd", int(cfg.n_trees), _mode_id(cfg.mode), int(cfg.bin_count),
                       1 if cfg.two_level_binning else 0, 1 if be is not None else 0,
                       int(be) if be is not None else 0, float(cfg.bootstrap_fraction))
    out += struct.pack("<BQQQQQ", 1 if md is not None else 0, int(md) if md is not None else 0,
                       int(cfg.min_samples_split), int(cfg.max_split_retries), int(cfg.n_workers),
                       int(cfg.seed) % 2**64)
    out += struct.pack("<QQdQBQQ", co.n_min, co.n_max, co.budget_seconds, co.bin_count,
                       1 if co.two_level else 0, co.repetitions, co.seed)
    fb = int(forest.breakeven if breakeven is None else breakeven)
    out += struct.pack("<Q", fb)
    if calibration is None:
        out += b"\x00"
    else:
        out += struct.pack("<BQdBQ", 1, calibration.breakeven, calibration.elapsed_seconds,
                           1 if calibration.fallback else 0, len(calibration.samples))
        for n, e, h in calibration.samples:
            out += struct.pack("<Qdd", n, e, h)
    n_trees = len(forest.tree_off) - 1
    out += struct.pack("<Q", n_trees)
    tree_off = np.asarray(forest.tree_off, np.int64)
    term_off = np.asarray(forest.term_off, np.int64)
    feat = np.asarray(forest.feat, np.uint32)
    weight = np.asarray(forest.weight, np.float32)
    left = np.asarray(forest.left, np.int32)
    right = np.asarray(forest.right, np.int32)
    pred = np.asarray(forest.pred, np.int32)
    thr = np.asarray(forest.thr, np.float32)
    # vectorised node records: u32 nterms | (u32 feat, f32 weight)* | f32 thr | i32 l | i32 r | i32 p
    for t in range(n_trees):
        a, b = int(tree_off[t]), int(tree_off[t + 1])
        out += struct.pack("<Q", b - a)
        nt = (term_off[a + 1:b + 1] - term_off[a:b]).astype(np.uint32)
        rec_len = 4 + 8 * nt.astype(np.int64) + 16
        buf = np.zeros(int(rec_len.sum()), np.uint8)
        pos = np.concatenate([[0], np.cumsum(rec_len)[:-1]])
        view32 = buf.view(np.uint32) if len(buf) % 4 == 0 else None
        assert view32 is not None
        w32 = view32
        p4 = pos // 4
        w32[p4] = nt
        # terms
        ta, tb = int(term_off[a]), int(term_off[b])
        if tb > ta:
            node_of_term = np.repeat(np.arange(b - a), nt)
            local = np.arange(tb - ta) - (term_off[a:b] - ta)[node_of_term]
            tpos = p4[node_of_term] + 1 + 2 * local
            w32[tpos] = feat[ta:tb]
            w32[tpos + 1] = weight[ta:tb].view(np.uint32)
        tail = p4 + 1 + 2 * nt.astype(np.int64)
        w32[tail] = thr[a:b].view(np.uint32)
        w32[tail + 1] = left[a:b].view(np.uint32)
        w32[tail + 2] = right[a:b].view(np.uint32)
        w32[tail + 3] = pred[a:b].view(np.uint32)
        out += buf.tobytes()
    payload = bytes(out)
    crc = zlib.crc32(payload) & 0xFFFFFFFF
    return MAGIC + struct.pack("<I", VERSION) + payload + struct.pack("<I", crc)


def save_model(forest, cfg, path: str, **kw) -> None:
    """soforest::save_model (model_io.hpp:124-184) for a flat forest trained with `cfg`."""
    data = model_bytes(forest, cfg, **kw)
    with open(path, "wb") as fh:
        fh.write(data)


class _Reader:
    def __init__(self, b: bytes):
        self.b, self.p = b, 0

    def take(self, fmt: str):
        n = struct.calcsize(fmt)
        if self.p + n > len(self.b):
            raise RuntimeError("model file truncated")
        v = struct.unpack_from(fmt, self.b, self.p)
        self.p += n
        return v if len(v) > 1 else v[0]

    def str(self) -> str:
        n = self.take("<I")
        if self.p + n > len(self.b):
            raise RuntimeError("model file truncated")
        s = self.b[self.p:self.p + n].decode()
        self.p += n
        return s


def load_model(path: str):
    """soforest::load_model<float> (model_io.hpp:186-283) with the same validation.
    Returns (Forest, TrainConfig, label_names)."""
    from . import Forest, TrainConfig

    with open(path, "rb") as fh:
        data = fh.read()
    if len(data) < 16 or data[:8] != MAGIC:
        raise RuntimeError(f"{path}: not a forest model file")
    (version,) = struct.unpack_from("<I", data, 8)
    if version != VERSION:
        raise RuntimeError(f"{path}: unsupported model format version {version}")
    payload = data[12:-4]
    (crc,) = struct.unpack_from("<I", data, len(data) - 4)
    if zlib.crc32(payload) & 0xFFFFFFFF != crc:
        raise RuntimeError(f"{path}: model file corrupted (checksum mismatch)")
    r = _Reader(payload)
    if r.take("<B") != 4:
        raise RuntimeError(f"{path}: model stores non-float values")
    n_features = r.take("<I")
    k = r.take("<i")
    if k < 2:
        raise RuntimeError(f"{path}: invalid class count")
    names = [r.str() for _ in range(r.take("<I"))]
    if len(names) != k:
        raise RuntimeError(f"{path}: label name count mismatch")
    n_trees, mode, bins, two_level, has_be, be, frac = r.take("<QBQBBQd")
    if mode > 2:
        raise RuntimeError(f"{path}: invalid split mode")
    has_md, md, mss, retries, workers, seed = r.take("<BQQQQQ")
    co = CalibrationOptions(*r.take("<QQdQBQQ"))
    co.two_level = bool(co.two_level)
    breakeven = r.take("<Q")
    calibration = None
    if r.take("<B"):
        cb, ce, cf = r.take("<QdB")
        calibration = Calibration(cb, ce, bool(cf), [r.take("<Qdd") for _ in range(r.take("<Q"))])
    cfg = TrainConfig(calibration=co, n_trees=n_trees, mode=_MODE_NAMES[mode], bin_count=bins, two_level_binning=bool(two_level),
                      breakeven=be if has_be else None, bootstrap_fraction=frac,
                      max_depth=md if has_md else None, min_samples_split=mss, max_split_retries=retries,
                      n_workers=workers, seed=seed)
    tree_off, term_off = [0], [0]
    left, right, pred, thr, feat, weight = [], [], [], [], [], []
    for _ in range(r.take("<Q")):
        nn = r.take("<Q")
        if nn == 0:
            raise RuntimeError(f"{path}: empty tree")
        for _ in range(nn):
            nt = r.take("<I")
            for _ in range(nt):
                f, w = r.take("<If")
                if f >= n_features:
                    raise RuntimeError(f"{path}: projection feature out of range")
                feat.append(f)
                weight.append(w)
            t, lft, rgt, pc = r.take("<fiii")
            if lft < 0:
                if not 0 <= pc < k:
                    raise RuntimeError(f"{path}: leaf class out of range")
            elif lft <= 0 or rgt <= 0 or lft >= nn or rgt >= nn or nt == 0:
                raise RuntimeError(f"{path}: malformed internal node")
            left.append(lft)
            right.append(rgt)
            pred.append(pc)
            thr.append(t)
            term_off.append(len(feat))
        tree_off.append(len(left))
    if r.p != len(payload):
        raise RuntimeError(f"{path}: trailing bytes after model payload")
    f = Forest(np.array(tree_off, np.int64), np.array(left, np.int32), np.array(right, np.int32),
               np.array(pred, np.int32), np.array(thr, np.float32), np.array(term_off, np.int64),
               np.array(feat, np.uint32), np.array(weight, np.float32), breakeven, k, n_features, calibration)
    return f, cfg, names
