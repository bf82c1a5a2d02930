"""Loader for tests/golden/reference_goldens.{npz,txt} (made by tests/golden/make_golden.py from the
reference build). Test infrastructure only."""
from __future__ import annotations

import hashlib
import os
from dataclasses import dataclass

import numpy as np

import oracle_lib

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
_npz = None


def arrays():
    global _npz
    if _npz is None:
        _npz = dict(np.load(os.path.join(HERE, "reference_goldens.npz")))
    return _npz


@dataclass
class ForestCase:
    name: str
    n: int
    d: int
    data_seed: int
    n_trees: int
    mode: str
    breakeven: int | None
    seed: int
    bins: int
    sha_x: str
    sha_y: str

    def forest(self) -> oracle_lib.FlatForest:
        a = arrays()
        return oracle_lib.FlatForest(*(a[f"{self.name}_{k}"] for k in ("tree_off", "left", "right", "pred", "thr",
                                                                      "term_off", "feat", "weight")))

    def pred_labels(self):
        return arrays()[f"{self.name}_pred_labels"]

    def data(self, orc):
        """(X, y, X_holdout) regenerated with the oracle's generate_trunk, verified by checksum."""
        X, y = orc.generate_trunk(self.n, self.d, self.data_seed)
        assert hashlib.sha256(X.tobytes()).hexdigest() == self.sha_x, "generate_trunk drifted from the reference"
        assert hashlib.sha256(y.tobytes()).hexdigest() == self.sha_y
        Xh, _ = orc.generate_trunk(500, self.d, self.data_seed + 100)
        return X, y, Xh

    def config(self, **kw):
        return dict(n_trees=self.n_trees, mode=self.mode, breakeven=self.breakeven, seed=self.seed,
                    bin_count=self.bins, **kw)


def _lines(prefix: str):
    with open(os.path.join(HERE, "reference_goldens.txt")) as fh:
        for ln in fh:
            if ln.startswith("#") or not ln.strip():
                continue
            if prefix is None or ln.startswith(prefix):
                yield ln.split()


def forest_cases() -> list[ForestCase]:
    out = []
    for p in _lines(None):
        if p[0] in ("proj", "bnd"):
            continue
        be = int(p[6])
        out.append(ForestCase(p[0], int(p[1]), int(p[2]), int(p[3]), int(p[4]), p[5], None if be < 0 else be,
                              int(p[7]), int(p[8]), p[9], p[10]))
    return out


def projection_cases():
    """(d, seed, consumed, row_ptr, feat, weight)"""
    a = arrays()
    for p in _lines("proj "):
        d, seed, used = int(p[1]), int(p[2]), int(p[3])
        yield d, seed, used, a[f"proj_{d}_{seed}_row_ptr"], a[f"proj_{d}_{seed}_feat"], a[f"proj_{d}_{seed}_weight"]


def boundary_cases():
    """(values, bins, seed, consumed, boundaries)"""
    a = arrays()
    for p in _lines("bnd "):
        i, bins, seed, used = int(p[1]), int(p[3]), int(p[4]), int(p[5])
        yield a[f"bnd_{i}_values"], bins, seed, used, a[f"bnd_{i}_out"]
