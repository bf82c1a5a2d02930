"""The C-ABI boundary (include/sofg.h) without a GPU: the library loads, exports every declared
entry point, carries sm_100a code, and fails loudly (no CPU fallback) when no device is usable."""
from __future__ import annotations

import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sofg.h")


def declared_functions() -> list[str]:
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(sofg_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    import paper_2603_00326_b200 as sofg

    return sofg.load()


def test_header_declares_the_drop_in_surface():
    names = declared_functions()
    for must in ("sofg_create", "sofg_destroy", "sofg_upload_dataset", "sofg_train_forest", "sofg_train_tree",
                 "sofg_predict", "sofg_find_node_split", "sofg_apply_projection", "sofg_sample_projection",
                 "sofg_forest_export", "sofg_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, f"libsofg.so lacks {missing}"


def test_library_is_sm100a_native():
    import paper_2603_00326_b200 as sofg

    out = subprocess.run(["cuobjdump", "--list-elf", sofg.lib_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out, out[:500]


def test_product_library_does_not_link_the_oracle():
    import paper_2603_00326_b200 as sofg

    syms = subprocess.run(["nm", "-D", sofg.lib_path()], capture_output=True, text=True).stdout
    assert "orc_" not in syms
    deps = subprocess.run(["ldd", sofg.lib_path()], capture_output=True, text=True).stdout
    assert "oracle" not in deps and "soforest_ref" not in deps


def test_default_config_mirrors_reference_train_config(lib):
    import paper_2603_00326_b200 as sofg

    c = sofg._Cfg()
    lib.sofg_default_config(C.byref(c))
    # forest.hpp:38-53 defaults
    assert (c.n_trees, c.mode, c.bin_count, c.min_samples_split, c.max_split_retries, c.seed) == (100, 2, 256, 2, 1, 0)
    assert abs(c.bootstrap_fraction - 0.632) < 1e-15 and c.has_breakeven == 0 and c.has_max_depth == 0
    # calibrate.hpp:22-32 CalibrationOptions defaults
    k = c.calibration
    assert (k.n_min, k.n_max, k.bin_count, k.two_level, k.repetitions, k.seed) == (64, 65536, 256, 1, 5,
                                                                                  0xCA11B8A7E5EED)
    assert k.budget_seconds == 0.1 and c.instrument == 0


def test_no_gpu_fails_loudly(lib):
    """Without a CUDA device every compute entry point must fail (there is no CPU fallback)."""
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("a GPU is visible")
    except Exception:
        pass
    h = C.c_void_p()
    rc = lib.sofg_create(0, C.byref(h))
    assert rc != 0
    msg = lib.sofg_last_error().decode()
    assert msg, "sofg_last_error must describe the failure"
    import paper_2603_00326_b200 as sofg

    with pytest.raises((sofg.SofgError, ValueError)):
        sofg.Context(0)


def test_null_context_is_rejected(lib):
    rc = lib.sofg_train_forest(None, None, None)
    assert rc != 0 and lib.sofg_last_error()
