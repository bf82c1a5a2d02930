"""The C++ drop-in (include/sofg/soforest_gpu.hpp) on the reference's own types: the test binary
(tests/cpp/dropin_test.cpp, built by `make -C oracle dropin` against the reference headers and
libsofg.so) trains through soforest::gpu::train_forest / train_tree and checks Tree== against
soforest::train_forest / train_tree, soforest::predict and save_model / load_model on the GPU
forest, the reference's exception types and messages, the calibration record and the bench.hpp
profiles (CSV schema through soforest::write_csv)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_test")


@pytest.mark.gpu
def test_cpp_dropin_against_reference(tmp_path):
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/dropin_test not built (needs the reference headers at build time)")
    r = subprocess.run([BIN, str(tmp_path)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all checks passed" in r.stdout
    assert (tmp_path / "dropin_depth_profile.csv").read_text().startswith("depth,mode,seconds,nodes,samples\n")


def test_cpp_dropin_links_the_product_library():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/dropin_test not built")
    deps = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "libsofg.so" in deps and "not found" not in deps
