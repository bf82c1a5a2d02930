"""Host binomial draw (host_rng.hpp FastBinomial: the reference's std::binomial_distribution
restated with the lgamma pair tabulated) against libstdc++ itself, draw for draw."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_fast_binomial_matches_libstdcxx(tmp_path):
    exe = tmp_path / "binomial_test"
    src = os.path.join(ROOT, "tests", "cpp", "binomial_test.cpp")
    inc = os.path.join(ROOT, "paper_2603_00326_b200", "csrc")
    # the product's host flags (csrc/Makefile HOSTFLAGS): same contraction of the draw's expressions
    subprocess.run(["g++", "-std=c++20", "-O2", "-march=x86-64-v3", "-I", inc, src,
                    os.path.join(inc, "host_rng.cpp"), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe), "20000"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "mismatches: 0" in out.stdout


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_bootstrap_indices_match_std_sample(tmp_path):
    """bootstrap_indices (vectorised mt19937_64 + the selection-sampling restatement) against
    std::sample with std::mt19937_64, the reference's own call (dataset.hpp:332-349)."""
    exe = tmp_path / "bootstrap_test"
    src = os.path.join(ROOT, "tests", "cpp", "bootstrap_test.cpp")
    inc = os.path.join(ROOT, "paper_2603_00326_b200", "csrc")
    subprocess.run(["g++", "-std=c++20", "-O2", "-march=x86-64-v3", "-I", inc, src,
                    os.path.join(inc, "host_rng.cpp"), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "mismatches: 0" in out.stdout
