"""Known-answer tests for the CPU oracle (CPU only, no GPU).

Every expected value below is a known answer from the reference's own test-suite
(/root/reference/proj/tests/*_test.cpp, cited per test). They pin the oracle — the checker the
GPU parity tests compare against — to the reference's published behaviour. Both oracle builds are
exercised: "port" (oracle/port, the C++ restatement) and "reference" (oracle/_ref, the reference
headers compiled as-is by oracle/Makefile) when it is present.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

import oracle_lib

KINDS = ["port"] + (["reference"] if oracle_lib.have_reference() else [])


@pytest.fixture(params=KINDS)
def orc(request):
    return oracle_lib.get(request.param)


# random_test.cpp:15-23 — SplitMix64 output function.
def test_split_mix64_known_answers(orc):
    gamma = 0x9E3779B97F4A7C15
    assert orc.split_mix64(1234567) == 6457827717110365317
    assert orc.split_mix64((1234567 + gamma) % 2**64) == 3203168211198807973
    assert orc.split_mix64((1234567 + 2 * gamma) % 2**64) == 9817491932198370423
    assert orc.split_mix64(0) == 0xE220A8397B1DCDAF


# random_test.cpp:25-29 — bijective on a prefix.
def test_split_mix64_bijective_prefix(orc):
    assert len({orc.split_mix64(x) for x in range(2000)}) == 2000


def _mt19937_64(seed: int):
    """Pure-Python std::mt19937_64 ([rand.predef]); yields outputs."""
    M64 = (1 << 64) - 1
    n, m = 312, 156
    mt = [seed & M64]
    for i in range(1, n):
        mt.append((6364136223846793005 * (mt[-1] ^ (mt[-1] >> 62)) + i) & M64)
    idx = n
    while True:
        if idx >= n:
            for i in range(n):
                x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % n] & 0x7FFFFFFF)
                xa = (x >> 1) ^ (0xB5026F5AA96619E9 if x & 1 else 0)
                mt[i] = mt[(i + m) % n] ^ xa
            idx = 0
        y = mt[idx]
        idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        yield y & M64


def test_python_mt19937_64_standard_kat():
    # C++ standard [rand.predef]: the 10000th output of a default-constructed mt19937_64 (seed 5489)
    g = _mt19937_64(5489)
    for _ in range(9999):
        next(g)
    assert next(g) == 9981545732273789042


# random.hpp:10,26 — make_rng(seed) = std::mt19937_64(split_mix64(seed)).
def test_make_rng_stream(orc):
    for seed in (0, 7, 123456789):
        g = _mt19937_64(orc.split_mix64(seed))
        want = [next(g) for _ in range(700)]  # crosses a twist boundary (312)
        assert orc.rng_outputs(seed, 0, 700).tolist() == want
    assert orc.rng_outputs(7, 10, 54).tolist() == orc.rng_outputs(7, 0, 64)[10:].tolist()


# random.hpp:22-24 — derive_seed(seed, key) = split_mix64(seed ^ split_mix64(key + C)).
def test_derive_seed(orc):
    sm = orc.split_mix64
    for s, k in ((0, 0), (7, 1), (7, 2), (2**63 + 5, 99)):
        assert orc.derive_seed(s, k) == sm(s ^ sm((k + 0x632BE59BD9B4E019) % 2**64))


# split_test.cpp:18-29 — entropy known values (bits).
def test_entropy_known_values(orc):
    assert orc.entropy([1, 1]) == 1.0
    assert orc.entropy([5, 0]) == 0.0
    assert orc.entropy([2, 2, 2, 2]) == 2.0
    assert abs(orc.entropy([3, 1]) - 0.811278) < 1e-6


# projection_test.cpp:16-34 — ProjectionConfig::for_features formulas.
def test_projection_config_formulas(orc):
    assert orc.projection_config(100) == (15, 30, 30.0 / 1500.0)
    assert orc.projection_config(4) == (3, 6, 0.5)
    assert orc.projection_config(1) == (2, 3, 1.0)
    # the shapes the bench uses
    assert orc.projection_config(4096)[:2] == (96, 192)
    assert orc.projection_config(512)[:2] == (34, 68)
    assert orc.projection_config(64)[:2] == (12, 24)


# projection_test.cpp:138-156 — apply_projection goldens.
def test_apply_projection_goldens(orc):
    X = np.array([[1, 2, 3, 4], [10, 20, 30, 40], [100, 200, 300, 400]], np.float32)
    f = np.array([0, 2], np.uint32)
    w = np.array([1, -1], np.float32)
    assert orc.apply_projection(X, f, w, [0, 1, 2, 3]).tolist() == [-99, -198, -297, -396]
    assert orc.apply_projection(X, f, w, [3, 1]).tolist() == [-396, -198]
    assert orc.apply_projection(X, np.zeros(0, np.uint32), np.zeros(0, np.float32), [3, 1]).tolist() == [0, 0]
    assert orc.apply_projection(X, [1], [-1], [0, 1, 2, 3]).tolist() == [-10, -20, -30, -40]


# histogram_test.cpp:19-38 — boundaries are midpoints of all distinct values for small nodes.
def test_sample_boundaries_small_nodes(orc):
    b, used = orc.sample_boundaries([1, 2, 3, 4], 256, 1)
    assert b.tolist() == [1.5, 2.5, 3.5] and used == 0
    assert orc.sample_boundaries([1, 1, 2, 2], 256, 1)[0].tolist() == [1.5]
    assert orc.sample_boundaries([3, 3, 3], 256, 1)[0].tolist() == []
    assert orc.sample_boundaries([3], 256, 1)[0].tolist() == []
    assert orc.sample_boundaries([4, 1, 3, 2], 256, 1)[0].tolist() == [1.5, 2.5, 3.5]


# histogram_test.cpp:40-46 — no RNG draws when n <= bin_count.
def test_sample_boundaries_no_draws_when_small(orc):
    assert orc.sample_boundaries([5, 1, 9], 16, 5)[1] == 0


# histogram_test.cpp:48-58 — bin_count caps the boundary count; strictly increasing.
def test_sample_boundaries_capped(orc):
    b, used = orc.sample_boundaries(np.arange(1000, dtype=np.float32), 64, 2)
    assert 32 <= len(b) <= 63 and used >= 64
    assert np.all(np.diff(b) > 0) and b[0] >= 0 and b[-1] < 999


# histogram_test.cpp:60-68 — adjacent floats clamp to the lower value.
def test_midpoint_clamps_adjacent_floats(orc):
    a = np.float32(1.0)
    b = np.nextafter(a, np.float32(2.0))
    bnd, _ = orc.sample_boundaries(np.array([a, b], np.float32), 256, 3)
    assert bnd.tolist() == [1.0]


# histogram_test.cpp:175-191 — hand-computed histogram (bin-major counts, boundary goes right).
def test_build_histogram_hand_counts(orc):
    c = orc.build_histogram([0.5, 1, 1.5, 2.5, 2.5, 9], [0, 1, 0, 1, 1, 0], [1, 2, 3], 2)
    assert c.tolist() == [1, 0, 1, 1, 0, 2, 1, 0]


# split_test.cpp:61-71 — perfect separation.
def test_exact_perfect_split(orc):
    s = orc.best_split_exact([1, 2, 10, 11], [0, 0, 1, 1], 2)
    assert s.found and s.gain == 1.0 and s.threshold == 6.0 and (s.n_left, s.n_right) == (2, 2)


# split_test.cpp:73-84 — a tie keeps the smallest threshold; -0 and +0 are one group.
def test_exact_tie_smallest_threshold(orc):
    s = orc.best_split_exact([-1, -0.0, 0.0, 1], [0, 0, 1, 1], 2)
    assert s.found and s.threshold == -0.5 and s.n_left == 1
    assert abs(s.gain - (1.0 - 0.75 * (math.log2(3.0) - 2.0 / 3.0))) < 1e-12


# split_test.cpp:86-91 — signed zeros form one group: no split.
def test_exact_signed_zeros(orc):
    assert not orc.best_split_exact([-0.0, 0.0], [0, 1], 2).found


# split_test.cpp:93-113 — n_left equals the count of values <= threshold.
def test_exact_threshold_inside_gap(orc):
    rng = np.random.default_rng(11)
    for _ in range(100):
        n = 2 + int(rng.integers(0, 60))
        v = rng.uniform(-50, 50, n).astype(np.float32)
        y = rng.integers(0, 3, n).astype(np.int32)
        s = orc.best_split_exact(v, y, 3)
        if not s.found:
            continue
        nl = int(np.sum(v <= np.float32(s.threshold)))
        assert nl == s.n_left and n - nl == s.n_right


# split_test.cpp:199-208 — histogram tie keeps the first boundary.
def test_histogram_tie_first_boundary(orc):
    s = orc.best_split_histogram([1, 2, 3], [1, 0, 0, 1, 0, 1, 1, 0], 2)
    assert s.found and s.threshold == 1.0


# split_test.cpp:210-229 — degenerate histogram inputs give no split.
def test_histogram_degenerate(orc):
    assert not orc.best_split_histogram([], [3, 4], 2).found
    assert not orc.best_split_histogram([1], [2, 0, 3, 0], 2).found
    assert not orc.best_split_histogram([1], [1, 0, 0, 0], 2).found


# dataset_test.cpp:226-243 — bootstrap size, sortedness, distinctness, determinism.
def test_bootstrap_properties(orc):
    s = orc.bootstrap(1000, 0.632, 17)
    assert len(s) == 632 and np.all(np.diff(s.astype(np.int64)) > 0) and s[-1] < 1000
    assert np.array_equal(s, orc.bootstrap(1000, 0.632, 17))
    assert not np.array_equal(s, orc.bootstrap(1000, 0.632, 18))
    assert len(orc.bootstrap(1000, 1.0, 1)) == 1000


# forest_test.cpp:383 / bench_test.cpp:63 — root sample counts.
def test_root_sample_counts(orc):
    assert len(orc.bootstrap(20000, 0.632, 5)) == 12640
    assert len(orc.bootstrap(1500, 0.632, 5)) == 948
