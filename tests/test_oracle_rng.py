"""Pins the oracle's NormalStream (random.hpp:14-42) bit-for-bit against libstdc++'s
std::mt19937_64 golden vectors (tests/golden/normal_stream.json, made by
oracle/gen_golden_rng.cpp)."""
import json
import os

import numpy as np

from oracle import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "normal_stream.json")))


def test_raw_engine_matches_libstdcxx():
    for seed, vals in GOLD["raw"].items():
        s = O.NormalStream(int(seed))
        got = [s.raw() for _ in range(len(vals))]
        assert got == [int(v) for v in vals], seed


def test_normals_bit_exact():
    for seed, vals in GOLD["normal"].items():
        got = O.NormalStream(int(seed)).draw(len(vals))
        assert np.array_equal(got, np.array(vals)), seed


def test_gaussian_matrix_column_major_fill():
    # randevd.cpp:16-21 + random.hpp:28-31; the shape of test_randevd.cpp:24-30
    G = O.gaussian_matrix(40, 7, 99)
    ref = np.array(GOLD["gaussian_40x7_seed99"]).reshape(7, 40).T
    assert np.array_equal(G, ref)
    assert np.array_equal(G, O.gaussian_matrix(40, 7, 99))
    assert np.abs(G - O.gaussian_matrix(40, 7, 100)).max() > 0.0


def test_long_stream_checksum():
    g = GOLD["seed7_1e6"]
    v = O.NormalStream(7).draw(1000000)
    assert v[-1] == g["last"]
    assert abs(v.sum() - g["sum"]) <= 1e-9 * abs(g["sum2"])


def test_standard_moments():
    # test_randevd.cpp:32-38
    g = O.gaussian_matrix(1000, 1000, 7)
    assert abs(g.mean()) <= 0.01
    assert abs(g.var(ddof=1) - 1.0) <= 0.01
