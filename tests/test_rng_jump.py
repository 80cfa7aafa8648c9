"""MT19937-64 jump-ahead of the device NormalStream (SURVEY §7 hard part 3), host side:
the library's GF(2) jump polynomial x^D mod p and window-XOR jump reproduce libstdc++'s
std::mt19937_64 at large offsets (golden vectors from oracle/gen_golden_rng.cpp, made with
std::mt19937_64::discard)."""
import json
import os

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "normal_stream.json")))


@pytest.mark.parametrize("offset", sorted(GOLD["raw_at"]["1"], key=int))
def test_host_jump_matches_libstdcxx(offset):
    import paper_2101_07249_b200 as w
    got = w.mt19937_raw_host(1, int(offset), 8)
    assert [int(v) for v in got] == [int(v) for v in GOLD["raw_at"]["1"][offset]]


def test_host_jump_other_seed_and_start():
    import paper_2101_07249_b200 as w
    got = w.mt19937_raw_host(5, 100000000, 8)
    assert [int(v) for v in got] == [int(v) for v in GOLD["raw_at"]["5"]["100000000"]]
    for seed, vals in GOLD["raw"].items():  # offset 0: the plain stream, 700 draws (2 twists)
        assert [int(v) for v in w.mt19937_raw_host(int(seed), 0, 700)] == [int(v) for v in vals]
