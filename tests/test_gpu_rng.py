"""Device NormalStream with MT19937-64 jump-ahead (random.hpp:14-42, randevd.cpp:16-21):
raw engine outputs bit-exact with libstdc++ std::mt19937_64 at large offsets, and the
normals of far columns / row blocks of gaussian_matrix within a few ulp of the reference's
glibc Box-Muller (golden vectors: oracle/gen_golden_rng.cpp)."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
W = pytest.importorskip("paper_2101_07249_b200")
torch = pytest.importorskip("torch")

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "normal_stream.json")))
ULP_TOL = 8  # device log / cos / sqrt vs glibc: a few ulp


def ulps(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return np.abs(a - b) / np.spacing(np.maximum(np.abs(a), np.abs(b)))


def block(n_total, rows, cols, seed, row0=0, col0=0):
    out = torch.empty((cols, rows), dtype=torch.float64, device="cuda")
    W.gaussian_block_dev(out, n_total, seed, row0=row0, col0=col0)
    torch.cuda.synchronize()
    return out.cpu().numpy().T  # rows x cols, column-major view


@pytest.mark.parametrize("offset", sorted(GOLD["raw_at"]["1"], key=int))
def test_device_raw_engine_bit_exact(offset):
    got = W.mt19937_raw_dev(1, int(offset), 8)
    assert [int(v) for v in got] == [int(v) for v in GOLD["raw_at"]["1"][offset]]


def test_device_raw_plain_stream():
    for seed, vals in GOLD["raw"].items():
        assert [int(v) for v in W.mt19937_raw_dev(int(seed), 0, 700)] == [int(v) for v in vals]


def test_gaussian_matrix_40x7_within_ulps():
    G = block(40, 40, 7, 99)
    ref = np.array(GOLD["gaussian_40x7_seed99"]).reshape(7, 40).T
    assert ulps(G, ref).max() <= ULP_TOL


def test_far_columns_and_row_blocks():
    for c, vals in GOLD["gaussian_cols_rows17e6_seed1"].items():
        G = block(17_000_000, 4, 1, 1, col0=int(c))
        assert ulps(G[:, 0], vals).max() <= ULP_TOL, c
    G = block(1_000_003, 4, 1, 1, row0=500_000, col0=3)
    assert ulps(G[:, 0], GOLD["gaussian_rows_n1000003_col3_row500000_seed1"]).max() <= ULP_TOL


def test_block_equals_host_stream_everywhere():
    n, m = 5003, 37  # rows not a multiple of the 156-normal twist, odd column count
    G = block(n, n, m, 7)
    H = W.gaussian_matrix(n, m, 7)
    u = ulps(G, H)
    assert u.max() <= ULP_TOL, u.max()
    # sub-blocks are slices of the same matrix (column and row shards)
    S = block(n, 1000, 5, 7, row0=1234, col0=30)
    assert ulps(S, H[1234:2234, 30:35]).max() <= ULP_TOL
