"""Thread safety of one operator handle (apply / apply_block are const and
reentrant).  The reference calls apply from its column fan-out workers and from concurrent
jobs on the same operator (operators.cpp:12-17, runner.cpp:110-113); test_operators.cpp:188-209
requires block apply == column apply independent of the worker count.  Here several host
threads hammer ONE device handle with block applies, single-column applies and sketches at
once; every result must equal the serial one bitwise and the apply counter must add up."""
import threading

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
W = pytest.importorskip("paper_2101_07249_b200")
from paper_2101_07249_b200 import configs  # noqa: E402


def test_concurrent_calls_on_one_handle():
    wl = configs.small_advdiff(n=300, N=6, s=4, m=10, k=5)
    op = wl.hessian(0)
    n = op.dim()
    blocks = [O.gaussian_matrix(n, 3 + (t % 4), 100 + t) for t in range(8)]
    serial = [op.apply_block(V) for V in blocks]
    cols = [op.apply(V[:, 0]) for V in blocks]
    cfg = W.SketchConfig(wl.k, wl.m - wl.k, 1, "nystrom")
    sk_serial = W.sketch_eigenpairs(op, cfg)
    op.reset_apply_count()
    out = [None] * 8
    errs = []

    def worker(t):
        try:
            res = []
            for _ in range(5):
                res.append(op.apply_block(blocks[t]))
                res.append(op.apply(blocks[t][:, 0]))
                if t % 4 == 0:
                    res.append(W.sketch_eigenpairs(op, cfg).values)
            out[t] = res
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=worker, args=(t,)) for t in range(8)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs, errs
    expect = 0
    for t in range(8):
        res = out[t]
        step = 3 if t % 4 == 0 else 2
        for r in range(5):
            assert np.array_equal(res[r * step], serial[t])
            assert np.array_equal(res[r * step + 1], cols[t])
            assert np.array_equal(res[r * step + 1], serial[t][:, 0])  # column == block column
            if step == 3:
                assert np.array_equal(res[r * step + 2], sk_serial.values)
        expect += 5 * (blocks[t].shape[1] + 1) + (5 * 2 * wl.m if t % 4 == 0 else 0)
    assert op.apply_count() == expect
