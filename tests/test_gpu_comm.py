"""The C-ABI NCCL plumbing for a C++ host on the one GPU this round
has: a one-rank communicator through unique id -> create -> collectives -> destroy; at one
rank the all-reduce / all-gather / transposes must reproduce their input exactly.  The
partition and packing of the transposes are the ones the gloo tests of distributed.py
exercise at world size 2."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

W = pytest.importorskip("paper_2101_07249_b200")
torch = pytest.importorskip("torch")
lib = W.wc4dvar.lib


def _vp(t):
    return ctypes.c_void_p(t.data_ptr())


def test_one_rank_communicator_roundtrip():
    uid = ctypes.create_string_buffer(128)
    assert lib.wc4dvar_gpu_comm_unique_id(uid) == 0
    comm = ctypes.c_void_p()
    assert lib.wc4dvar_gpu_comm_create(uid, 0, 1, 0, ctypes.byref(comm)) == 0, lib.wc4dvar_gpu_last_error()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    g = torch.Generator(device="cuda").manual_seed(3)
    nrows, ncols = 1003, 17
    A = torch.randn(ncols, nrows, dtype=torch.float64, device="cuda", generator=g)  # column-major nrows x ncols
    buf = A.clone()
    assert lib.wc4dvar_gpu_comm_allreduce_sum(comm, _vp(buf), buf.numel(), st) == 0
    gat = torch.empty_like(A)
    assert lib.wc4dvar_gpu_comm_allgather(comm, _vp(A), A.numel(), _vp(gat), st) == 0
    rows = torch.empty_like(A)
    assert lib.wc4dvar_gpu_comm_cols_to_rows(comm, _vp(A), nrows, ncols, _vp(rows), st) == 0
    back = torch.empty_like(A)
    assert lib.wc4dvar_gpu_comm_rows_to_cols(comm, _vp(rows), nrows, ncols, _vp(back), st) == 0
    torch.cuda.synchronize()
    for t in (buf, gat, rows, back):
        assert torch.equal(t, A)
    assert lib.wc4dvar_gpu_comm_destroy(comm) == 0


def test_comm_argument_errors():
    comm = ctypes.c_void_p()
    uid = ctypes.create_string_buffer(128)
    assert lib.wc4dvar_gpu_comm_create(uid, 2, 2, 0, ctypes.byref(comm)) == 1  # rank out of range
    assert b"comm_create" in lib.wc4dvar_gpu_last_error()
