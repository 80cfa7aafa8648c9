"""CPU checks of the C-ABI boundary: the library loads without a GPU, exports exactly the
entry points declared in include/wc4dvar_gpu.h, and compute calls fail loudly (no CPU
fallback) when no device is present."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "wc4dvar_gpu.h")).read()
    return set(re.findall(r"\b(wc4dvar_gpu_\w+)\s*\(", src))


def test_library_exports_every_header_symbol():
    import paper_2101_07249_b200 as w
    out = subprocess.run(["nm", "-D", "--defined-only", w.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (wc4dvar_gpu_\w+)", out))
    declared = header_symbols()
    assert declared, "no declarations parsed"
    assert declared <= exported, declared - exported
    assert declared == set(w.SIGNATURES), declared ^ set(w.SIGNATURES)


def test_sm100a_code_only():
    import paper_2101_07249_b200 as w
    out = subprocess.run(["cuobjdump", "--list-elf", w.LIB_PATH], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_\d+a?", out))
    assert arches == {"sm_100a"}, arches
    sass = subprocess.run(["cuobjdump", "-sass", w.LIB_PATH], capture_output=True, text=True).stdout
    assert "DMMA" in sass  # fp64 tensor-core path is compiled in


def test_host_rng_matches_golden():
    import json
    import paper_2101_07249_b200 as w
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "normal_stream.json")))
    G = w.gaussian_matrix(40, 7, 99)
    ref = np.array(gold["gaussian_40x7_seed99"]).reshape(7, 40).T
    assert np.array_equal(G, ref)
    for seed, vals in gold["normal"].items():
        assert np.array_equal(w.gaussian_matrix(len(vals), 1, int(seed))[:, 0], np.array(vals))


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2101_07249_b200 as w
    with pytest.raises(w.DeviceError):
        w.DenseOperator(np.eye(4))


def test_cpp_host_header_compiles():
    """include/wc4dvar_gpu.hpp (the C++ mirror of the reference API) and its test program
    compile and link against the library without a GPU."""
    out = "/tmp/_w4_test_cpp_api"
    cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "test_cpp_api.cpp"), "-L", os.path.join(ROOT, "paper_2101_07249_b200"),
           "-lwc4dvar_gpu", "-L", os.path.join(ROOT, "oracle"), "-loracle", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
