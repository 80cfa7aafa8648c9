"""Check and time the fused four-step circulant D^{1/2} (fft4.cu) on the GPU.

Parity: n = 1e4 against the oracle's direct circulant convolution (full Hessian apply_block,
which exercises the add / identity epilogue), n = 1e5 / 1e6 / 2e6 against a numpy FFT
convolution of each window column.  Timing: device-resident D^{1/2} of the C3 / C4 blocks
through apply_block_dev stage timers (fused path vs WC4DVAR_FFT4=0 in a child process)."""
import json
import math
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import paper_2101_07249_b200 as W  # noqa: E402
from paper_2101_07249_b200 import configs  # noqa: E402


def relerr(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300))


def np_dhalf(bh, qh, v, n, N):
    fb, fq = np.fft.rfft(bh.half), np.fft.rfft(qh.half)
    out = np.empty_like(v)
    for i in range(N + 1):
        f = fb if i == 0 else fq
        out[i * n:(i + 1) * n] = np.fft.irfft(np.fft.rfft(v[i * n:(i + 1) * n]) * f, n)
    return out


def parity():
    from oracle import oracle as O
    from gpu_helpers import pair
    res = {}
    n, N, m = 10000, 3, 5
    bh = configs.circulant_sqrt(configs.soar_first_column(1.0, 5.0, n))
    qh = configs.circulant_sqrt(configs.soar_first_column(math.sqrt(0.05), 5.0, n))
    g, o = pair(W.AdvDiffLinearized(n, N, 0.5, 0.2, 3), W.ObservationNetwork.build(n, N, 4, 1), bh, qh, 0.1)
    V = O.gaussian_matrix(g.dim(), m, 1)
    res["1e4_apply_block"] = relerr(g.apply_block(V), o.apply_block(V))
    res["1e4_dhalf"] = relerr(g.apply_D_half(V[:, 0]), o.apply_D_half(V[:, 0]))
    res["1e4_dhalf_inv"] = relerr(g.apply_D_half_inv(V[:, 1]), o.apply_D_half_inv(V[:, 1]))
    for n, N, L in ((100000, 2, 4.0), (1000000, 2, 50.0), (2000000, 1, 4.0)):
        bh = configs.circulant_sqrt(configs.soar_first_column(1.0, L, n))
        qh = configs.circulant_sqrt(configs.soar_first_column(math.sqrt(0.05), L, n))
        g = W.HessianOperator(W.AdvDiffLinearized(n, N, 0.5, 0.2, 2), W.ObservationNetwork.build(n, N, 10, 1),
                              bh, qh, 0.1)
        v = np.random.default_rng(3).standard_normal(n * (N + 1))
        res[f"{n}_dhalf"] = relerr(g.apply_D_half(v), np_dhalf(bh, qh, v, n, N))
    return res


def timing():
    import torch
    out = {}
    for name, wl, m in (("c3", configs.config3(), 64), ("c4", configs.config4(64), 64)):
        op = wl.hessian(0)
        n = op.dim()
        gen = torch.Generator(device="cuda").manual_seed(1)
        V = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=gen)
        Y = torch.empty_like(V)
        sp = torch.cuda.current_stream().cuda_stream
        op.apply_block_dev(V, Y, sp)
        op.profile(True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        e0.record()
        for _ in range(reps):
            op.apply_block_dev(V, Y, sp)
        e1.record()
        torch.cuda.synchronize()
        st, calls = op.profile_read()
        out[name] = {"ms_per_apply": e0.elapsed_time(e1) / reps, "stage_ms": [x / max(calls, 1) for x in st]}
        del V, Y, op
        torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "timing":
        print(json.dumps(timing()), flush=True)
        sys.exit(0)
    print(json.dumps({"parity": parity()}), flush=True)
    for flag in ("1", "0"):
        p = subprocess.run([sys.executable, __file__, "timing"], env=dict(os.environ, WC4DVAR_FFT4=flag),
                           capture_output=True, text=True, timeout=1200)
        print(json.dumps({"WC4DVAR_FFT4": flag, "rc": p.returncode,
                          "out": p.stdout.strip()[-2000:], "err": p.stderr.strip()[-1500:]}), flush=True)
