#!/usr/bin/env python
"""Benchmark of the randomized-LMP hot path on the largest single-GPU BASELINE config.

Metric (BASELINE.json): "Hessian-block apply columns/s and LMP build ms; fraction of HBM
roofline".  Headline workload: configs[3] (C4) -- advection-diffusion n = 1e6, Nsw = 16,
10 TL sub-steps per subwindow (n_A = 1.7e7), circulant SOAR L = 50 B^{1/2} / Q^{1/2}, every
10th point observed -- with the widest sketch k = 256 columns.  One step = one block
product A*Omega (operators.cpp:127-144) of the 256-column sketch drawn from the
reference's NormalStream(1) (device jump-ahead generator, random.hpp:14-42).
Multi-GPU: the 256 columns of the ONE global sketch shard across ranks (strong scaling,
no data-path collective); `value` is whole-job columns/s, timed on the device as the max
over ranks.

Secondary keys (N = 1 only): per-config applies (C2, C3, C5 rank share), LMP build ms
(REVD / Nystrom / ritzit at C2, C3 and C4 k = 256), LMP-PCG time-to-solution (C2, C3, C4),
and the CPU baseline (oracle port, all host cores, bounded column sample).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--no-extras]

`--gpus N` without torchrun re-launches itself under torch.distributed.run with N ranks.
`--impl reference` times the CPU oracle port of the same path (the reference itself is
not buildable here: Eigen is absent) WITHOUT importing the product package.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Hessian-block apply columns/s (A*Omega, C4 n_A=1.7e7, k=256); LMP build ms"
UNIT = "columns/s"
M_GLOBAL = 256           # C4 sketch width (the widest of BASELINE configs[3]'s k in {16, 64, 256})
OMEGA_SEED = 1           # the reference's sketch_base = 1 (proj/configs/advection.cfg:39)
RHS_SEED = 2
CPU_SAMPLE_COLS = 16     # CPU legs: columns of the same sketch per step


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-extras", action="store_true", help="headline only (no secondary configs / LMP / PCG)")
    return ap.parse_args()


def env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: re-launch under torch.distributed.run."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def c4_counts(n=1_000_000, N=16, s=10, q=1_600_000, m=M_GLOBAL):
    """SURVEY §8(d) per-column algorithmic counts for C4, times m columns."""
    nA = n * (N + 1)
    fft_launch = (N + 1) * m * (5.0 * n * math.log2(n) + n)      # one D^{1/2} (real-FFT convention)
    flops = (10.0 * N * s * n + 2.0 * (N + 1) * (5.0 * n * math.log2(n) + n)) * m
    bytes_ = 8.0 * (3 * nA + 2 * q) * m
    return nA, fft_launch, flops, bytes_


def c4_config(world: int, m_per_gpu: int) -> dict:
    """The `config` object of both arms (identical keys and values at the same N)."""
    n, N, s, q = 1_000_000, 16, 10, 1_600_000
    nA = n * (N + 1)
    return {"workload": "C4-advdiff-n1e6-N16-s10-k256", "n": n, "Nsw": N, "substeps": s, "n_A": nA,
            "sketch_columns": M_GLOBAL, "sketch_columns_per_gpu": m_per_gpu, "q": q,
            "covariance": "circulant SOAR L=50", "parallelism": f"column-sharded x{world} (one global sketch)",
            "l2": "inputs larger than L2 (sketch block %.1f GB per GPU); no flush" % (8e-9 * nA * m_per_gpu)}


def profile_traffic(name: str, kernel: str):
    """DRAM bytes per launch of `kernel` from a committed `ncu --set full` summary."""
    path = os.path.join(ROOT, "profiles", name)
    try:
        ks = [k for k in json.load(open(path))["kernels"] if kernel in k["kernel"]]
        return sum(k["traffic_bytes"] for k in ks) / len(ks), os.path.relpath(path, ROOT)
    except (OSError, KeyError, ValueError, ZeroDivisionError):
        return None, None


# ------------------------------------------------------------------------------ reference
def oracle_c4(threads: int, cols: int):
    """The C4 operator and the first `cols` columns of the same NormalStream(1) sketch, from
    the CPU oracle alone (oracle/workloads.py: never imports the product package)."""
    from oracle import oracle as O
    from oracle import workloads as OW
    wl = OW.config4(M_GLOBAL, threads=threads)
    V = O.gaussian_matrix(wl.dim, cols, OMEGA_SEED)
    return wl, V


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    cols = CPU_SAMPLE_COLS
    wl, V = oracle_c4(threads, cols)
    cfg = c4_config(world, M_GLOBAL // world)
    assert (wl.n, wl.N, wl.substeps, wl.dim, wl.q) == (cfg["n"], cfg["Nsw"], cfg["substeps"], cfg["n_A"], cfg["q"])
    for _ in range(args.warmup):
        wl.op.apply_block_fast(V, threads)
    secs = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        wl.op.apply_block_fast(V, threads)
        secs.append(time.perf_counter() - t0)
    total = sum(secs)
    value = cols * args.steps / total
    sample = (f"{cols} of the {M_GLOBAL} sketch columns per step (columns 0..{cols - 1} of NormalStream(1)); "
              f"oracle port of HessianOperator::apply_block (reference not buildable: Eigen absent): "
              f"circulant D^1/2 as a batched real FFT (scipy.fft, {threads} workers), TL/adjoint sweeps in C "
              f"with the reference's column fan-out over {threads} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (NormalStream(1) sketch, BASELINE configs[3] operator)",
        "config": cfg,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------ ours
def run_ours(args):
    import numpy as np
    import torch

    rank, world, local = env_rank()
    if args.gpus != world:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if M_GLOBAL % world:
        raise SystemExit(f"bench.py: {M_GLOBAL} sketch columns do not split over {world} ranks")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    import paper_2101_07249_b200 as W
    from paper_2101_07249_b200 import configs

    m = M_GLOBAL // world
    wl = configs.config4(M_GLOBAL)
    op = wl.hessian(local)
    nA = op.dim()
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    # this rank's columns [rank m, (rank + 1) m) of gaussian_matrix(n_A, 256, 1)
    V = torch.empty((m, nA), dtype=torch.float64, device=dev)
    W.gaussian_block_dev(V, nA, OMEGA_SEED, col0=rank * m, stream=sp)
    out = torch.empty_like(V)
    fp64_peak = W.probe_dmma_peak(local)

    def maxrank(x):
        if not dist:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(max(args.warmup, 3)):
        op.apply_block_dev(V, out, sp)
    torch.cuda.synchronize()

    op.profile(True)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = W.launch_count()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            starts[i].record(stream)
            op.apply_block_dev(V, out, sp)
            ends[i].record(stream)
        torch.cuda.synchronize()
    launches = W.launch_count() - l0
    if dist:
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = maxrank(sum(step_ms))
    stage_ms, calls = op.profile_read()
    op.profile(False)
    value = M_GLOBAL * args.steps / (total_ms / 1e3)
    step_mean_ms = total_ms / args.steps
    clocks = clk.summary()

    # ---- roofline of the dominant kernel
    # Fourier-space apply (the default for C4): forward transform, window recurrence, inverse
    # transform + identity; the inverse transform is the longest launch.  Its algorithmic work
    # is HALF a convolution, (N+1) m 2.5 n log2 n flops (real-FFT convention),
    # against 24 n_A m bytes (spectra in, v in, result out): the HBM roof binds it.
    # Grid-space apply (WC4DVAR_SPECTRAL=0): the fused convolution, fp64-bound.
    spectral = op.spectral()
    _, fft_flops_launch, flops_step, bytes_step = c4_counts(m=m)
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        peaks = {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    st3 = [x / max(calls, 1) for x in stage_ms]
    if spectral:
        inv_ms, fwd_ms, win_ms = st3[2], st3[0], st3[1]
        inv_bytes, fwd_bytes, win_bytes = 24.0 * nA * m, 16.0 * nA * m, 16.0 * nA * m
        half_flops = 0.5 * (fft_flops_launch - (wl.model.N + 1) * m * wl.model.n)
        traffic, traffic_src = profile_traffic("r02e_c4_spectral_m256.json", "1, 1, 2>")
        roofline = {"bound": "hbm", "achieved": inv_bytes / (inv_ms * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                    "frac": inv_bytes / (inv_ms * 1e-3) / 1e9 / hbm_peak, "traffic": traffic,
                    "traffic_source": traffic_src,
                    "kernel": "fftconv_kernel MODE 2 (inverse four-step transform of the window spectra + identity)",
                    "bytes_per_launch": inv_bytes, "launch_ms": inv_ms,
                    "bytes_per_unit": "24 n_A per sketch column: 8 n_A of spectra in (two columns per complex "
                                      "transform), 8 n_A of v in, 8 n_A out",
                    "flops_per_launch": half_flops, "fp64_tflops": half_flops / (inv_ms * 1e-3) / 1e12,
                    "fp64_frac": half_flops / (inv_ms * 1e-3) / 1e12 / fp64_peak,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs (sustained copy); fp64 peak measured in this run "
                                   "(all-SM mma.sync.f64 probe)",
                    "other_kernels": {
                        "fftconv_kernel MODE 1 (forward transform)": {
                            "launch_ms": fwd_ms, "bytes_per_launch": fwd_bytes,
                            "hbm_frac": fwd_bytes / (fwd_ms * 1e-3) / 1e9 / hbm_peak,
                            "fp64_frac": half_flops / (fwd_ms * 1e-3) / 1e12 / fp64_peak},
                        "spectral_window_kernel (window recurrences per frequency class)": {
                            "launch_ms": win_ms, "bytes_per_launch": win_bytes,
                            "hbm_frac": win_bytes / (win_ms * 1e-3) / 1e9 / hbm_peak}}}
        stage_names = ("transform_forward", "window_recurrence", "transform_inverse_plus_identity")
    else:
        fft_ms = st3[0]   # the first D^{1/2}: one fftconv_kernel launch
        achieved = fft_flops_launch / (fft_ms * 1e-3) / 1e12
        traffic, traffic_src = profile_traffic("r02d_c4_fftconv_m256.json", "PlanE6, 2, 0")
        roofline = {"bound": "fp64", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                    "frac": achieved / fp64_peak, "traffic": traffic, "traffic_source": traffic_src,
                    "kernel": "fftconv_kernel (circulant D^1/2: fused four-step FFT convolution)",
                    "flops_per_launch": fft_flops_launch, "launch_ms": fft_ms,
                    "flops_per_unit": "(N+1)(5 n log2 n + n) per sketch column (real-FFT convention, SURVEY §8(d))",
                    "peak_source": "measured in this run: all-SM mma.sync.f64 probe (the FP64 FMA pipe "
                                   "measures the same ~36-37 TF/s, profiles/r01_fp64_pipes_probe.txt)"}
        stage_names = ("d_half_in", "sweep", "d_half_out_plus_identity")
    t_roof = max(flops_step / (fp64_peak * 1e12), bytes_step / (hbm_peak * 1e9)) * 1e3

    # ---- e2e: the reference-facing C-ABI (wc4dvar_gpu_op_apply_block) with pinned HOST buffers
    Vh = torch.empty((m, nA), dtype=torch.float64, pin_memory=True)
    Vh.copy_(V)
    Oh = torch.empty((m, nA), dtype=torch.float64, pin_memory=True)
    del V, out
    torch.cuda.empty_cache()
    op.apply_block_host_ptr(Vh.data_ptr(), nA, m, Oh.data_ptr(), nA)
    if dist:
        dist.barrier()
    e2e_steps = max(2, min(args.steps, 5))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        op.apply_block_host_ptr(Vh.data_ptr(), nA, m, Oh.data_ptr(), nA)
    e2e_s = maxrank(time.perf_counter() - t0)
    e2e_value = M_GLOBAL * e2e_steps / e2e_s
    check = float(Oh[0, :4].sum())  # read back (the step's result on the host)
    del Vh, Oh

    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_mean_ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded N(0,1) sketch = the reference NormalStream(1) stream, generated on the "
                    "device with MT19937-64 jump-ahead; BASELINE configs[3] operator)",
            "config": c4_config(world, m),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * nA * m,
                    "d2h_bytes_per_step": 8 * nA * m, "steps": e2e_steps,
                    "path": "wc4dvar_gpu_op_apply_block (host pointers, pinned): two-slot chunk ring, H2D / "
                            "compute / D2H on three streams", "checksum": check},
            "gpu_launches": launches,
            "roofline": roofline,
            "apply_path": "fourier-space (forward transform, window recurrence per frequency class, inverse "
                          "transform)" if spectral else "grid-space (convolution, stencil sweeps, convolution)",
            "apply_roofline": {"t_roof_ms": t_roof, "frac": t_roof / step_mean_ms,
                               "bound": "fp64" if flops_step / (fp64_peak * 1e12) >= bytes_step / (hbm_peak * 1e9)
                               else "hbm",
                               "definition": "SURVEY §8(d) algorithmic counts of the grid-space apply (two "
                                             "convolutions + stencil sweeps), whichever path runs",
                               "flops_per_step": flops_step, "bytes_per_step": bytes_step,
                               "hbm_gbs": bytes_step / (step_mean_ms * 1e-3) / 1e9, "hbm_peak_gbs": hbm_peak,
                               "hbm_frac": bytes_step / (step_mean_ms * 1e-3) / 1e9 / hbm_peak},
            "stage_ms": dict(zip(stage_names, st3)),
            "clocks": clocks,
        }
    del op
    torch.cuda.empty_cache()

    if not args.no_extras and rank == 0 and world == 1:
        extras = {}
        for key, fn in (("configs", lambda: run_configs(W, configs, fp64_peak, hbm_peak)),
                        ("lmp", lambda: run_lmp(W, configs, dev)),
                        ("cpu_baseline", lambda: cpu_baseline())):
            try:
                extras[key] = fn()
            except Exception as e:  # report, never lose the headline line
                extras[key] = {"error": f"{type(e).__name__}: {e}"[:400]}
            torch.cuda.empty_cache()
        cb = extras.pop("cpu_baseline")
        line["cpu_baseline"] = cb
        line.update(extras)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def cpu_baseline():
    threads = os.cpu_count() or 1
    wl, V = oracle_c4(threads, CPU_SAMPLE_COLS)
    wl.op.apply_block_fast(V, threads)
    t0 = time.perf_counter()
    wl.op.apply_block_fast(V, threads)
    secs = time.perf_counter() - t0
    return {"value": CPU_SAMPLE_COLS / secs, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{CPU_SAMPLE_COLS} of the {M_GLOBAL} C4 sketch columns (NormalStream(1) columns 0..15), "
                      f"one warm apply; oracle port (reference not buildable: Eigen absent): batched real-FFT "
                      f"circulant D^1/2 (scipy.fft, {threads} workers) + C sweeps, {threads}-thread column fan-out"}


def _apply_timing(W, wl, m, fp64_peak, hbm_peak, reps=3):
    import torch
    op = wl.hessian(0)
    nA, q = op.dim(), wl.net.q
    n, N, s = wl.model.n, wl.model.N, wl.model.substeps
    V = torch.empty((m, nA), dtype=torch.float64, device="cuda")
    W.gaussian_block_dev(V, nA, OMEGA_SEED)
    Y = torch.empty_like(V)
    sp = torch.cuda.current_stream().cuda_stream
    for _ in range(2):
        op.apply_block_dev(V, Y, sp)
    op.profile(True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        op.apply_block_dev(V, Y, sp)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    st, calls = op.profile_read()
    op.profile(False)
    spectral = op.spectral()
    if wl.b_half.kind == "dense":
        f_cov = 4.0 * n * n * (N + 1)
    else:
        f_cov = 2.0 * (N + 1) * (5.0 * n * math.log2(n) + n)
    f_model = (92.0 if wl.model.kind == "l96" else 10.0) * N * s * n
    t_f = (f_model + f_cov) * m / (fp64_peak * 1e12)
    t_b = 8.0 * (3 * nA + 2 * q) * m / (hbm_peak * 1e9)
    t_roof = max(t_f, t_b) * 1e3
    return {"workload": wl.name, "m": m, "ms_per_apply": ms, "columns_per_s": m / (ms * 1e-3),
            "apply_path": "fourier-space" if spectral else "grid-space",
            "stage_ms": dict(zip(("transform_forward", "window_recurrence", "transform_inverse_plus_identity")
                                 if spectral else ("d_half_in", "sweep", "d_half_out_plus_identity"),
                                 [x / max(calls, 1) for x in st])),
            "roofline": {"t_roof_ms": t_roof, "bound": "fp64" if t_f >= t_b else "hbm", "frac": t_roof / ms}}


def run_configs(W, configs, fp64_peak, hbm_peak):
    """Block applies of the other BASELINE configs (N = 1): C2 (dense SOAR, m = 100), C3
    (Lorenz-96, m = 64), C4 at k = 16 / 64, and C5 at one rank's 32-column share of its
    8-GPU sketch."""
    out = {}
    for name, mk, m in (("C2", configs.config2, 100), ("C3", configs.config3, 64),
                        ("C4_k16", lambda: configs.config4(16), 16), ("C4_k64", lambda: configs.config4(64), 64),
                        ("C5_rank_share", lambda: configs.config5(32), 32)):
        try:
            out[name] = _apply_timing(W, mk(), m, fp64_peak, hbm_peak)
        except Exception as e:
            out[name] = {"error": f"{type(e).__name__}: {e}"[:300]}
    return out


def run_lmp(W, configs, dev):
    """LMP build ms (Omega resident on the device -> U, Theta on the device; second, warm call)
    per method, and LMP-PCG time-to-solution to relative residual 1e-6 (krylov.cpp:22-99).
    C5_k64 is BASELINE configs[4]'s inner loop on ONE GPU with a 64-column Nystrom / REVD
    sketch (the k = 256 sketch needs 4 x 86 GB blocks: the 8-GPU configuration)."""
    import numpy as np
    import torch
    res = {}
    for name, mk, pcg_methods, max_iter in (
            ("C2", configs.config2, ("none", "revd", "nystrom", "ritzit"), 1000),
            ("C3", configs.config3, ("none", "nystrom"), 20000),
            ("C4_k256", lambda: configs.config4(256), ("none", "nystrom"), 2000),
            ("C5_k64", lambda: configs.config5(64), ("none", "revd", "nystrom"), 100)):
        r = {"build_ms": {}, "build_stage_ms": {}, "pcg": {}}
        try:
            wl = mk()
            op = wl.hessian(0)
            nA, m, k = op.dim(), wl.m, wl.k
            r.update({"workload": wl.name, "m": m, "k": k})
            Om = torch.empty((m, nA), dtype=torch.float64, device=dev)
            W.gaussian_block_dev(Om, nA, OMEGA_SEED)
            U = torch.empty((k, nA), dtype=torch.float64, device=dev)
            th = torch.empty(k, dtype=torch.float64, device=dev)
            kept = {}
            methods = ("revd", "ritzit", "nystrom") if name != "C5_k64" else ("revd", "nystrom")
            for method in methods:
                cfg = W.SketchConfig(k, m - k, OMEGA_SEED, method, 1)
                W.sketch_eigenpairs_dev(op, cfg, Om, U, th)          # warm (grows workspaces)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                kk = W.sketch_eigenpairs_dev(op, cfg, Om, U, th)
                torch.cuda.synchronize()
                wall = 1e3 * (time.perf_counter() - t0)
                t = W.last_sketch_timing()
                r["build_ms"][method] = t["total_ms"]
                r["build_stage_ms"][method] = dict({kk_: v for kk_, v in t.items() if kk_ != "total_ms"},
                                                   wall_ms=wall)
                r.setdefault("theta_head", {})[method] = th[:3].cpu().tolist()
                if method in pcg_methods:
                    if method == methods[-1]:   # last: free the sketch blocks before the factor copies U
                        del Om
                        op.release_workspaces()
                        torch.cuda.empty_cache()
                    kept[method] = W.build_spectral_lmp_dev(U, th, kk, 0)
            del U, th
            op.release_workspaces()
            torch.cuda.empty_cache()
            b = torch.empty((1, nA), dtype=torch.float64, device=dev)
            W.gaussian_block_dev(b, nA, RHS_SEED)
            bh = b[0].cpu().numpy()
            del b
            for method in pcg_methods:
                f = kept.get(method)
                t0 = time.perf_counter()
                pr = W.pcg_split(op, bh, f, opts=W.PcgOptions(max_iter=max_iter, rel_tol=1e-6))
                ms = 1e3 * (time.perf_counter() - t0)
                r["pcg"][method] = {"ms": ms, "iterations": pr.history.iterations,
                                    "converged": pr.history.converged,
                                    "ms_per_iteration": ms / max(pr.history.iterations, 1)}
            del kept, op
        except Exception as e:
            r["error"] = f"{type(e).__name__}: {e}"[:400]
        torch.cuda.empty_cache()
        res[name] = r
    return res


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
