#!/usr/bin/env python
"""Benchmark of the randomized-LMP hot path on BASELINE.json configs[1] (C2).

Metric (BASELINE.json): "Hessian-block apply columns/s and LMP build ms; fraction of HBM
roofline".  One step = one block product A*Omega of the first-level-preconditioned
inner-loop Hessian (operators.cpp:127-144) with an n_A x m Gaussian sketch, m = 100,
n_A = 2000 * 21 = 42 000 (advection-diffusion, 10 TL sub-steps per subwindow, dense SOAR
B^{1/2}, Q^{1/2}).  Multi-GPU: the sketch columns shard by rank with no data-path
collective (weak scaling, each rank applies its own 100-column block).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Hessian-block apply columns/s (A*Omega, C2); LMP build ms"
UNIT = "columns/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-extras", action="store_true", help="skip LMP-build / PCG timings")
    return ap.parse_args()


def env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


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


def build_workload():
    from paper_2101_07249_b200 import configs
    return configs.config2()


def algorithmic_counts(wl, m):
    n, N, q = wl.model.n, wl.model.N, wl.net.q
    nA = n * (N + 1)
    s = wl.model.substeps
    flops_gemm = 2.0 * n * n * (N + 1) * m             # one D^{1/2} application (B and Q blocks)
    flops_model = 10.0 * N * s * n * m                  # adv-diff TL + adjoint stencils
    bytes_step = 8.0 * (3 * nA * m + 2 * q * m + 4 * n * n)  # v twice, Av once, y w+r, factors
    return nA, flops_gemm, flops_model, bytes_step


def gemm_traffic():
    """DRAM bytes per launch of the D^1/2 GEMM from the committed `ncu --set full` capture
    (dram__bytes_read.sum + dram__bytes_write.sum, averaged over the captured launches)."""
    path = os.path.join(ROOT, "profiles", "r01_gemm_sym_stream_k.json")
    try:
        ks = [k for k in json.load(open(path))["kernels"] if "gemm_sym_ws" in k["kernel"]]
        return sum(k["traffic_bytes"] for k in ks) / len(ks), os.path.relpath(path, ROOT)
    except (OSError, KeyError, ValueError, ZeroDivisionError):
        return None, None


def cpu_reference(wl, columns, threads, seed_cols_offset=0):
    """Time the oracle port of HessianOperator::apply_block (the reference's column
    fan-out over std::thread, threads.cpp:25-44) on `columns` sketch columns."""
    from oracle import oracle as O
    o = O.HessianOperator(
        O.LinearizedModel(wl.model.kind, wl.model.n, wl.model.N, wl.model.substeps, wl.model.courant,
                          wl.model.diffusion),
        O.ObservationNetwork(wl.net.n, wl.net.N, wl.net.space_stride, wl.net.time_stride,
                             list(wl.net.times), list(wl.net.points), wl.net.q),
        O.CovarianceFactor(wl.b_half.half, wl.b_half.half_inv),
        O.CovarianceFactor(wl.q_half.half, wl.q_half.half_inv), wl.sigma_obs, threads=threads)
    V = O.gaussian_matrix(o.dim(), columns, 1)
    t0 = time.perf_counter()
    o.apply_block(V)
    return time.perf_counter() - t0


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    wl = build_workload()
    threads = os.cpu_count() or 1
    m = wl.m
    cols = min(m, max(8, 2 * threads))
    for _ in range(args.warmup):
        cpu_reference(wl, cols, threads)
    secs = [cpu_reference(wl, cols, threads) for _ in range(args.steps)]
    total = sum(secs)
    value = cols * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded N(0,1) sketch, BASELINE configs[1] operator)",
        "config": {"workload": wl.name, "n": wl.model.n, "Nsw": wl.model.N, "substeps": wl.model.substeps,
                   "n_A": wl.dim, "sketch_columns": m, "q": wl.net.q},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{cols} of {m} sketch columns per step, oracle/wc4dvar_oracle.c "
                                   f"(reference not buildable: Eigen absent), pthread column fan-out"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def run_ours(args):
    import numpy as np
    import torch

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2101_07249_b200 as W
    from paper_2101_07249_b200 import configs

    wl = build_workload()
    m = wl.m
    op = wl.hessian(local)
    nA = op.dim()
    # this rank's columns [rank*m, (rank+1)*m) of the global sketch stream (column-major fill)
    Om = W.gaussian_matrix(nA, (rank + 1) * m, configs.OMEGA_SEED)[:, rank * m:]
    dev = torch.device("cuda", local)
    V = torch.from_numpy(np.ascontiguousarray(Om.T)).to(dev)  # (m, nA) row-major == column-major Omega
    out = torch.empty_like(V)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 256 MiB > 126 MB L2
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream

    dmma_peak = W.probe_dmma_peak(local)

    for _ in range(max(args.warmup, 3)):
        op.apply_block_dev(V, out, sp)
    torch.cuda.synchronize()

    op.profile(True)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))  # L2 flush between timed steps (excluded from step time)
            starts[i].record(stream)
            op.apply_block_dev(V, out, sp)
            ends[i].record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = sum(step_ms)
    stage_ms, calls = op.profile_read()
    op.profile(False)
    if dist:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = world * m * args.steps / (total_ms / 1e3)

    # ---- e2e: the public C-ABI with HOST buffers (pinned), H2D + D2H inside the timed region
    Vh = torch.from_numpy(np.ascontiguousarray(Om.T)).pin_memory()
    Oh = torch.empty_like(Vh).pin_memory()
    op.apply_block_host_ptr(Vh.data_ptr(), nA, m, Oh.data_ptr(), nA)
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        op.apply_block_host_ptr(Vh.data_ptr(), nA, m, Oh.data_ptr(), nA)
    e2e_s = time.perf_counter() - t0
    if dist:
        t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = world * m * args.steps / e2e_s

    # ---- roofline of the dominant kernel (the D^{1/2} DMMA GEMM)
    nA_, flops_gemm, flops_model, bytes_step = algorithmic_counts(wl, m)
    gemm_ms = (stage_ms[0] + stage_ms[2]) / (2 * max(calls, 1))
    achieved_tf = flops_gemm / (gemm_ms * 1e-3) / 1e12
    traffic, traffic_src = gemm_traffic()
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        peaks = {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    step_mean_ms = total_ms / args.steps
    clocks = clk.summary()

    extras = {}
    if not args.no_extras and rank == 0:
        extras = run_extras(W, configs, wl, op, Om, dev)
        if world == 1:
            extras["large_configs"] = run_large(W, configs, dmma_peak, hbm_peak)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_mean_ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded N(0,1) sketch from the reference NormalStream, BASELINE configs[1] operator)",
            "config": {"workload": wl.name, "n": wl.model.n, "Nsw": wl.model.N, "substeps": wl.model.substeps,
                       "n_A": nA, "sketch_columns_per_gpu": m, "q": wl.net.q, "covariance": "dense SOAR",
                       "parallelism": f"column-sharded x{world}",
                       "l2": "flushed between timed steps (256 MiB write), flush excluded from step time"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * nA * m,
                    "d2h_bytes_per_step": 8 * nA * m},
            "gpu_launches": 3 * args.steps,
            "roofline": {"bound": "tensor", "achieved": achieved_tf, "peak": dmma_peak, "unit": "TFLOP/s",
                         "frac": achieved_tf / dmma_peak, "traffic": traffic,
                         "traffic_source": traffic_src,
                         "kernel": "gemm_sym_ws_kernel (D^1/2 block-diagonal DMMA GEMM, stream-K)",
                         "flops_per_launch": flops_gemm, "launch_ms": gemm_ms,
                         "peak_source": "measured in this run: all-SM mma.sync.f64 probe "
                                        "(MEASURED_PEAKS.json has bf16/HBM only)"},
            "hbm_roofline": {"bytes_per_step": bytes_step, "achieved_gbs": bytes_step / (step_mean_ms * 1e-3) / 1e9,
                             "peak_gbs": hbm_peak, "frac": bytes_step / (step_mean_ms * 1e-3) / 1e9 / hbm_peak,
                             "note": "C2 is fp64-compute bound (dense D^1/2 is 99% of flops)"},
            "stage_ms": {"d_half_in": stage_ms[0] / max(calls, 1), "sweep": stage_ms[1] / max(calls, 1),
                         "d_half_out_plus_identity": stage_ms[2] / max(calls, 1)},
            "clocks": clocks,
        }
        line.update(extras)
        if world == 1:
            threads = os.cpu_count() or 1
            cols = min(m, max(8, 2 * threads))
            secs = cpu_reference(wl, cols, threads)
            line["cpu_baseline"] = {"value": cols / secs, "unit": UNIT, "cores": threads, "kind": "port",
                                    "sample": f"{cols} of {m} sketch columns, oracle/wc4dvar_oracle.c "
                                              f"(reference not buildable: Eigen absent), pthread column fan-out"}
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    return 0


def run_extras(W, configs, wl, op, Om, dev):
    """LMP build ms per method (Omega resident on device -> U, Theta on device) and
    LMP-PCG time/iterations on the same operator."""
    import numpy as np
    import torch
    out = {"lmp_build_ms": {}, "lmp_build_stage_ms": {}, "pcg": {}}
    nA = op.dim()
    k, l = wl.k, wl.m - wl.k
    pairs = {}
    for method in ("revd", "nystrom", "ritzit"):
        cfg = W.SketchConfig(k, l, configs.OMEGA_SEED, method, 1)
        W.sketch_eigenpairs(op, cfg, Om)  # warm (grows the sketch workspaces)
        pairs[method] = W.sketch_eigenpairs(op, cfg, Om)
        t = W.last_sketch_timing()  # the second, warm call
        out["lmp_build_ms"][method] = t["total_ms"]
        out["lmp_build_stage_ms"][method] = {kk: v for kk, v in t.items() if kk != "total_ms"}
    b = W.gaussian_matrix(nA, 1, configs.RHS_SEED)[:, 0]
    for method in ("none", "revd", "nystrom", "ritzit"):
        f = None if method == "none" else W.build_spectral_lmp(pairs[method])
        t0 = time.perf_counter()
        r = W.pcg_split(op, b, f, opts=W.PcgOptions(max_iter=500, rel_tol=1e-6))
        out["pcg"][method] = {"ms": 1e3 * (time.perf_counter() - t0), "iterations": r.history.iterations,
                              "converged": r.history.converged}
    return out


def run_large(W, configs, peak_tfs, hbm_gbs):
    """BASELINE configs[2] (C3, Lorenz-96 n=1e5), configs[3] (C4, adv-diff n=1e6, circulant
    factors) block applies at m = 64 and configs[4] (C5, Lorenz-96 n=2e6, Nsw=20) at one
    rank's 32-column share of its 8-GPU sketch, on one GPU: device-drawn N(0,1) Omega (torch,
    throughput only; parity at these shapes is property-based in tests/), CUDA-event timing,
    per-stage split, and the SURVEY §8(d) roofline t_roof = max(B/BW, F/P) per block with
    B = 8 (3 n_A + 2 q) m and F = (F_model + F_cov) m."""
    import torch
    out = {}
    for name, mk in (("C3", lambda: configs.config3()), ("C4", lambda: configs.config4(64)),
                     ("C5", lambda: configs.config5(32))):
        try:
            wl = mk()
            t0 = time.perf_counter()
            op = wl.hessian(0)
            setup_s = time.perf_counter() - t0
            m, nA, q = wl.m, op.dim(), wl.net.q  # C5: one rank's 32-column share of the 8-GPU sketch
            n, N, s = wl.model.n, wl.model.N, wl.model.substeps
            g = torch.Generator(device="cuda").manual_seed(1)
            V = torch.randn(m, nA, dtype=torch.float64, device="cuda", generator=g)
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
            ms = e0.elapsed_time(e1) / reps
            st, calls = op.profile_read()
            op.profile(False)
            f_model = (92.0 if wl.model.kind == "l96" else 10.0) * N * s * n
            f_cov = 2.0 * (N + 1) * (5.0 * n * math.log2(n) + n)
            t_f = (f_model + f_cov) * m / (peak_tfs * 1e12)
            t_b = 8.0 * (3 * nA + 2 * q) * m / (hbm_gbs * 1e9)
            t_roof = max(t_f, t_b) * 1e3
            out[name] = {"workload": wl.name, "m": m, "ms_per_apply": ms, "columns_per_s": m / (ms * 1e-3),
                         "stage_ms": {"d_half_in": st[0] / max(calls, 1), "sweep": st[1] / max(calls, 1),
                                      "d_half_out_plus_identity": st[2] / max(calls, 1)},
                         "roofline": {"t_roof_ms": t_roof, "bound": "fp64" if t_f >= t_b else "hbm",
                                      "frac": t_roof / ms},
                         "operator_setup_s": setup_s, "omega": "device N(0,1) (torch), seed 1"}
            del V, Y, op
            torch.cuda.empty_cache()
        except Exception as e:  # report, do not fail the headline line
            out[name] = {"error": f"{type(e).__name__}: {e}"[:300]}
    return out


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
