"""Summarise an ncu report (``--set full`` capture) into a small JSON + Markdown pair under
profiles/: per kernel launch the duration, DRAM bytes (traffic), tensor / fp64 pipe
activity, occupancy, registers and the top warp-stall reasons.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_gemm
"""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_active_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}
UNITS = {"dram_read": None, "dram_write": None}


def to_bytes(val: str, unit: str) -> float:
    f = float(val.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return f * scale.get(unit, 1)


def main(rep, out_prefix):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for row in rows[2:]:
        if len(row) != len(hdr):
            continue
        k = {"kernel": row[hdr.index("Kernel Name")][:120]}
        for name, key in WANT.items():
            if name in hdr:
                i = hdr.index(name)
                try:
                    if key.startswith("dram_r") or key.startswith("dram_w"):
                        k[key] = to_bytes(row[i], units[i])
                    elif key == "duration_us":
                        v = float(row[i].replace(",", ""))
                        scale = {"nsecond": 1e-3, "ns": 1e-3, "msecond": 1e3, "ms": 1e3, "second": 1e6,
                                 "s": 1e6}
                        k[key] = v * scale.get(units[i], 1.0)
                    else:
                        k[key] = float(row[i].replace(",", ""))
                except ValueError:
                    k[key] = row[i]
        stalls = {}
        for name, val in zip(hdr, row):
            if name.startswith("smsp__average_warps_issue_stalled_") and name.endswith("_per_issue_active.ratio"):
                try:
                    stalls[name[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(val)
                except ValueError:
                    pass
        k["top_stalls"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:5])
        if "dram_read" in k and "dram_write" in k:
            k["traffic_bytes"] = k["dram_read"] + k["dram_write"]
        kernels.append(k)
    json.dump({"report": rep, "kernels": kernels}, open(out_prefix + ".json", "w"), indent=1)
    with open(out_prefix + ".md", "w") as f:
        f.write(f"# ncu summary of `{rep}`\n\n")
        f.write("| kernel | us | DRAM MB | tensor % | fp64 % | occ % | regs | top stalls |\n|---|---|---|---|---|---|---|---|\n")
        for k in kernels:
            f.write(f"| {k['kernel'][:60]} | {k.get('duration_us', 0):.1f} | {k.get('traffic_bytes', 0) / 1e6:.1f} | "
                    f"{k.get('tensor_active_pct', 0):.1f} | {k.get('fp64_active_pct', 0):.1f} | "
                    f"{k.get('achieved_occupancy_pct', 0):.1f} | {k.get('registers', 0):.0f} | "
                    f"{', '.join(f'{a}={b:.2f}' for a, b in k['top_stalls'].items())} |\n")
    print(open(out_prefix + ".md").read())


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
