"""Per-kernel summary of an ncu --set full report: duration, pipe utilisation, top stalls and
the dynamic SASS opcode mix (per `unit` work items if given):
    python tools/ncu_mix.py rep.ncu-rep [units_per_kernel]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h = r[0]
for row in r[2:]:
    d = dict(zip(h, row))
    print(d["Kernel Name"][:90], "| us", d.get("gpu__time_duration.sum"), "| regs", d.get("launch__registers_per_thread"))
    for k in ["sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
              "l1tex__throughput.avg.pct_of_peak_sustained_active", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active"]:
        print("   %-70s %s" % (k, d.get(k)))
    st = []
    for k in h:
        if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
            try:
                st.append((float(d[k]), k[34:-23]))
            except ValueError:
                pass
    print("   stalls:", ", ".join(f"{n}={c:.2f}" for c, n in sorted(st, reverse=True)[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
blocks, cur = [], []
for row in rows:
    if row and row[0] == "Kernel Name":
        if cur:
            blocks.append(cur)
        cur = [row]
    else:
        cur.append(row)
blocks.append(cur)
seen = set()
for bl in blocks:
    name = bl[0][1] if len(bl[0]) > 1 else "?"
    if name in seen:
        continue
    seen.add(name)
    hdr = None
    for i, row in enumerate(bl):
        if row and row[0] == "Address":
            hdr, start = row, i + 1
            break
    if hdr is None:
        continue
    ie = hdr.index("Instructions Executed")
    c = Counter()
    for row in bl[start:]:
        if len(row) != len(hdr):
            continue
        t = row[1].strip().split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") else t[0]
        c[op.split(".")[0]] += int(row[ie] or 0)
    tot = sum(c.values())
    scale = 32.0 / units if units else 1.0 / max(tot, 1)
    print(name[:90], "| warp instr", tot)
    print("   " + ", ".join(f"{op} {n * scale:.2f}" for op, n in c.most_common(24)))
