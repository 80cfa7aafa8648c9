"""Top stall-sampled SASS instructions of the first kernel in an ncu report:
    python tools/sass_hotspots.py rep.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    if len(r) == len(hdr):
        data.append(r)
i_s = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[i_s]) for r in data)
print("kernel:", rows[0][1][:100], "| samples", tot, "| instructions", len(data))
stall_cols = [j for j, h in enumerate(hdr) if h.startswith("stall_")]
top = sorted(range(len(data)), key=lambda k: -int(data[k][i_s]))[:ntop]
for k in sorted(top):
    r = data[k]
    st = sorted(((int(r[j]) if r[j].isdigit() else 0, hdr[j][6:]) for j in stall_cols), reverse=True)[:2]
    print(f"{k:5d} {r[1].strip()[:64]:64s} {int(r[i_s]) / tot * 100:5.1f}% {st}")
