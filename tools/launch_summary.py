"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel:
    python tools/launch_summary.py launches.csv out.md "title" [share-kernel-regex]
Shares are of the summed time of the kernels matching the regex (the apply's kernels)."""
import csv
import re
import sys
from collections import OrderedDict

src, out, title = sys.argv[1], sys.argv[2], sys.argv[3]
pat = re.compile(sys.argv[4]) if len(sys.argv) > 4 else None
rows = [r for r in csv.reader(open(src)) if len(r) > 14 and r[0].isdigit()]
agg = OrderedDict()
for r in rows:
    name = r[4]
    short = re.sub(r"\(.*", "", name.replace("void ", ""))[:70]
    t = float(r[14].replace(",", "")) / (1000.0 if r[13] == "ns" else 1.0)
    a = agg.setdefault(short, [0, 0.0, name])
    a[0] += 1
    a[1] += t
tot = sum(v[1] for k, v in agg.items() if pat and pat.search(k)) or 1.0
with open(out, "w") as f:
    f.write(f"# {title}\n\nRaw list: `{src.split('/')[-1]}`.  Times are ncu's serialised, cold-cache "
            "launch durations: compare SHARES, not absolutes, with the bench line.\n\n")
    f.write("| kernel | launches | total us | share of apply kernels |\n|---|---|---|---|\n")
    for k, (n, t, _) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        share = f"{100 * t / tot:.1f} %" if pat and pat.search(k) else ""
        f.write(f"| `{k}` | {n} | {t:.1f} | {share} |\n")
print(open(out).read())
