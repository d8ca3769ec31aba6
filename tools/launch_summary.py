"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel launches, total time and share.  Usage:
python tools/launch_summary.py launches.csv[.gz] > summary.txt"""
import csv
import gzip
import re
import sys
from collections import defaultdict

path = sys.argv[1]
op = gzip.open if path.endswith(".gz") else open
with op(path, "rt") as f:
    lines = [ln for ln in f if ln.startswith('"')]
rows = list(csv.reader(lines))
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
ui = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[1:]:
    if len(r) <= max(ki, mi, vi) or r[mi] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ki])
    name = re.sub(r"^(void )?(hydot::)?(\(anonymous namespace\)::|<unnamed>::)?", "", name)
    v = float(r[vi].replace(",", ""))
    unit = r[ui] if ui is not None else "ns"
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
    tot[name] += v * scale
    cnt[name] += 1
T = sum(tot.values())
print(f"total {T:.1f} ms over {sum(cnt.values())} launches")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k[:52]:52s} {cnt[k]:7d} {tot[k]:10.2f} ms {100 * tot[k] / T:5.1f}%")
