"""profiles/traffic_r02.json from an ncu --set full raw CSV export: per
kernel class, the mean dram__bytes_read.sum + dram__bytes_write.sum per
launch and the mean algorithmic bytes of the same launches (GEMM: 8 (mk +
kn + mn) from the grid / args is not in the CSV, so only DRAM bytes and
duration are recorded, with the launch names).
Usage: python tools/traffic_from_ncu.py raw.csv[.gz] class=regex ..."""
import csv
import gzip
import json
import re
import sys


SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "ns": 1.0, "us": 1e3, "ms": 1e6}


def rows(path):
    """raw-page CSV: header row, units row, one row per launch; values scaled
    to bytes / nanoseconds"""
    op = gzip.open if path.endswith(".gz") else open
    with op(path, "rt") as f:
        r = list(csv.reader(f))
    head, units = r[0], r[1]
    out = []
    for x in r[2:]:
        if len(x) != len(head):
            continue
        d = {}
        for h, u, v in zip(head, units, x):
            sc = SCALE.get(u.strip())
            if sc is not None:
                try:
                    d[h] = float(v.replace(",", "")) * sc
                    continue
                except ValueError:
                    pass
            d[h] = v
        out.append(d)
    return out


def num(v):
    if isinstance(v, float):
        return v
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def main():
    src = sys.argv[1]
    classes = dict(a.split("=", 1) for a in sys.argv[2:])
    data = rows(src)
    out = {}
    for cls, rx in classes.items():
        sel = [d for d in data if re.search(rx, d.get("Kernel Name", ""))]
        if not sel:
            continue
        rd = [num(d.get("dram__bytes_read.sum")) for d in sel]
        wr = [num(d.get("dram__bytes_write.sum")) for d in sel]
        du = [num(d.get("gpu__time_duration.sum")) for d in sel]
        tot = [a + b for a, b in zip(rd, wr) if a is not None and b is not None]
        out[cls] = {"dram_bytes_per_launch": sum(tot) / len(tot) if tot else None,
                    "launches": len(sel), "mean_duration_ns": sum(x for x in du if x) / len(sel),
                    "kernels": sorted({d.get("Kernel Name", "")[:80] for d in sel}),
                    "source": src.split("/")[-1]}
    json.dump(out, sys.stdout, indent=1)


if __name__ == "__main__":
    main()
