"""Summarises an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel.

    python tools/ncu_summary.py gpurun_out/launches.csv [--skip N]
"""
import csv
import re
import sys
from collections import defaultdict


def short(name):
    name = re.sub(r"\(anonymous namespace\)::", "", name)
    name = name.replace("gmg_dev::", "")
    return name[:150]


def main(path, skip=0):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.DictReader(lines)
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(unit, 1e-3)
        rows.append((short(r["Kernel Name"]), v * scale))
    rows = rows[skip:]
    tot = sum(t for _, t in rows)
    agg = defaultdict(lambda: [0, 0.0])
    for k, t in rows:
        agg[k][0] += 1
        agg[k][1] += t
    print(f"{len(rows)} launches, {tot/1e3:.3f} ms total (serialised, cold-cache)")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:40]:
        print(f"{t/1e3:9.3f} ms {100*t/tot:5.1f}%  {c:5d}x  {t/c:9.2f} us  {k}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
