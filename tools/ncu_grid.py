"""Per (kernel, grid) breakdown of an ncu launch list (gpu__time_duration.sum CSV).

    python tools/ncu_grid.py gpurun_out/launches.csv [top]
"""
import csv
import sys
from collections import defaultdict

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = [r for r in csv.DictReader(lines) if r["Metric Name"] == "gpu__time_duration.sum"]
d = defaultdict(list)
for r in rows:
    n = r["Kernel Name"].split("(")[0].replace("void ", "")
    d[(n, r["Grid Size"])].append(float(r["Metric Value"].replace(",", "")) / 1000)
tot = sum(sum(v) for v in d.values())
print(f"{len(rows)} launches, {tot / 1e3:.3f} ms")
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1]))[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print("%-44s %-14s %4d %9.1f us %9.1f us %5.1f%%" % (k[0][:44], k[1], len(v), sum(v) / len(v), sum(v),
                                                         100 * sum(v) / tot))
