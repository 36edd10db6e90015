"""Side-by-side table of `ncu --page details --csv` exports: python tools/ncu_details.py a.csv [b.csv ...]"""
import csv
import sys

SECTIONS = ("GPU Speed Of Light Throughput", "Compute Workload Analysis", "Occupancy", "Warp State Statistics",
            "Memory Workload Analysis", "Launch Statistics", "Scheduler Statistics", "Instruction Statistics")


def load(fn):
    d, order = {}, []
    rows = list(csv.reader(open(fn)))
    hdr = rows[0]
    for r in rows[1:]:
        rec = dict(zip(hdr, r))
        k = (rec.get("Section Name", ""), rec.get("Metric Name", ""))
        if k not in d:
            order.append(k)
        d[k] = rec.get("Metric Value", "")
        d["__kernel"] = rec.get("Kernel Name", "")
    return d, order


tabs = [load(f) for f in sys.argv[1:]]
for i, (t, _) in enumerate(tabs):
    print(f"[{i}] {t['__kernel'][:100]}")
for k in tabs[0][1]:
    if k[0] in SECTIONS and k[1]:
        print("%-28s %-44s" % (k[0][:28], k[1][:44]) + "".join("%16s" % t.get(k, "")[:16] for t, _ in tabs))
