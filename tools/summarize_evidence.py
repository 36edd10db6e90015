"""Summarises `ncu --set full` exports (tools/ncu_capture.sh) into compact JSON files
under profiles/: python tools/summarize_evidence.py <prefix> name [name ...]
reads gpurun_out/<name>.details.csv and .raw.csv, writes profiles/<name>_full_summary.json."""
import csv
import json
import os
import sys

KEYS = [("GPU Speed Of Light Throughput", "Duration"), ("GPU Speed Of Light Throughput", "DRAM Throughput"),
        ("GPU Speed Of Light Throughput", "Memory Throughput"), ("GPU Speed Of Light Throughput", "SM Frequency"),
        ("Compute Workload Analysis", "Issue Slots Busy"), ("Compute Workload Analysis", "Executed Ipc Active"),
        ("Memory Workload Analysis", "L2 Hit Rate"), ("Occupancy", "Achieved Occupancy"),
        ("Occupancy", "Theoretical Occupancy"), ("Launch Statistics", "Registers Per Thread"),
        ("Launch Statistics", "Grid Size"), ("Launch Statistics", "Block Size"),
        ("Launch Statistics", "Waves Per SM"), ("Warp State Statistics", "Warp Cycles Per Issued Instruction"),
        ("Instruction Statistics", "Executed Instructions")]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_wait",
       "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle", "smsp__pcsamp_warps_issue_stalled_barrier",
       "smsp__pcsamp_warps_issue_stalled_branch_resolving", "smsp__pcsamp_warps_issue_stalled_no_instructions",
       "smsp__pcsamp_warps_issue_stalled_mio_throttle", "smsp__pcsamp_warps_issue_stalled_lg_throttle",
       "smsp__pcsamp_warps_issue_stalled_short_scoreboard", "smsp__pcsamp_warps_issue_stalled_not_selected",
       "smsp__pcsamp_warps_issue_stalled_selected", "smsp__pcsamp_warps_issue_stalled_sleeping"]


def details(fn):
    out, kernel = {}, ""
    rows = list(csv.reader(open(fn)))
    hdr = rows[0]
    for r in rows[1:]:
        rec = dict(zip(hdr, r))
        kernel = rec.get("Kernel Name", kernel)
        k = (rec.get("Section Name"), rec.get("Metric Name"))
        if k in KEYS:
            out[f"{k[1]} [{rec.get('Metric Unit', '')}]"] = rec.get("Metric Value")
    return kernel, out


def raw(fn):
    rows = list(csv.reader(open(fn)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    return {f"{k} [{u.get(k, '')}]": d[k] for k in RAW if k in d}


for name in sys.argv[1:]:
    kern, det = details(f"gpurun_out/{name}.details.csv")
    rw = raw(f"gpurun_out/{name}.raw.csv")
    obj = {"kernel": kern, "capture": "ncu --set full --clock-control none --import-source on (tools/ncu_capture.sh)",
           "details": det, "raw": rw}
    path = os.path.join("profiles", f"{name}_full_summary.json")
    json.dump(obj, open(path, "w"), indent=1)
    print("wrote", path)
