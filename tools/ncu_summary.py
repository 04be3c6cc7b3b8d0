#!/usr/bin/env python3
"""Summarise ncu reports / launch lists into profiles/ (run here, on the CPU box).

  python tools/ncu_summary.py <report.ncu-rep> <out.json> [algorithmic_bytes] [flops]
  python tools/ncu_summary.py --launches <launches.csv> <out.json>
"""
import collections
import csv
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_bytes_read",
    "dram__bytes_write.sum": "dram_bytes_write",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "memory_throughput_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9,
              "msecond": 1e6, "second": 1e9}


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    res = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else None}
    for k, name in KEYS.items():
        if k in hdr:
            i = hdr.index(k)
            try:
                v = float(vals[i].replace(",", ""))
            except ValueError:
                continue
            res[name] = v * UNIT_SCALE.get(units[i], 1)
    stalls = {}
    for i, k in enumerate(hdr):
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(vals[i])
            except ValueError:
                pass
    res["top_stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda x: -x[1])[:6])
    if "dram_bytes_read" in res:
        res["dram_bytes_per_launch"] = res["dram_bytes_read"] + res.get("dram_bytes_write", 0)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    iK, iV = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        if len(r) > iV:
            try:
                v = float(r[iV].replace(",", ""))
            except ValueError:
                continue
            k = r[iK].split("(")[0]
            agg[k][0] += 1
            agg[k][1] += v
    tot = sum(t for _, t in agg.values())
    return {"total_ns": tot, "kernels": [{"kernel": k, "launches": n, "ns": t, "share": t / tot}
                                         for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])]}


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        res = launches(sys.argv[2])
        out = sys.argv[3]
    else:
        res = raw(sys.argv[1])
        out = sys.argv[2]
        if len(sys.argv) > 3:
            alg = float(sys.argv[3])
            res["algorithmic_bytes_per_launch"] = alg
            if "dram_bytes_per_launch" in res:
                res["traffic_over_algorithmic"] = res["dram_bytes_per_launch"] / alg
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1)[:1500])
