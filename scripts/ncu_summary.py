"""Summarise an ncu report (details page) into the metrics we track: prints
and optionally writes JSON.  Usage: python scripts/ncu_summary.py rep.ncu-rep [out.json]"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["Duration", "SM Frequency", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput", "Compute (SM) Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy", "No Eligible", "Warp Cycles Per Issued Instruction", "Registers Per Thread", "Dynamic Shared Memory Per Block", "Achieved Occupancy", "Theoretical Occupancy", "Grid Size", "Block Size", "Executed Instructions"]


def summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ni, vi, ui, ki = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("Kernel Name")
    res = {}
    for r in rows[1:]:
        k = r[ki]
        d = res.setdefault(k, {})
        if r[ni] in KEYS:
            d[r[ni]] = f"{r[vi]} {r[ui]}".strip()
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) > 2:
        hh = rr[0]
        for row in rr[2:]:
            k = row[hh.index("Kernel Name")]
            for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_tc.sum"):
                for i, name in enumerate(hh):
                    if name.startswith(m):
                        res.setdefault(k, {})[name] = f"{row[i]} {rr[1][i]}".strip()
    return res


if __name__ == "__main__":
    r = summary(sys.argv[1])
    for k, d in r.items():
        print(k)
        for m, v in d.items():
            print(f"   {m:60s} {v}")
    if len(sys.argv) > 2:
        json.dump(r, open(sys.argv[2], "w"), indent=1)
