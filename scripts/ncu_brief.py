"""Brief per-kernel summary of an ncu report: python scripts/ncu_brief.py rep.ncu-rep"""
import csv
import subprocess
import sys

WANT = ["Duration", "Executed Instructions", "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy",
        "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Warp Cycles Per Issued Instruction", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
cur = None
for r in rows[1:]:
    if r[mi] in WANT:
        if r[ki] != cur:
            cur = r[ki]
            print(cur)
        print(f"   {r[mi]:<64} {r[vi]:>14} {r[ui]}")
