"""Turn raw gpurun_out/ captures into the tracked summaries under profiles/.

    python scripts/profiles_update.py <tag> <ncu_full.ncu-rep> <launches.csv> [bench.json]

Writes profiles/<tag>_ncu_full.{json,txt} (per-kernel SOL / occupancy / dram
bytes / tensor-pipe %), profiles/<tag>_launches_summary.txt (share of device
time per kernel from the --metrics gpu__time_duration.sum launch list) and
profiles/dominant_traffic.json (dram read+write bytes per launch of each
profiled Canvas kernel at batch 256, consumed by bench.py's roofline.traffic).
"""
import collections
import csv
import json
import os
import re
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))
from ncu_summary import summary  # noqa: E402


TRAFFIC_KEY = os.environ.get("TRAFFIC_KEY", "seed7_k1|resnet18|64x64@56x56/s1|b256")


def main():
    tag, rep, launches = sys.argv[1:4]
    bench = sys.argv[4] if len(sys.argv) > 4 else None
    out = os.path.join(ROOT, "profiles")
    os.makedirs(out, exist_ok=True)
    s = summary(rep)
    json.dump(s, open(os.path.join(out, f"{tag}_ncu_full.json"), "w"), indent=1)
    with open(os.path.join(out, f"{tag}_ncu_full.txt"), "w") as f:
        f.write(f"ncu --set full --clock-control none (scripts/kbench.py layer1 seed7_k1 64->64 56^2 batch 256), source {os.path.basename(rep)}\n")
        for k, d in s.items():
            f.write(k + "\n")
            for m, v in d.items():
                f.write(f"   {m:62s} {v}\n")
    traffic_path = os.path.join(out, "dominant_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for k, d in s.items():
        rd = float(d.get("dram__bytes_read.sum", "0 byte").split()[0]) * _unit(d.get("dram__bytes_read.sum", "0 byte"))
        wr = float(d.get("dram__bytes_write.sum", "0 byte").split()[0]) * _unit(d.get("dram__bytes_write.sum", "0 byte"))
        inst = d.get("Executed Instructions", "0 inst").split()[0].replace(",", "")
        # keyed by the workload that produced the counters (bench.traffic_key): the
        # capture is the ResNet-18 layer1 target of config 2 (seed-7 #1, 64x64 @ 56x56, b256)
        traffic.setdefault(TRAFFIC_KEY, {})[k.split("_", 1)[1]] = {"batch": 256, "dram_bytes": int(rd + wr), "warp_instructions": int(float(inst)), "source": f"profiles/{tag}_ncu_full.json"}
    traffic.pop("seed7_k1", None)  # pre-workload-key format
    json.dump(traffic, open(traffic_path, "w"), indent=1)
    rows = list(csv.reader(open(launches)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hi], rows[hi + 1 :]
    # drop the warm-up steps (cuDNN autotuner trials) — keep the last 3 steps' launches
    per_step = int(os.environ.get("LAUNCHES_PER_STEP", "0"))
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    if per_step:
        data = data[-3 * per_step :]
    elif os.environ.get("STEP_MARKER"):  # "<kernel name>:<launches per step>": keep the last 3 steps
        name, cnt = os.environ["STEP_MARKER"].rsplit(":", 1)
        pos = [i for i, r in enumerate(data) if r[ki] == name]
        if len(pos) >= 3 * int(cnt):
            data = data[pos[len(pos) - 3 * int(cnt)] :]
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = canvas = 0.0
    for r in data:
        v = float(r[vi].replace(",", ""))
        tot += v
        if re.match(r"k\d+_(fwd|bwd)", r[ki]):
            canvas += v
        agg[re.sub(r"^k\d+_", "", r[ki])[:90]][0] += 1
        agg[re.sub(r"^k\d+_", "", r[ki])[:90]][1] += v
    with open(os.path.join(out, f"{tag}_launches_summary.txt"), "w") as f:
        f.write("ncu --metrics gpu__time_duration.sum --clock-control none -- python bench.py --steps 1 --warmup 3 --no-cpu --no-context\n")
        f.write("(cold-cache, serialised per-launch times of the CUDA-graph kernel nodes; warm-up steps dropped, last timed + 2 e2e steps kept: compare SHARES, not absolutes)\n")
        f.write(f"total {tot / 1e6:.1f} ms over {len(data)} launches; Canvas kernels {100 * canvas / tot:.1f}% of device time\n\n")
        for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:45]:
            f.write(f"{100 * v / tot:6.2f}% {n:5d} launches {v / n / 1e3:9.1f} us/launch  {k}\n")
    if bench:
        shutil.copy(bench, os.path.join(out, f"{tag}_bench.json"))


def _unit(s):
    u = s.split()[-1] if " " in s else "byte"
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


if __name__ == "__main__":
    main()
