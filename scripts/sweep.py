"""Config 4: candidate-parallel sweep of the reference sampler's 256 kernels.

    python scripts/sweep.py [--count 256] [--gpus N] [--out sweep.json]

One worker process per GPU (replicas only, no collective).  Each worker plans,
compiles and times fwd+bwd of a kernel at config-1 shapes (N=8, C=64, 56^2,
G=4, K=3).  The kernels are drawn by the sampler mirror,
Sampler(SamplerConfig(nodes=10, seed=7)).sample_many(256) by default — the
same texts the reference emits (tests/golden/sampler_10_7_256.cir, sha256
f1638a90...; checked before the sweep when that config is used).
Free variables are solved proportionally (x := smallest legal multiple >= C).
"""

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2304_07741_b200.evaluator import CandidateEvaluator  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--count", type=int, default=256)
    ap.add_argument("--gpus", type=int, default=0)
    ap.add_argument("--out", default="")
    ap.add_argument("--nodes", type=int, default=10)
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--prefetch", type=int, default=-1, help="kernels compiled ahead per worker on host threads (-1: host cores per GPU - 1, max 8)")
    a = ap.parse_args()
    import torch

    n = a.gpus or torch.cuda.device_count()
    from paper_2304_07741_b200.canvas import ir
    from paper_2304_07741_b200.canvas.sampler import Sampler, SamplerConfig

    texts = [ir.emit(k) for k in Sampler(SamplerConfig(nodes=a.nodes, seed=a.seed)).sample_many(a.count)]
    golden = os.path.join(ROOT, f"tests/golden/sampler_{a.nodes}_{a.seed}_{a.count}.cir")
    if os.path.exists(golden):
        assert "".join(texts) == open(golden).read(), "sampler mirror diverged from the reference golden"
    t0 = time.perf_counter()
    pf = a.prefetch if a.prefetch >= 0 else min(8, max(1, (os.cpu_count() or 2) // max(n, 1) - 1))
    res = CandidateEvaluator(list(range(n)), prefetch=pf).run(texts)
    wall = time.perf_counter() - t0
    ok = [r for r in res if r.status == "ok"]
    lat = [r.fwd_ms + r.bwd_ms for r in ok]
    summary = {
        "metric": "candidate kernels evaluated/s (plan+compile+fwd/bwd timing), config-1 shapes",
        "value": round(len(res) / wall, 3),
        "unit": "kernels/s",
        "n_gpus": n,
        "kernels": len(res),
        "ok": len(ok),
        "nonfinite": sum(r.status == "nonfinite" for r in res),
        "failed": sum(r.status == "failed" for r in res),
        "wall_s": round(wall, 2),
        "compile_ahead": pf,
        "fwd_bwd_ms_median": round(statistics.median(lat), 4) if lat else None,
        "fwd_bwd_ms_p90": round(sorted(lat)[int(0.9 * (len(lat) - 1))], 4) if lat else None,
        "timing": "CUDA-graph replay per (plan, direction); eager launches in fwd_bwd_ms_eager_*",
        "fwd_bwd_ms_eager_median": round(statistics.median(r.extra.get("fwd_ms_eager", 0) + r.extra.get("bwd_ms_eager", 0) for r in ok), 4) if ok else None,
        "launches_fwd_bwd_median": statistics.median(r.extra.get("launches_fwd", 0) + r.extra.get("launches_bwd", 0) for r in ok) if ok else None,
        "plan_ms_median": round(statistics.median(r.plan_ms for r in res if r.plan_ms), 1) if ok else None,
        "errors": sorted({r.error[:120] for r in res if r.error})[:10],
    }
    print(json.dumps(summary))
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"summary": summary, "results": [r.as_dict() for r in res]}, f)


if __name__ == "__main__":
    main()
