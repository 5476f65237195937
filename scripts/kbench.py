"""Per-launch timing of one replaced conv layer (fwd + bwd) on the GPU.

    python scripts/kbench.py [--kernel seed7_k1] [--cin 64 --cout 64 --hw 56 --stride 1] [--batch 256] [--json out.json]

Every launch record of the plan is timed with CUDA events recorded by
libcanvas around that launch (canvas_plan_profile), averaged over --iters
fwd+bwd passes; prints achieved GB/s (algorithmic bytes) and TFLOP/s (useful
FC FLOPs) per kernel next to the measured peaks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2304_07741_b200 import zoo  # noqa: E402
from paper_2304_07741_b200.executor import device_plan, plan_for  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernel", default="seed7_k1")
    ap.add_argument("--cin", type=int, default=64)
    ap.add_argument("--cout", type=int, default=64)
    ap.add_argument("--hw", type=int, default=56)
    ap.add_argument("--stride", type=int, default=1)
    ap.add_argument("--k", type=int, default=3, help="replaced conv kernel size (KH = KW)")
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--json", default="")
    ap.add_argument("--no-tc", action="store_true")
    a = ap.parse_args()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    pk2 = os.path.join(ROOT, "profiles", "r02_peaks.json")
    tf32_peak = json.load(open(pk2))["tf32_tcgen05_tflops_sustained"] if os.path.exists(pk2) else peaks["bf16_tflops"] / 2
    text = zoo.ALL.get(a.kernel) or open(a.kernel).read()
    if a.no_tc:
        from paper_2304_07741_b200.executor import solve_target
        from paper_2304_07741_b200.graph import build_graph
        from paper_2304_07741_b200.lowering import lower

        t, asg = solve_target(text, c_in=a.cin, c_out=a.cout, h=a.hw, w=a.hw, k=a.k, stride=a.stride)
        plan = lower(build_graph(t, asg), c_in=a.cin, c_out=a.cout, stride=a.stride, h_in=a.hw, w_in=a.hw, use_tc=False)
    else:
        plan = plan_for(text, c_in=a.cin, c_out=a.cout, h=a.hw, w=a.hw, k=a.k, stride=a.stride)
    dp = device_plan(plan, 0)
    dev = torch.device("cuda:0")
    n = a.batch
    ho = -(-a.hw // a.stride)
    x = torch.randn(n, a.cin, a.hw, a.hw, device=dev)
    ws = [torch.randn(o, k, device=dev) / k**0.5 for _ in range(plan.copies) for (o, k) in (plan.graph.fc_shape(v) for v in plan.graph.fc_nodes)]
    y = torch.empty(n, a.cout, ho, ho, device=dev)
    sb, wb = dp.sizes(n)
    saved = torch.empty(max(sb, 1), dtype=torch.uint8, device=dev)
    work = torch.empty(max(wb, 1), dtype=torch.uint8, device=dev)
    dy = torch.randn_like(y)
    dx = torch.empty_like(x)
    dws = [torch.empty_like(w) for w in ws]
    st = torch.cuda.current_stream().cuda_stream

    def step():
        dp.forward(x, ws, y, saved, st)
        dp.backward(x, ws, saved, dy, dx, dws, work, st)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    # whole-layer time
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        step()
    e1.record()
    torch.cuda.synchronize()
    layer_ms = e0.elapsed_time(e1) / a.iters
    # the same fwd+bwd captured once as a CUDA graph and replayed (no host launch
    # overhead: the figure that matters at small batch, e.g. config 1 at N = 8)
    g = torch.cuda.CUDAGraph()
    s_cap = torch.cuda.Stream()
    s_cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s_cap):
        st_cap = s_cap.cuda_stream
        dp.forward(x, ws, y, saved, st_cap)
        dp.backward(x, ws, saved, dy, dx, dws, work, st_cap)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s_cap):
            dp.forward(x, ws, y, saved, st_cap)
            dp.backward(x, ws, saved, dy, dx, dws, work, st_cap)
    torch.cuda.synchronize()
    for _ in range(3):
        g.replay()
    e0.record()
    for _ in range(a.iters * 4):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    graph_ms = e0.elapsed_time(e1) / (a.iters * 4)
    # context: cuDNN nn.Conv2d of the replaced shape, fwd + dgrad + wgrad, TF32 off / on
    ctx = {}
    conv = torch.nn.Conv2d(a.cin, a.cout, a.k, a.stride, padding=a.k // 2, bias=False).to(dev)
    xc = x.clone().requires_grad_(True)
    torch.backends.cudnn.benchmark = True
    for tf32 in (False, True):
        torch.backends.cudnn.allow_tf32 = tf32
        for _ in range(3):
            conv(xc).backward(dy)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.iters):
            conv(xc).backward(dy)
        e1.record()
        torch.cuda.synchronize()
        ctx["cudnn_conv_tf32" if tf32 else "cudnn_conv_fp32"] = round(e0.elapsed_time(e1) / a.iters, 4)
    torch.backends.cudnn.allow_tf32 = False
    rows = []
    for i, L in enumerate(plan.launches):
        if L.kind != "kernel":
            continue
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.iters * plan.copies)]
        for u, v in evs:
            u.record()
            v.record()
        dp.profile(i, evs)
        for _ in range(a.iters):
            step()
        torch.cuda.synchronize()
        cnt = dp.profile_count(i)
        dp.profile(i, [])
        ts = [u.elapsed_time(v) for u, v in evs[: min(cnt, len(evs))]]
        ms = statistics.median(ts)
        gbs = L.bytes_per_image * n / (ms * 1e-3) / 1e9 if L.bytes_per_image else 0.0
        tf = L.flops_per_image * n / (ms * 1e-3) / 1e12 if L.flops_per_image else 0.0
        rows.append({"name": L.name, "what": L.what, "ms": round(ms, 4), "GBps": round(gbs, 1), "TFLOPs": round(tf, 2), "hbm_frac": round(gbs / peaks["hbm_gbs"], 3), "tf32_frac": round(tf / tf32_peak, 4)})
    tot = sum(r["ms"] for r in rows)
    print(f"layer {a.kernel} {a.cin}->{a.cout} {a.hw}^2 s{a.stride} batch {n}: fwd+bwd {layer_ms:.3f} ms (sum of launches {tot:.3f} ms; CUDA-graph replay {graph_ms:.3f} ms)")
    print(f"  context: cuDNN nn.Conv2d {a.cin}->{a.cout} k{a.k} s{a.stride} fwd+bwd: fp32 {ctx['cudnn_conv_fp32']:.3f} ms, TF32 {ctx['cudnn_conv_tf32']:.3f} ms")
    for r in rows:
        print(f"  {r['ms']:8.3f} ms {100 * r['ms'] / tot:5.1f}%  {r['GBps']:8.1f} GB/s  {r['TFLOPs']:7.2f} TF/s  {r['name']:28s} {r['what']}")
    if a.json:
        with open(a.json, "w") as f:
            json.dump({"args": vars(a), "layer_ms": layer_ms, "graph_ms": graph_ms, "context": ctx, "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
