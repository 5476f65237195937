"""Canvas-ResNet-18 training throughput on B200 (BASELINE.json metric, config 2).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--kernel seed7_k1] [--batch 256]

Workload (config 2): torchvision ResNet-18 with all 16 3x3 convs
replaced by one sampled Canvas kernel (default: seed-7 kernel #1, the
Unfold+FC tensor case; G=4, K=3, stride-2 targets subsample first, Fig.-2
r-copy concat), synthetic ImageNet 224^2, per-GPU batch 256 (weak scaling),
fp32, CE loss + SGD(momentum) step.  One step = one fwd+bwd+update of one
batch per GPU.  N>1: one process per GPU (torchrun), DDP gradient allreduce
over NCCL — the only collective.

Timing: W warm-up steps, barrier + synchronize, CUDA events around K steps
on the compute stream, synchronize + barrier, max over ranks.  Inputs are
larger than L2 (154 MB of images per step + >1 GB of activations), so no
explicit flush.  ``e2e`` repeats the step with the batch copied from pinned
host memory and the loss read back every step.  ``roofline`` times the
dominant Canvas kernel (the K=9C FC GEMM of the layer1 targets) with CUDA
events recorded by libcanvas around each of its launches during the timed
region.  ``cpu_baseline`` / ``--impl reference`` time the CPU restatement
(oracle/torch_ref.py, torch fp32 on all host cores) on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
import torch.nn.functional as F  # noqa: E402

from paper_2304_07741_b200 import zoo  # noqa: E402

METRIC = "images/sec fwd+bwd (Canvas-ResNet-18, 224²) at 1/2/4/8 B200; % roofline/kernel"
WORKLOADS = {
    "resnet18": "config 2: torchvision ResNet-18, all 16 3x3 convs -> one Canvas kernel, fwd+bwd+SGD",
    "resnet29": "config 3: CIFAR ResNet-29 (bottleneck, 30 standard convs) -> one Canvas kernel, fwd+bwd+SGD",
    "resnext29_2x64d": "config 3: CIFAR ResNeXt-29 2x64d (21 standard convs; grouped 3x3 kept) -> one Canvas kernel, fwd+bwd+SGD",
    "mobilenet_v2": "config 5: torchvision MobileNetV2, 32 standard convs -> one Canvas kernel, fwd+bwd+SGD",
    "efficientnet_b0": "config 5: torchvision EfficientNet-B0, 60 standard convs -> one Canvas kernel, fwd+bwd+SGD",
    "vgg16": "config 5: torchvision VGG-16, 12 standard 3x3 convs -> one Canvas kernel, fwd+bwd+SGD",
}


def metric_of(model: str) -> str:
    if model == "resnet18":
        return METRIC
    from paper_2304_07741_b200.backbones import SPECS

    return f"images/sec fwd+bwd (Canvas-{model}, {SPECS[model]['input'][-1]}²) on B200; % roofline/kernel"


def peaks() -> dict:
    """Roofline denominators: MEASURED_PEAKS.json (driver-measured HBM copy
    bandwidth, cuBLAS bf16) plus the tcgen05 TF32 / bf16 and FP32-FFMA peaks
    measured on a B200 of this pool by scripts/peaks.cu (profiles/r02_peaks.json:
    burst = best short launch, sustained = median over 4 s back to back)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
    except OSError:
        pk = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "fallback": True}
    try:
        with open(os.path.join(ROOT, "profiles", "r02_peaks.json")) as f:
            pk["tcgen05"] = json.load(f)
    except (OSError, ValueError):
        pass
    return pk


def tf32_peak(pk: dict) -> tuple[float, str]:
    """Sustained TF32 dense peak (TFLOP/s) for kernels timed inside a seconds-long step."""
    t = pk.get("tcgen05", {})
    if t.get("tf32_tcgen05_tflops_sustained"):
        return float(t["tf32_tcgen05_tflops_sustained"]), "measured tcgen05 kind::tf32 dense peak, sustained (profiles/r02_peaks.json, scripts/peaks.cu)"
    return pk.get("bf16_tflops_sustained", pk["bf16_tflops"]) / 2.0, "1/2 of MEASURED_PEAKS.json bf16_tflops_sustained (no measured TF32 figure)"


def build_model(kernel: str, device=None, cpu_reference: bool = False, fuse_bn: bool = True, model: str = "resnet18"):
    """The workload network (backbones.py) with every standard conv replaced by
    ``kernel``; the CPU reference path uses the oracle modules instead."""
    import math

    from paper_2304_07741_b200 import backbones

    text = zoo.ALL[kernel]
    factory = None
    if cpu_reference:
        from oracle.torch_ref import CanvasConvRef

        def factory(conv):
            k = conv.kernel_size[0]
            g = math.gcd(min(conv.in_channels, conv.out_channels), 4)
            return CanvasConvRef(text, conv.in_channels, conv.out_channels, 8, 8, k, k, stride=conv.stride[0], g=g, seed=None)

    m, names = backbones.build(model, text, g=4, fuse_bn=fuse_bn, factory=factory)
    if model == "resnet18":
        assert len(names) == 16, names
    return m.to(device) if device is not None else m


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""

    Q = "index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, index: int):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        rows = [r.split(", ") for r in self.f.read().strip().splitlines() if r.strip()]
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) >= 9 for i in range(4) if r[5 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


class CpuReference:
    """CPU restatement (oracle/torch_ref.py, torch fp32, all host threads) of Canvas-ResNet-18."""

    def __init__(self, kernel: str, batch: int = 2, model: str = "resnet18"):
        from paper_2304_07741_b200.backbones import SPECS

        torch.set_num_threads(os.cpu_count() or 1)
        self.kernel, self.batch, self.model = kernel, batch, model
        self.m = build_model(kernel, cpu_reference=True, model=model)
        self.opt = torch.optim.SGD(self.m.parameters(), lr=0.01, momentum=0.9)
        g = torch.Generator().manual_seed(0)
        spec = SPECS[model]
        self.x = torch.randn(batch, *spec["input"], generator=g)
        self.y = torch.randint(0, spec["classes"], (batch,), generator=g)

    def step(self) -> None:
        self.opt.zero_grad(set_to_none=True)
        F.cross_entropy(self.m(self.x), self.y).backward()
        self.opt.step()

    @staticmethod
    def cores_desc() -> str:
        model = ""
        try:
            with open("/proc/cpuinfo") as f:
                model = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), "")
        except OSError:
            pass
        return f"{os.cpu_count()} threads, {model}"


def cpu_full_batch(kernel: str, batch: int, model: str = "resnet18") -> dict:
    """One full training step at the GPU arm's per-GPU batch through the CPU
    restatement (">= 1 full batch-256 step"), after a batch-2
    warm-up step; the same network, kernel, loss and optimizer."""
    warm = CpuReference(kernel, 2, model)
    warm.step()
    del warm
    ref = CpuReference(kernel, batch, model)
    t0 = time.perf_counter()
    ref.step()
    dt = time.perf_counter() - t0
    return {"value": batch / dt, "unit": "images/s", "cores": torch.get_num_threads(), "seconds": round(dt, 2), "same_config": True, "sample": f"1 full fwd+bwd+SGD step of batch {batch} at {ref.x.shape[-1]}^2 through Canvas-{model} ({kernel}) in torch fp32 on CPU ({CpuReference.cores_desc()}), after a batch-2 warm-up step"}


def traffic_key(kernel: str, model: str, mod, in_shape, batch: int) -> str:
    return f"{kernel}|{model}|{mod.in_channels}x{mod.out_channels}@{in_shape[2]}x{in_shape[3]}/s{mod.stride}|b{batch}"


def run_reference(args, rank: int, world: int) -> None:
    """Reference arm: the CPU restatement of the path on the host cores (rank 0
    only), on the GPU arm's config: every timed step is one full fwd+bwd+SGD
    step at the per-GPU batch (``--batch``, 256).  Warm-up steps run at batch 2.
    Timed steps stop early (at least one) once ``--ref-seconds`` is spent so the
    whole run stays within a few minutes; the line says how many ran."""
    if rank != 0:
        return
    warm = CpuReference(args.kernel, batch=2, model=args.model)
    for _ in range(max(1, args.warmup)):
        warm.step()
    del warm
    ref = CpuReference(args.kernel, batch=args.batch, model=args.model)
    times = []
    t_all = time.perf_counter()
    for _ in range(max(1, args.steps)):
        t0 = time.perf_counter()
        ref.step()
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_all >= args.ref_seconds:
            break
    val = args.batch * len(times) / sum(times)
    sample = f"{len(times)} full fwd+bwd+SGD steps of batch {args.batch} at {ref.x.shape[-1]}^2 through Canvas-{args.model} ({args.kernel}) in torch fp32 on CPU ({CpuReference.cores_desc()}); {max(1, args.warmup)} batch-2 warm-up steps"
    line = {
        "impl": "reference",
        "metric": metric_of(args.model),
        "value": round(val, 3),
        "unit": "images/s",
        "n_gpus": world,
        "steps": args.steps,
        "steps_timed": len(times),
        "warmup": args.warmup,
        "ms_per_step": round(1000.0 * statistics.mean(times), 1),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": WORKLOADS[args.model] + " (CPU restatement, oracle/torch_ref.py)", "kernel": args.kernel, "model": args.model, "global_batch": args.batch, "per_gpu_batch": args.batch},
        "cpu_baseline": {"value": round(val, 3), "unit": "images/s", "cores": torch.get_num_threads(), "kind": "port", "sample": sample, "same_config": True},
        "e2e": {"value": round(val, 3), "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def make_step(model, params, opt, world: int, bucket_mb: float = 25.0, dp: bool | None = None):
    """The training step of every arm: CE loss, backward, data-parallel gradient
    average (N > 1: bucketed all-reduce overlapped with the backward,
    paper_2304_07741_b200.dp.GradBuckets — the only collective),
    SGD(momentum) update.  Returns (step, fwd_bwd_update, buckets):
    ``fwd_bwd_update`` is the capturable part (no host sync, grads live in the
    bucket buffer for N > 1); ``step`` also resets the gradients."""
    from paper_2304_07741_b200.dp import GradBuckets

    dp = world > 1 if dp is None else dp
    buckets = GradBuckets(params, world, bucket_mb, collective=dp) if dp else None

    def fwd_bwd_update(xb, yb):
        if buckets is not None:
            buckets.zero()
        loss = F.cross_entropy(model(xb), yb)
        loss.backward()
        if buckets is not None:
            buckets.finish()
        opt.step()
        return loss

    def step(xb, yb):
        if buckets is None:
            opt.zero_grad(set_to_none=True)
        return fwd_bwd_update(xb, yb)

    return step, fwd_bwd_update, buckets


def relaunch_distributed(n: int) -> None:
    """``--gpus N`` without a torchrun environment: re-exec this command as N
    ranks (one process per GPU) under torch.distributed.run on 127.0.0.1."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    raise SystemExit(subprocess.call(cmd))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=0, help="per-GPU batch (default: the workload's, SURVEY §8d: 512 for config 3, else 256)")
    ap.add_argument("--kernel", default="seed7_k1", choices=sorted(zoo.ALL))
    ap.add_argument("--model", default="resnet18", help="workload backbone (backbones.SPECS): resnet18 = config 2 (default), resnet29 / resnext29_2x64d = config 3, mobilenet_v2 / efficientnet_b0 / vgg16 = config 5")
    ap.add_argument("--impl", default="canvas", choices=["canvas", "reference"])
    ap.add_argument("--ref-seconds", type=float, default=120.0, help="reference arm: stop timing full-batch CPU steps after this many seconds (>= 1 step)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-context", action="store_true")
    ap.add_argument("--no-fuse-bn", action="store_true", help="keep the backbone's cuDNN BatchNorm2d + ReLU")
    ap.add_argument("--no-graph", action="store_true", help="launch the step eagerly instead of replaying one captured CUDA graph")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "canvas" else args.warmup
    if args.batch <= 0:
        from paper_2304_07741_b200.backbones import SPECS

        args.batch = SPECS[args.model].get("batch", 256)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_distributed(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # CANVAS_DP_SELFTEST=1 under torchrun with one rank: the data-parallel path
    # (NCCL process group, bucketed all-reduce captured in the step graph, max
    # over ranks) runs on a single GPU — its smoke test on a 1-GPU box
    dp_on = world > 1 or ("WORLD_SIZE" in os.environ and os.environ.get("CANVAS_DP_SELFTEST") == "1")
    if dp_on:
        dist.init_process_group("nccl", device_id=dev)
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.benchmark = True

    from paper_2304_07741_b200.backbones import SPECS

    spec = SPECS[args.model]
    model = build_model(args.kernel, dev, fuse_bn=not args.no_fuse_bn, model=args.model)
    use_graph = not args.no_graph
    params = list(model.parameters())
    opt = torch.optim.SGD(params, lr=0.01, momentum=0.9)
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    x = torch.randn(args.batch, *spec["input"], device=dev, generator=gen)
    lab = torch.randint(0, spec["classes"], (args.batch,), device=dev, generator=gen)
    step, fwd_bwd_update, buckets = make_step(model, params, opt, world, dp=dp_on)

    t_build = time.perf_counter()
    for _ in range(args.warmup):
        step(x, lab)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t_build

    # --- per-kernel events for the layer1 target (64->64 at 56x56): every FC GEMM launch
    # (forward, dgrad, wgrad) is bracketed by CUDA events libcanvas records on its
    # launch stream during the timed region; the dominant one is reported ---
    from paper_2304_07741_b200.module import CanvasConv2d

    core = model.module if hasattr(model, "module") else model
    # dominant target: the first replaced conv at the network's finest resolution
    # (ResNet-18: layer1.0.conv1, 64->64 at 56x56); its input shape is traced
    shapes = {}
    def _trace(mod, i, o):
        shapes.setdefault(id(mod), tuple(i[0].shape))  # returns None: output unchanged

    hooks = [m.register_forward_hook(_trace) for m in core.modules() if isinstance(m, CanvasConv2d)]
    with torch.no_grad():
        core(x[:1])
    for h in hooks:
        h.remove()
    l1 = max((m for m in core.modules() if isinstance(m, CanvasConv2d)), key=lambda m: shapes[id(m)][2] * shapes[id(m)][3] * min(m.in_channels, m.out_channels) ** 2 / m.stride ** 2)
    dp = l1.device_plan(x.new_empty(1, *shapes[id(l1)][1:]))
    recs = [i for i, L in enumerate(dp.plan.launches) if L.kind == "kernel" and L.flops_per_image and L.what.startswith("tc ")]
    per_rec_events = {}
    for i in recs:
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(4 * 2 * args.steps)]
        for ea, eb in evs:
            ea.record()
            eb.record()
        dp.profile(i, evs)
        per_rec_events[i] = evs

    per_step_launches = 0
    for m in core.modules():
        if isinstance(m, CanvasConv2d):
            for p in m._plans.values():
                per_step_launches += p.launches(0) + p.launches(1)
    from paper_2304_07741_b200.post import FusedBatchNorm2d

    from paper_2304_07741_b200.post import FusedMaxPool2d

    per_step_launches += 4 * sum(isinstance(m, FusedBatchNorm2d) for m in core.modules())  # stats+apply, reduce+apply
    per_step_launches += 2 * sum(isinstance(m, FusedMaxPool2d) for m in core.modules())  # fwd, bwd
    from paper_2304_07741_b200.dense_conv import TcConv2d

    per_step_launches += 4 * sum(isinstance(m, TcConv2d) for m in core.modules())  # pack, fwd, wgrad, reduce

    # --- CUDA graph of the whole step (forward, backward, all-reduce, SGD): one
    # replay per step, so host launch overhead leaves the critical path.  The
    # kernel-timing events above are captured as external event nodes (libcanvas
    # records them with CU_EVENT_RECORD_EXTERNAL while the stream is capturing). ---
    graph_note = "off (--no-graph)"
    if use_graph:
        try:
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                for _ in range(2):
                    step(x, lab)
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            static_x, static_y = x.clone(), lab.clone()
            for i, evs in per_rec_events.items():  # re-arm: slots 0.. are the captured launches
                dp.profile(i, evs)
            graph = torch.cuda.CUDAGraph()
            if buckets is None:
                opt.zero_grad(set_to_none=True)
            with torch.cuda.graph(graph):
                static_loss = fwd_bwd_update(static_x, static_y)
            graph.replay()
            torch.cuda.synchronize()
            graph_note = "whole step captured once, replayed per step"

            def step(xb, yb):  # noqa: F811
                if xb is not static_x:  # host (pinned) or device batch -> the graph's input
                    static_x.copy_(xb, non_blocking=True)
                    static_y.copy_(yb, non_blocking=True)
                graph.replay()
                return static_loss

            x, lab = static_x, static_y
        except Exception as err:  # capture unsupported here: measure the eager step
            use_graph = False
            graph_note = f"capture failed ({type(err).__name__}: {str(err)[:120]}); eager step"
            torch.cuda.synchronize()

    clocks = Clocks(local)
    if dp_on:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step(x, lab)
    e1.record()
    torch.cuda.synchronize()
    if dp_on:
        dist.barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    k_times = {}
    for i, evs in per_rec_events.items():
        cnt = dp.profile_count(i)
        dp.profile(i, [])
        k_times[i] = [ea.elapsed_time(eb) for ea, eb in evs[: min(cnt, len(evs))]]
    if dp_on:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * args.batch * 1000.0 / ms

    # --- e2e: batch from pinned host memory each step, loss read back each step ---
    xh = x.cpu().pin_memory()
    lh = lab.cpu().pin_memory()
    if dp_on:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record()
    e2e_steps = max(4, args.steps)  # the pipeline's first (unoverlapped) copy is amortised over as many steps as the timed run
    if use_graph:
        # double-buffered input pipeline: step i+1's batch is copied host -> device
        # on a copy stream while step i's graph runs (every step still moves its
        # own 154 MB inside the timed region, it just overlaps compute)
        cs = torch.cuda.Stream()
        stage = [(torch.empty_like(x), torch.empty_like(lab)) for _ in range(2)]
        ready = [torch.cuda.Event() for _ in range(2)]
        free = [torch.cuda.Event() for _ in range(2)]

        def prefetch(b):
            with torch.cuda.stream(cs):
                cs.wait_event(free[b])
                stage[b][0].copy_(xh, non_blocking=True)
                stage[b][1].copy_(lh, non_blocking=True)
                ready[b].record(cs)

        # the loss of every step is read back to the host too, two steps behind: its
        # D2H copy is queued after the step and the host reads step i-2's value while
        # steps i-1 and i are queued (a blocking .item() per step would drain the GPU
        # queue and add the graph-launch latency to every step; one step of slack
        # left the GPU idle whenever the host thread was descheduled)
        LAG = 2
        lhost = torch.empty(LAG + 1, dtype=torch.float32).pin_memory()
        lready = [torch.cuda.Event() for _ in range(LAG + 1)]
        for b in range(2):
            free[b].record()
        prefetch(0)
        for i in range(e2e_steps):
            b = i % 2
            torch.cuda.current_stream().wait_event(ready[b])
            x.copy_(stage[b][0], non_blocking=True)
            lab.copy_(stage[b][1], non_blocking=True)
            free[b].record()
            if i + 1 < e2e_steps:
                prefetch(1 - b)
            loss = step(x, lab)
            li = i % (LAG + 1)
            lhost[li : li + 1].copy_(loss.detach().reshape(1).float(), non_blocking=True)
            lready[li].record()
            if i >= LAG:
                lj = (i - LAG) % (LAG + 1)
                lready[lj].synchronize()
                float(lhost[lj])
        for i in range(max(0, e2e_steps - LAG), e2e_steps):
            lready[i % (LAG + 1)].synchronize()
            float(lhost[i % (LAG + 1)])
    else:
        for _ in range(e2e_steps):
            loss = step(xh.to(dev, non_blocking=True), lh.to(dev, non_blocking=True))
            float(loss.item())
    e3.record()
    torch.cuda.synchronize()
    ms_e2e = e2.elapsed_time(e3) / e2e_steps
    if dp_on:
        t = torch.tensor([ms_e2e], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())
    del t0
    e2e = world * args.batch * 1000.0 / ms_e2e

    # --- roofline of the dominant kernel (largest total time among the layer1 GEMMs) ---
    pk = peaks()
    tf32_pk, tf32_src = tf32_peak(pk)
    kern = []
    for i, ts in k_times.items():
        L = dp.plan.launches[i]
        avg_ms = statistics.mean(ts) if ts else float("nan")
        flops = float(L.flops_per_image) * args.batch
        ach = flops / (avg_ms * 1e-3) / 1e12
        kern.append({"kernel": L.name, "what": L.what, "launch_ms": round(avg_ms, 4), "launches_timed": len(ts), "useful_tflops": round(ach, 2), "frac_tf32": round(ach / tf32_pk, 4), "issued_frac_tf32": round(3 * ach / tf32_pk, 4), "total_ms": sum(ts)})
    if not kern:
        raise SystemExit(f"no tensor-core launch in the dominant target of {args.model}: nothing to put on the roofline")
    dom = max(kern, key=lambda r: r["total_ms"])
    L = dp.plan.launches[next(i for i in k_times if dp.plan.launches[i].name == dom["kernel"])]
    roofline = {
        "bound": "tensor",
        "kernel": dom["kernel"],
        "achieved": dom["useful_tflops"],
        "peak": round(tf32_pk, 1),
        "unit": "TFLOP/s",
        "frac": dom["frac_tf32"],
        "traffic": None,
        "launch_ms": dom["launch_ms"],
        "launches_timed": dom["launches_timed"],
        "issued_frac": dom["issued_frac_tf32"],
        "algorithmic": f"{L.flops_per_image}*{args.batch} FLOP per launch = 2 x FC MACs of '{L.what}' (SURVEY §8d); 3xTF32 issues 3x that",
        "peak_source": tf32_src,
        "layer1_gemms": [{k: v for k, v in r.items() if k != "total_ms"} for r in kern],
    }
    # ncu counters of the dominant kernel, keyed by the workload that produced them:
    # (kernel, model, dominant target c_in x c_out @ h x w / stride, batch)
    tkey = traffic_key(args.kernel, args.model, l1, shapes[id(l1)], args.batch)
    roofline["traffic_key"] = tkey
    prof_json = os.path.join(ROOT, "profiles", "dominant_traffic.json")
    if os.path.exists(prof_json):
        try:
            with open(prof_json) as f:
                tr = json.load(f).get(tkey, {}).get(roofline["kernel"].split("_", 1)[1])
            if tr:
                roofline["traffic"] = tr["dram_bytes"]
                roofline["traffic_source"] = tr.get("source")
                if tr.get("warp_instructions") and clk.get("sm_mhz"):
                    # the computed-operand GEMMs are bound by SIMT operand production,
                    # so the SM issue rate (4 warp-instructions / clock / SM) is the
                    # roofline that binds them: ncu instruction count of one launch over
                    # its live duration, against 148 SMs x 4 x the measured SM clock
                    ips = tr["warp_instructions"] / (roofline["launch_ms"] * 1e-3)
                    roofline["issue"] = {"achieved_warp_inst_per_s": round(ips / 1e9, 1), "peak_warp_inst_per_s": round(148 * 4 * clk["sm_mhz"] * 1e6 / 1e9, 1), "unit": "G warp-instructions/s", "frac": round(ips / (148 * 4 * clk["sm_mhz"] * 1e6), 3), "source": tr.get("source")}
        except (OSError, ValueError):
            pass
    net = network_roofline(core, x[:1], args.batch, ms, pk["hbm_gbs"], tf32_pk)

    line = {
        "metric": metric_of(args.model),
        "value": round(value, 2),
        "unit": "images/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic",
        "config": {
            "workload": WORKLOADS[args.model],
            "kernel": args.kernel,
            "model": args.model,
            "global_batch": args.batch * world,
            "per_gpu_batch": args.batch,
            "image": "x".join(map(str, spec["input"])) + " synthetic N(0,1), random-init weights",
            "parallelism": f"dp{world}",
            "G": 4,
            "K": 3,
            "l2": "inputs larger than L2 (no flush)",
            "cuda_graph": graph_note,
            "precision": "fp32 storage; FC contractions 3xTF32 on tcgen05 (hi*hi + hi*lo + lo*hi, fp32 accumulate in TMEM), everything else fp32",
            "semantics": {"stride_policy": "x[..., ::s, ::s] first, kernel at output resolution (App. A.10)", "replication": "Fig.-2 r copies: concat (C_out = r C_in) / chunk-sum (C_in = r C_out)", "bn_post_pass": "off (SPEC.md:658); the backbone BN after each replaced conv runs as the fused native post-pass", "ties": "fold max: even split; bcast min/max: 1/2-1/2; relu'(0) = abs'(0) = 0 (App. A.5/A.6/A.8)", "bcast_order": "tile (lhs index r mod L)"},
        },
        "e2e": {"value": round(e2e, 2), "unit": "images/s", "h2d_bytes_per_step": int(xh.numel() * 4 + lh.numel() * 8), "d2h_bytes_per_step": 4},
        "gpu_launches": per_step_launches * args.steps,
        "roofline": roofline,
        "network_roofline": net,
        "clocks": clk,
        "warmup_s": round(t_build, 1),
    }
    if rank == 0 and world == 1 and not args.no_context:
        line["context"] = context_numbers(args, dev)
    if rank == 0 and world == 1 and not args.no_cpu:
        cb = cpu_full_batch(args.kernel, args.batch, model=args.model)
        line["cpu_baseline"] = {k: v for k, v in cb.items() if k in ("value", "unit", "cores", "sample", "same_config")}
        line["cpu_baseline"]["kind"] = "port"
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dp_on:
        dist.destroy_process_group()


def network_roofline(core, x1, batch: int, ms_step: float, hbm_gbs: float, tf32_tflops: float) -> dict:
    """SURVEY §8(d) network roofline: roofline images/s = 1 / sum_k max(bytes_k /
    BW, flops_k / peak_k) over every kernel the step launches, per image.

    Canvas plans and the dense tcgen05 convs carry per-launch algorithmic
    bytes / useful FLOPs (lowering.Launch); their FLOPs are counted as issued
    3xTF32 (3 MMAs per useful MAC — the fp32-accuracy requirement, SURVEY §7
    decision 4) against the measured tcgen05 TF32 peak.  The fused BN
    post-pass, max-pool, head, loss and the SGD(momentum) update are
    HBM-bound: their compulsory bytes per launch (activation reads / writes,
    1-byte masks, 20 B per parameter for the update).  ``frac`` = measured
    images/s / roofline images/s."""
    from paper_2304_07741_b200.dense_conv import TcConv2d, lower_conv2d
    from paper_2304_07741_b200.module import CanvasConv2d
    from paper_2304_07741_b200.post import FusedBatchNorm2d, FusedMaxPool2d

    io = {}

    def hook(mod, i, o):
        io[id(mod)] = (tuple(i[0].shape), tuple(o.shape), len(i) > 1 and i[1] is not None)

    hooks = [m.register_forward_hook(hook) for m in core.modules() if isinstance(m, (CanvasConv2d, TcConv2d, FusedBatchNorm2d, FusedMaxPool2d, torch.nn.Linear))]
    with torch.no_grad():
        core(x1)
    for h in hooks:
        h.remove()
    bw = hbm_gbs * 1e9
    pk = tf32_tflops * 1e12
    parts = {"canvas": 0.0, "dense_conv": 0.0, "bn": 0.0, "pool": 0.0, "head": 0.0, "sgd": 0.0}

    def plan_time(plan):
        t = 0.0
        for L in plan.launches:
            if L.kind == "kernel":
                t += max(L.bytes_per_image / bw, 3 * L.flops_per_image / pk)
        return t

    for m in core.modules():
        if id(m) not in io:
            continue
        ishape, oshape, has_res = io[id(m)]
        ni, no = math_prod(ishape[1:]), math_prod(oshape[1:])
        if isinstance(m, CanvasConv2d):
            parts["canvas"] += plan_time(m.plan(ishape[2], ishape[3]))
        elif isinstance(m, TcConv2d):
            parts["dense_conv"] += plan_time(lower_conv2d(m.in_channels, m.out_channels, m.kernel_size[0], m.stride[0], m.padding[0], ishape[2], ishape[3], m.in_channels != 3))
        elif isinstance(m, FusedBatchNorm2d):
            # fwd: stats read x; apply read x (+res) write y (+1 B relu mask)
            # bwd: reduce read dy, x (mask); apply read dy, x (mask) write dx (+dres)
            b = 4 * ni * (1 + 2 + has_res) + (ni if m.relu else 0)
            b += 4 * ni * (2 + 2 + 1 + (1 if has_res and m.relu else 0)) + (2 * ni if m.relu else 0)
            parts["bn"] += b / bw
        elif isinstance(m, FusedMaxPool2d):
            parts["pool"] += (4 * ni + 5 * no + (5 * no + 4 * ni)) / bw
        elif isinstance(m, torch.nn.Linear):
            parts["head"] += max(4 * (ni + no) * 3 / bw, 3 * 2 * m.in_features * m.out_features / 74e12)
    nparam = sum(p.numel() for p in core.parameters())
    parts["sgd"] = 20.0 * nparam / batch / bw  # p, g, momentum read; p, momentum written (per image share)
    t_img = sum(parts.values())
    roof = 1.0 / t_img
    meas = batch * 1000.0 / ms_step
    return {
        "roofline_images_s": round(roof, 1),
        "measured_images_s": round(meas, 1),
        "frac": round(meas / roof, 4),
        "share": {k: round(v / t_img, 4) for k, v in parts.items()},
        "how": "sum over launched kernels of max(algorithmic bytes / HBM, issued 3xTF32 FLOPs / measured TF32 tcgen05 peak) per image (SURVEY §8d); HBM = MEASURED_PEAKS.json hbm_gbs",
    }


def math_prod(t) -> int:
    r = 1
    for v in t:
        r *= int(v)
    return r


def context_numbers(args, dev) -> dict:
    """The unreplaced backbone (cuDNN, fp32 with TF32 off) for context only."""
    from paper_2304_07741_b200.backbones import SPECS, backbone

    torch.manual_seed(0)
    m = backbone(args.model).to(dev)
    opt = torch.optim.SGD(m.parameters(), lr=0.01, momentum=0.9)
    spec = SPECS[args.model]
    x = torch.randn(args.batch, *spec["input"], device=dev)
    y = torch.randint(0, spec["classes"], (args.batch,), device=dev)

    def step():
        opt.zero_grad(set_to_none=True)
        F.cross_entropy(m(x), y).backward()
        opt.step()

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        step()
    b.record()
    torch.cuda.synchronize()
    return {f"{args.model}_cudnn_fp32_images_s": round(args.batch * 5 * 1000.0 / a.elapsed_time(b), 1)}


if __name__ == "__main__":
    main()
