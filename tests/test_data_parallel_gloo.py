"""Batch-sharded data parallelism on CPU (gloo, world_size 2) through the
repo's own DP code: bench.make_step + paper_2304_07741_b200.dp.GradBuckets.

Canvas kernels are per-image independent and FC wgrad is a sum over images
(SURVEY §8e-1), so after the bucketed all-reduce (sum) and the 1/world scale,
each rank's gradients of its half batch must equal the full-batch gradients
(CE loss, mean reduction), and one SGD(momentum) step must leave identical
parameters on every rank and equal to the single-process step.  The stand-in
network is the CPU reference module of a Canvas kernel (oracle.torch_ref,
Fig.-2 replication + stride 2) inside a small conv net, in fp64 — the same
step function bench.py captures into its CUDA graph over NCCL on GPUs.  Small
buckets force several buckets (reverse order, issued from the gradient hooks).
"""

import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2304_07741_b200 import zoo


def _net():
    from oracle.torch_ref import CanvasConvRef

    torch.manual_seed(0)
    return torch.nn.Sequential(
        torch.nn.Conv2d(3, 8, 3, padding=1, bias=False),
        torch.nn.ReLU(),
        CanvasConvRef(zoo.SEED7_K1, 8, 16, 8, 8, 3, 3, stride=2, g=4),
        torch.nn.ReLU(),
        torch.nn.AdaptiveAvgPool2d(1),
        torch.nn.Flatten(),
        torch.nn.Linear(16, 10),
    ).double()


def _data():
    g = torch.Generator().manual_seed(1)
    return torch.randn(8, 3, 8, 8, dtype=torch.float64, generator=g), torch.randint(0, 10, (8,), generator=g)


def _rank(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    m = _net()
    params = list(m.parameters())
    opt = torch.optim.SGD(params, lr=0.1, momentum=0.9)
    step, _, buckets = bench.make_step(m, params, opt, world, bucket_mb=0.0005)
    assert buckets is not None and len(buckets.buckets) >= 3
    x, y = _data()
    sh = slice(rank * 4, (rank + 1) * 4)
    step(x[sh], y[sh])
    grads = [p.grad.clone() for p in params]
    assert all(p.grad.data_ptr() >= buckets.flat.data_ptr() for p in params)  # still views of the flat buffer
    step(x[sh], y[sh])  # a second step: buffer re-zeroed, momentum applied
    torch.save({"grads": grads, "params": [p.detach().clone() for p in params]}, f"{out}.{rank}")
    dist.destroy_process_group()


def test_sharded_step_equals_full_batch(tmp_path):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "r")
    mp.spawn(_rank, args=(2, port, out), nprocs=2, join=True)
    import bench

    m = _net()
    params = list(m.parameters())
    opt = torch.optim.SGD(params, lr=0.1, momentum=0.9)
    step, _, buckets = bench.make_step(m, params, opt, 1)
    assert buckets is None
    x, y = _data()
    step(x, y)
    ref_grads = [p.grad.clone() for p in params]
    step(x, y)
    r0, r1 = torch.load(f"{out}.0"), torch.load(f"{out}.1")
    for a, b, c in zip(r0["grads"], r1["grads"], ref_grads):
        assert torch.equal(a, b)
        assert torch.allclose(a, c, rtol=1e-10, atol=1e-12)
    for a, b, c in zip(r0["params"], r1["params"], params):
        assert torch.equal(a, b)
        assert torch.allclose(a, c.detach(), rtol=1e-10, atol=1e-12)
