"""Batch-sharded data parallelism contract on CPU (gloo, world_size 2).

Canvas kernels are per-image independent and FC wgrad is a sum over images
(SURVEY §8e-1), so averaging per-rank gradients of equal shards equals the
full-batch gradient.  Checked with the CPU reference module and
torch.distributed's allreduce — the per-gradient all-reduce (sum, then / world)
bench.py captures into its CUDA-graph step over NCCL on GPUs (DDP without
graphs issues the same sums, bucketed).
"""

import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2304_07741_b200 import zoo


def _rank(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.torch_ref import CanvasConvRef

    torch.manual_seed(0)
    m = CanvasConvRef(zoo.SEED7_K1, 8, 16, 6, 6, 3, 3, stride=2, g=4).double()
    x = torch.randn(4, 8, 6, 6, dtype=torch.float64, generator=torch.Generator().manual_seed(1))
    shard = x[rank * 2 : (rank + 1) * 2]
    m(shard).square().sum().backward()
    for p in m.parameters():
        dist.all_reduce(p.grad)
    if rank == 0:
        torch.save([p.grad.clone() for p in m.parameters()], out)
    dist.destroy_process_group()


def test_sharded_grads_equal_full_batch(tmp_path):
    out = str(tmp_path / "g.pt")
    mp.spawn(_rank, args=(2, 29511, out), nprocs=2, join=True)
    from oracle.torch_ref import CanvasConvRef

    torch.manual_seed(0)
    m = CanvasConvRef(zoo.SEED7_K1, 8, 16, 6, 6, 3, 3, stride=2, g=4).double()
    x = torch.randn(4, 8, 6, 6, dtype=torch.float64, generator=torch.Generator().manual_seed(1))
    m(x).square().sum().backward()
    got = torch.load(out)
    for a, b in zip(got, [p.grad for p in m.parameters()]):
        assert torch.allclose(a, b, rtol=1e-12, atol=1e-12)
