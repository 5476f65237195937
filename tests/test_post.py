"""BN post-pass (include/canvas_post.h): exports, the ResNet
rewiring, and GPU parity of the fused kernels against torch fp64 BatchNorm
(+ residual, + ReLU) — forward, backward and the running-stat update — and of
the native stem max-pool against torch (ties on ReLU zeros, NaN)."""

import copy
import re
from pathlib import Path

import pytest
import torch
import torch.nn.functional as F
from torch import nn

from paper_2304_07741_b200 import post

HDR = Path(__file__).resolve().parents[1] / "include" / "canvas_post.h"
RTOL, ATOL = 1e-4, 1e-5  # north star fp32 tolerance vs fp64


def test_exports_every_declared_symbol():
    lib = post.load_library()
    names = sorted(set(re.findall(r"^\w[\w\s\*]*?\b(canvas_\w+)\(", HDR.read_text(), re.M)))
    assert len(names) == 7, names
    for n in names:
        assert hasattr(lib, n), n
    assert lib.canvas_post_abi_version() == post.ABI_VERSION
    assert lib.canvas_bn_workspace(256, 64, 3136) > 0


def test_bad_arguments_fail_loudly():
    lib = post.load_library()
    rc = lib.canvas_bn_forward(0, 4, 4, *([None] * 9), 0.1, 1e-5, 1, None, None, None)
    assert rc == -5 and "bad arguments" in lib.canvas_post_last_error().decode()


def test_fuse_backbone_matches_unfused_on_cpu():
    """The rewired ResNet computes the same function (CPU path = torch BN)."""
    import torchvision

    torch.manual_seed(0)
    m = torchvision.models.resnet18(num_classes=10)
    f = copy.deepcopy(m)
    assert post.fuse_backbone(f) == 20  # stem + 16 block BNs + 3 downsample BNs
    x = torch.randn(2, 3, 64, 64)
    for mode in (True, False):
        m.train(mode)
        f.train(mode)
        torch.testing.assert_close(f(x), m(x), rtol=1e-5, atol=1e-5)
    assert torch.equal(f.layer1[0].bn1.running_mean, m.layer1[0].bn1.running_mean)


def _ref(x, res, bn, relu):
    xd = x.double().requires_grad_(True)
    rd = res.double().requires_grad_(True) if res is not None else None
    w = bn.weight.detach().double().requires_grad_(True)
    b = bn.bias.detach().double().requires_grad_(True)
    rm, rv = bn.running_mean.double().clone(), bn.running_var.double().clone()
    y = F.batch_norm(xd, rm, rv, w, b, True, bn.momentum, bn.eps)
    if rd is not None:
        y = y + rd
    if relu:
        y = F.relu(y)
    return y, xd, rd, w, b, rm, rv


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(8, 16, 56, 56), (256, 64, 7, 7), (5, 3, 5, 5), (32, 8, 14, 14), (3, 5, 2, 3)])
@pytest.mark.parametrize("relu,res", [(False, False), (True, False), (True, True), (False, True)])
def test_bn_parity(shape, relu, res):
    dev = torch.device("cuda:0")
    g = torch.Generator().manual_seed(0)
    x = torch.randn(shape, generator=g) * 2 + 0.5
    r = torch.randn(shape, generator=g) if res else None
    dy = torch.randn(shape, generator=g)
    bn = nn.BatchNorm2d(shape[1])
    with torch.no_grad():
        bn.weight.uniform_(0.5, 1.5, generator=g)
        bn.bias.uniform_(-0.5, 0.5, generator=g)
        bn.running_var.uniform_(0.5, 2.0, generator=g)
    yr, xd, rd, w, b, rm, rv = _ref(x, r, bn, relu)
    yr.backward(dy.double())

    fb = post.FusedBatchNorm2d.from_bn(bn, relu=relu).to(dev).train()
    xg = x.to(dev).requires_grad_(True)
    rg = r.to(dev).requires_grad_(True) if res else None
    y = fb(xg, rg)
    y.backward(dy.to(dev))
    torch.cuda.synchronize()

    def close(a, b_, what, rtol=RTOL, atol=ATOL):
        torch.testing.assert_close(a.detach().cpu().double(), b_.detach(), rtol=rtol, atol=atol, msg=what)

    close(y, yr, "y")
    close(xg.grad, xd.grad, "dx")
    if res:
        close(rg.grad, rd.grad, "dresidual")
    # parameter grads are sums over N*H*W terms: normwise check
    for got, want, what in ((fb.weight.grad, w.grad, "dgamma"), (fb.bias.grad, b.grad, "dbeta")):
        err = (got.cpu().double() - want).norm() / max(want.norm(), 1e-30)
        assert err < 1e-5, (what, float(err))
    close(fb.running_mean, rm, "running_mean")
    close(fb.running_var, rv, "running_var")
    assert int(fb.num_batches_tracked) == 1


@pytest.mark.gpu
def test_bn_deterministic():
    dev = torch.device("cuda:0")
    x = torch.randn(64, 32, 28, 28, device=dev)
    fb = post.FusedBatchNorm2d(32, relu=True).to(dev)
    outs = []
    for _ in range(2):
        xg = x.clone().requires_grad_(True)
        y = fb(xg)
        y.backward(torch.ones_like(y))
        outs.append((y.detach().clone(), xg.grad.clone(), fb.weight.grad.clone()))
        fb.weight.grad = None
    for a, b in zip(*outs):
        assert torch.equal(a, b)


@pytest.mark.gpu
def test_fused_resnet_training_step_matches_unfused():
    import torchvision

    dev = torch.device("cuda:0")
    torch.backends.cudnn.allow_tf32 = False
    torch.manual_seed(0)
    m = torchvision.models.resnet18(num_classes=10).to(dev).double()
    f = copy.deepcopy(m).float()
    post.fuse_backbone(f)
    x = torch.randn(4, 3, 64, 64, device=dev)
    y0 = m(x.double())
    y1 = f(x)
    torch.testing.assert_close(y1.double(), y0, rtol=1e-3, atol=1e-4)
    y0.sum().backward()
    y1.sum().backward()
    for (n0, p0), (n1, p1) in zip(m.named_parameters(), f.named_parameters()):
        assert n0 == n1
        err = (p1.grad.double() - p0.grad).norm() / max(p0.grad.norm(), 1e-30)
        assert err < 1e-3, (n0, float(err))


@pytest.mark.gpu
@pytest.mark.parametrize("shape,k,s,p", [((4, 8, 112, 112), 3, 2, 1), ((2, 3, 13, 16), 3, 2, 1), ((3, 2, 6, 4), 3, 2, 1), ((2, 3, 9, 7), 3, 2, 1), ((2, 4, 8, 8), 2, 2, 0), ((1, 2, 11, 10), 3, 1, 1)])
def test_maxpool_parity(shape, k, s, p):
    dev = torch.device("cuda:0")
    g = torch.Generator().manual_seed(0)
    x = torch.randn(shape, generator=g)
    x = torch.relu(x)  # ReLU zeros: exact ties in many windows (first maximum wins)
    dy = torch.randn(F.max_pool2d(x, k, s, p).shape, generator=g)
    xr = x.double().requires_grad_(True)
    yr = F.max_pool2d(xr, k, s, p)
    yr.backward(dy.double())
    m = post.FusedMaxPool2d(k, s, p)
    xg = x.to(dev).requires_grad_(True)
    y = m(xg)
    y.backward(dy.to(dev))
    assert torch.equal(y.cpu().double(), yr.detach())
    torch.testing.assert_close(xg.grad.cpu().double(), xr.grad, rtol=1e-6, atol=1e-6)


@pytest.mark.gpu
def test_maxpool_nan_propagates():
    x = torch.zeros(1, 1, 4, 4, device="cuda")
    x[0, 0, 3, 3] = float("nan")  # only window (1, 1) covers it
    y = post.FusedMaxPool2d(3, 2, 1)(x)
    assert torch.isnan(y[0, 0, 1, 1]) and not torch.isnan(y[0, 0, :1]).any() and not torch.isnan(y[0, 0, 1, 0])
