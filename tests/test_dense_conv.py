"""Dense (backbone) convolution on the tcgen05 GEMM templates (dense_conv.py):
plan construction on CPU; GPU parity of the forward and the weight gradient
against the fp64 oracle (F.conv2d) at the ResNet stem geometry."""

import pytest
import torch
import torch.nn.functional as F
from torch import nn

from paper_2304_07741_b200 import dense_conv

RTOL, ATOL = 1e-4, 1e-5


def test_stem_plan_lowers():
    p = dense_conv.lower_conv2d(3, 64, 7, 2, 3, 224, 224)
    names = [L.name for L in p.launches]
    assert any(n.endswith("fwd_conv") for n in names) and any("wgrad_conv" in n for n in names)
    assert "tc_gemm" in p.source and p.blob()[:8] == b"CNVSBLOB"


def test_cpu_path_is_torch():
    torch.manual_seed(0)
    c = nn.Conv2d(3, 8, 7, 2, 3, bias=False)
    t = dense_conv.TcConv2d.from_conv(c)
    x = torch.randn(2, 3, 20, 18)
    assert torch.equal(t(x), c(x))


@pytest.mark.gpu
@pytest.mark.parametrize("n,h,w", [(2, 224, 224), (3, 37, 29)])
def test_stem_conv_parity(n, h, w):
    torch.backends.cudnn.allow_tf32 = False
    g = torch.Generator().manual_seed(0)
    x = torch.randn(n, 3, h, w, generator=g)
    c = nn.Conv2d(3, 64, 7, 2, 3, bias=False)
    with torch.no_grad():
        c.weight.copy_(torch.randn(c.weight.shape, generator=g) / 12)
    dyshape = F.conv2d(x, c.weight, stride=2, padding=3).shape
    dy = torch.randn(dyshape, generator=g)
    wr = c.weight.detach().double().requires_grad_(True)
    yr = F.conv2d(x.double(), wr, stride=2, padding=3)
    yr.backward(dy.double())
    t = dense_conv.TcConv2d.from_conv(c).cuda()
    y = t(x.cuda())
    y.backward(dy.cuda())
    torch.testing.assert_close(y.cpu().double(), yr.detach(), rtol=RTOL, atol=ATOL)
    err = (t.weight.grad.cpu().double() - wr.grad).abs().max() / (ATOL + RTOL * wr.grad.abs().max())
    assert err <= 1.0, float(err)


@pytest.mark.gpu
@pytest.mark.parametrize("cin,cout,k,stride,pad,hw", [(64, 128, 1, 2, 0, 56), (128, 256, 1, 2, 0, 28), (16, 32, 3, 1, 1, 12), (8, 16, 3, 2, 1, 13), (3, 64, 7, 2, 3, 40)])
def test_conv_with_input_grad_parity(cin, cout, k, stride, pad, hw):
    """Downsample-style convs: forward, input gradient (col2im as a gather GEMM) and weight gradient."""
    g = torch.Generator().manual_seed(1)
    x = torch.randn(2, cin, hw, hw, generator=g)
    c = nn.Conv2d(cin, cout, k, stride, pad, bias=False)
    with torch.no_grad():
        c.weight.copy_(torch.randn(c.weight.shape, generator=g) / (cin * k * k) ** 0.5)
    dy = torch.randn(F.conv2d(x, c.weight, stride=stride, padding=pad).shape, generator=g)
    xr = x.double().requires_grad_(True)
    wr = c.weight.detach().double().requires_grad_(True)
    yr = F.conv2d(xr, wr, stride=stride, padding=pad)
    yr.backward(dy.double())
    t = dense_conv.TcConv2d.from_conv(c).cuda()
    xg = x.cuda().requires_grad_(True)
    y = t(xg)
    y.backward(dy.cuda())
    torch.testing.assert_close(y.cpu().double(), yr.detach(), rtol=RTOL, atol=ATOL)
    torch.testing.assert_close(xg.grad.cpu().double(), xr.grad, rtol=RTOL, atol=ATOL)
    err = (t.weight.grad.cpu().double() - wr.grad).abs().max() / (ATOL + RTOL * wr.grad.abs().max())
    assert err <= 1.0, float(err)


@pytest.mark.parametrize("cin,cout,k,stride,pad,h,w", [(3, 64, 7, 2, 3, 10, 9), (16, 32, 1, 2, 0, 9, 9), (16, 32, 1, 2, 0, 10, 8), (8, 16, 1, 3, 0, 7, 8), (8, 16, 3, 2, 1, 13, 11)])
def test_conv_plan_on_host_emulator(cin, cout, k, stride, pad, h, w):
    """The generated functors (forward, dgrad gather, wgrad in both operand
    orientations + the ordered / transposed partial reduce) run on the host
    emulator against fp64 F.conv2d."""
    import numpy as np

    from emu.runner import EmuPlan

    p = dense_conv.lower_conv2d(cin, cout, k, stride, pad, h, w, True)
    g = torch.Generator().manual_seed(3)
    x = torch.randn(2, cin, h, w, generator=g)
    wt = torch.randn(cout, cin, k, k, generator=g) / (cin * k * k) ** 0.5
    xr = x.double().requires_grad_(True)
    wr = wt.double().requires_grad_(True)
    yr = F.conv2d(xr, wr, stride=stride, padding=pad)
    dy = torch.randn(yr.shape, generator=g)
    yr.backward(dy.double())
    em = EmuPlan(p)
    xn, wn = x.numpy().copy(), [wt.reshape(cout, -1).numpy().copy()]
    y = np.zeros(tuple(yr.shape), np.float32)
    saved = [em._alloc(p.saved, 2)]
    em.run(0, xn, wn, y=y, saved=saved)
    dx = np.full_like(xn, np.nan)  # every dx element must be written (no memset in the plan)
    dws = [np.full_like(wn[0], np.nan)]
    em.run(1, xn, wn, dy=dy.numpy().copy(), dx=dx, dws=dws, saved=saved)
    torch.testing.assert_close(torch.from_numpy(y).double(), yr.detach(), rtol=RTOL, atol=ATOL)
    torch.testing.assert_close(torch.from_numpy(dx).double(), xr.grad, rtol=RTOL, atol=ATOL)
    torch.testing.assert_close(torch.from_numpy(dws[0]).double().view_as(wr), wr.grad, rtol=RTOL, atol=ATOL)
