"""Probe: cuDNN vs native ATen BatchNorm2d (train) fwd+bwd at ResNet-18 shapes (analysis only)."""
import torch
import torch.nn as nn
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_07741_b200.post import FusedBatchNorm2d

dev = torch.device("cuda:0")
torch.backends.cudnn.benchmark = True


def t(fn, it=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it


for (c, hw) in [(64, 112), (64, 56), (128, 28), (256, 14), (512, 7)]:
    x = torch.randn(256, c, hw, hw, device=dev, requires_grad=True)
    g = torch.randn_like(x)
    bn = nn.BatchNorm2d(c).to(dev)
    res = {}
    for name, en in (("cudnn", True), ("native", False)):
        def f():
            with torch.backends.cudnn.flags(enabled=en):
                y = bn(x)
            y.backward(g)
        res[name] = t(f)
    fb = FusedBatchNorm2d(c).to(dev)

    def f2():
        y = fb(x)
        y.backward(g)
    res["fused"] = t(f2)
    gb = x.numel() * 4 * 5 / 1e9
    print(f"C={c} HW={hw}: cudnn {res['cudnn']:.3f} ms  native {res['native']:.3f} ms  fused {res['fused']:.3f} ms  (5 passes {gb:.2f} GB -> {gb/6.5:.3f} ms at 6.5TB/s)")


from paper_2304_07741_b200.post import FusedMaxPool2d

x = torch.relu(torch.randn(256, 64, 112, 112, device=dev)).requires_grad_(True)
g = torch.randn(256, 64, 56, 56, device=dev)
tp = nn.MaxPool2d(3, 2, 1)
fp = FusedMaxPool2d(3, 2, 1)
for name, mod in (("torch", tp), ("fused", fp)):
    def f(mod=mod):
        y = mod(x)
        y.backward(g)
    def fwd(mod=mod):
        with torch.no_grad():
            mod(x)
    print(f"maxpool 3x3s2 256x64x112^2 {name}: fwd {t(fwd):.3f} ms  fwd+bwd {t(f):.3f} ms")
