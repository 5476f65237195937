"""Per-target parity at the exact shapes a 64x64 (CIFAR: 32x32) pass of each
workload network produces (analysis helper; prints ratio-to-tolerance)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import torch  # noqa: E402

from paper_2304_07741_b200 import backbones, zoo  # noqa: E402
from paper_2304_07741_b200.module import CanvasConv2d  # noqa: E402
from parity import assert_close, reference  # noqa: E402
from test_gpu_parity import run_gpu  # noqa: E402

names = sys.argv[1:] or list(backbones.SPECS)
for name in names:
    m, _ = backbones.build(name, zoo.SEED7_K1, fuse_bn=False)
    shapes = {}

    def hook(mod, i, o):
        shapes.setdefault((mod.in_channels, mod.out_channels, mod.kernel_size, mod.stride, mod.g, i[0].shape[2], i[0].shape[3]), None)

    for x in m.modules():
        if isinstance(x, CanvasConv2d):
            x.register_forward_hook(hook)
    c, h, w = backbones.SPECS[name]["input"]
    m = m.cuda()
    with torch.no_grad():
        m(torch.randn(2, c, min(h, 64), min(w, 64), device="cuda"))
    for (ci, co, k, s, g, hh, ww) in shapes:
        case = reference(zoo.SEED7_K1, ci, co, hh, ww, stride=s, n=2, g=g, k=k)
        y, dx, dws = run_gpu(case)
        try:
            r = assert_close(case, y, dx, dws)
            print(name, (ci, co, k, s, g, hh, ww), "ok", {a: round(b, 3) for a, b in r.items()}, flush=True)
        except AssertionError as e:
            print(name, (ci, co, k, s, g, hh, ww), "FAIL", str(e)[:300], flush=True)
