"""Teacher-forced layer check (analysis helper): capture one Canvas layer's real
input and output-gradient inside a network pass, rerun the layer through the
C ABI and the fp64 oracle with exactly those tensors, and report where they
differ (and whether the oracle has a near-tie there)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import torch_ref as R  # noqa: E402
from paper_2304_07741_b200 import backbones, zoo  # noqa: E402
from paper_2304_07741_b200.executor import solve_target  # noqa: E402
from paper_2304_07741_b200.module import CanvasConv2d  # noqa: E402

name, layer = sys.argv[1], sys.argv[2]
torch.backends.cudnn.allow_tf32 = False
m, _ = backbones.build(name, zoo.SEED7_K1)
m = m.cuda().eval()
mod = dict(m.named_modules())[layer]
cap = {}
mod.register_forward_hook(lambda md, i, o: cap.update(x=i[0].detach().clone(), y=o.detach().clone()))
mod.register_full_backward_hook(lambda md, gi, go: cap.update(dx=gi[0].detach().clone(), dy=go[0].detach().clone()))
c, h, w = backbones.SPECS[name]["input"]
x = torch.randn(4, c, min(h, 64), min(w, 64), generator=torch.Generator().manual_seed(0)).cuda().requires_grad_(True)
out = m(x)
out.backward(torch.randn(out.shape, generator=torch.Generator().manual_seed(1)).cuda())
dws = [p.grad.detach().cpu().double() for p in mod.weights]
t, a = solve_target(mod.ir_text, c_in=mod.in_channels, c_out=mod.out_channels, h=cap["x"].shape[2], w=cap["x"].shape[3], k=mod.kernel_size, g=mod.g, stride=mod.stride, xs=mod.xs)
ck = R.concretize(t, a)
xr = cap["x"].cpu().double().requires_grad_(True)
wr = [p.detach().cpu().double().requires_grad_(True) for p in mod.weights]
nf = len(wr) // mod.copies
yr = R.conv_replacement(ck, xr, [wr[i * nf:(i + 1) * nf] for i in range(mod.copies)], mod.in_channels, mod.out_channels, mod.stride)
yr.backward(cap["dy"].cpu().double())
def ratio(a, b):
    return np.abs(a - b) / (1e-5 + 1e-4 * np.abs(b))
ry = ratio(cap["y"].cpu().double().numpy(), yr.detach().numpy())
rdx = ratio(cap["dx"].cpu().double().numpy(), xr.grad.numpy())
print(layer, "y max ratio", ry.max(), "dx max ratio", rdx.max(), "dx elements > 1:", int((rdx > 1).sum()), "of", rdx.size)
for i, (g_, r_) in enumerate(zip(dws, wr)):
    e = float((g_ - r_.grad).norm() / r_.grad.norm())
    print(f"  dw{i} normwise rel {e:.2e}", "max elem ratio", float(ratio(g_.numpy(), r_.grad.numpy()).max()))
print("zeros in layer input:", float((cap["x"] == 0).float().mean()))
