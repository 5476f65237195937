"""Debug probe: which images of seed-7 #1 at batch 256 disagree with the fp64 oracle, and why."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np, torch
from oracle import torch_ref as R
from paper_2304_07741_b200 import zoo
from paper_2304_07741_b200.executor import device_plan, plan_for, solve_target

n, c, hw = 256, 64, 56
text = zoo.SEED7_K1
plan = plan_for(text, c_in=c, c_out=c, h=hw, w=hw)
t, a = solve_target(text, c_in=c, c_out=c, h=hw, w=hw)
ck = R.concretize(t, a)
dp = device_plan(plan, 0)
dev = torch.device("cuda:0")
wts = R.init_weights(ck, copies=1, seed=2, dtype=torch.float32)[0]
x = torch.randn(n, c, hw, hw, generator=torch.Generator().manual_seed(0))
dy = torch.randn(n, c, hw, hw, generator=torch.Generator().manual_seed(1))
xd, dyd, wd = x.to(dev), dy.to(dev), [w.to(dev) for w in wts]
sb, wb = dp.sizes(n)
saved = torch.empty(max(sb, 1), dtype=torch.uint8, device=dev)
work = torch.empty(max(wb, 1), dtype=torch.uint8, device=dev)
y = torch.empty((n, c, hw, hw), device=dev)
dx = torch.empty_like(xd)
dws = [torch.empty_like(w) for w in wd]
st = torch.cuda.current_stream().cuda_stream
dp.forward(xd, wd, y, saved, st)
dp.backward(xd, wd, saved, dyd, dx, dws, work, st)
torch.cuda.synchronize()
dx = dx.cpu().numpy()
w64 = [w.double() for w in wts]
for c0 in range(0, n, 16):
    xr = x[c0:c0 + 16].double().requires_grad_(True)
    gaps = {}
    class P(R.NearTies):
        def note(self, a_, b_):
            d = (a_ - b_).abs(); rel = d / torch.maximum(a_.abs(), b_.abs()).clamp_min(1e-300)
            rel = torch.where(d > 0, rel, torch.full_like(rel, 1.0))
            m = rel.reshape(rel.shape[0], -1).min(1).values
            gaps.setdefault("g", []).append(m)
    with P() as p:
        yr = R.conv_replacement(ck, xr, [w64], c, c, 1)
    yr.backward(dy[c0:c0 + 16].double())
    g = torch.stack(gaps["g"]).min(0).values
    r = np.abs(dx[c0:c0 + 16] - xr.grad.numpy()) / (1e-5 + 1e-4 * np.abs(xr.grad.numpy()))
    for i in range(16):
        if r[i].max() > 1:
            bad = np.argwhere(r[i] > 1)
            print("image", c0 + i, "ratio", float(r[i].max()), "nbad", len(bad), "pix", sorted({(int(b[1]), int(b[2])) for b in bad})[:4], "min rel gap", float(g[i]), flush=True)
print("done")
