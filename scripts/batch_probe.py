"""Debug probe: seed-7 #1 layer parity vs batch size (first 4 images checked)."""
import sys, os
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))), os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests")]
import numpy as np, torch
from oracle import torch_ref as R
from paper_2304_07741_b200 import zoo
from paper_2304_07741_b200.executor import device_plan, plan_for, solve_target

c, hw = int(os.environ.get("C", 64)), int(os.environ.get("HW", 56))
text = zoo.ALL[os.environ.get("K", "seed7_k1")]
plan = plan_for(text, c_in=c, c_out=c, h=hw, w=hw)
t, a = solve_target(text, c_in=c, c_out=c, h=hw, w=hw)
ck = R.concretize(t, a)
dp = device_plan(plan, 0)
dev = torch.device("cuda:0")
wts = R.init_weights(ck, copies=1, seed=2, dtype=torch.float32)[0]
for n in [int(v) for v in sys.argv[1:]]:
    x = torch.randn(n, c, hw, hw, generator=torch.Generator().manual_seed(0))
    dy = torch.randn(n, c, hw, hw, generator=torch.Generator().manual_seed(1))
    xd, dyd, wd = x.to(dev), dy.to(dev), [w.to(dev) for w in wts]
    sb, wb = dp.sizes(n)
    saved = torch.empty(max(sb, 1), dtype=torch.uint8, device=dev)
    work = torch.empty(max(wb, 1), dtype=torch.uint8, device=dev)
    y = torch.full((n, c, hw, hw), float("nan"), device=dev)
    dx = torch.full_like(xd, float("nan"))
    dws = [torch.full_like(w, float("nan")) for w in wd]
    st = torch.cuda.current_stream().cuda_stream
    dp.forward(xd, wd, y, saved, st)
    dp.backward(xd, wd, saved, dyd, dx, dws, work, st)
    torch.cuda.synchronize()
    out = {}
    reps = int(os.environ.get("REPS", "1"))
    if reps > 1:
        y0, dx0 = y.clone(), dx.clone()
        for _ in range(reps):
            dp.forward(xd, wd, y, saved, st)
            dp.backward(xd, wd, saved, dyd, dx, dws, work, st)
            torch.cuda.synchronize()
            print("rep identical y/dx:", bool(torch.equal(y, y0)), bool(torch.equal(dx, dx0)), "dx diff pixels:", torch.nonzero((dx != dx0).any(1)).tolist()[:8], flush=True)
    for lo in sorted({0, n // 2, n - 2} | set(int(v) for v in os.environ.get("LOS", "").split(",") if v)):
        xr = x[lo:lo + 2].double().requires_grad_(True)
        yr = R.conv_replacement(ck, xr, [[w.double() for w in wts]], c, c, 1)
        yr.backward(dy[lo:lo + 2].double())
        for k, a_, b_ in (("y", y[lo:lo + 2].cpu().numpy(), yr.detach().numpy()), ("dx", dx[lo:lo + 2].cpu().numpy(), xr.grad.numpy())):
            r = np.abs(a_ - b_) / (1e-5 + 1e-4 * np.abs(b_))
            out[f"{k}@{lo}"] = round(float(r.max()), 3)
            if r.max() > 1:
                idx = np.unravel_index(np.argmax(r), r.shape)
                out[f"{k}@{lo}_at"] = [int(i) for i in idx]
                out[f"{k}@{lo}_nbad"] = int((r > 1).sum())
                out[f"{k}@{lo}_badpix"] = sorted({(int(a), int(c), int(d)) for a, b, c, d in zip(*np.nonzero(r > 1))})[:6]
    print(n, sb, wb, out, flush=True)
