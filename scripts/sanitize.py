"""compute-sanitizer driver (run under `compute-sanitizer --tool T python scripts/sanitize.py`):
one fwd+bwd through the C ABI for every pinned kernel at a small shape, the Fig.-2
stride-2 concat case and the tensor-core paths (wide channels, so the tcgen05
templates with their mbarrier / TMEM / bulk-copy pipelines run), plus the dense
stem conv.  TEST INFRASTRUCTURE: checks only that the launches are clean; the
numerics are the parity tests' job."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2304_07741_b200 import zoo  # noqa: E402
from paper_2304_07741_b200.executor import device_plan, plan_for  # noqa: E402


def run(text, cin, cout, hw, stride=1, n=2):
    p = plan_for(text, c_in=cin, c_out=cout, h=hw, w=hw, k=3, g=4, stride=stride)
    dp = device_plan(p, 0)
    dev = torch.device("cuda:0")
    x = torch.randn(n, cin, hw, hw, device=dev)
    ho = hw // stride
    y = torch.empty(n, cout, ho, ho, device=dev)
    g = torch.Generator().manual_seed(2)
    from oracle import torch_ref as R
    from paper_2304_07741_b200.executor import solve_target

    t, a = solve_target(text, c_in=cin, c_out=cout, h=hw, w=hw, k=3, g=4, stride=stride)
    ws = [w.float().to(dev) for c in R.init_weights(R.concretize(t, a), copies=p.copies, seed=2, dtype=torch.float32) for w in c]
    del g
    saved_b, ws_b = dp.sizes(n)
    saved = torch.empty(max(saved_b, 1), dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    dp.forward(x, ws, y, saved, st)
    dx = torch.empty_like(x)
    dws = [torch.empty_like(w) for w in ws]
    work = torch.empty(max(ws_b, 1), dtype=torch.uint8, device=dev)
    dp.backward(x, ws, saved, torch.randn_like(y), dx, dws, work, st)
    torch.cuda.synchronize()
    print(f"ok {text.splitlines()[1] if len(text.splitlines()) > 1 else ''} {cin}->{cout} {hw}^2 s{stride}: fwd {dp.launches(0)} bwd {dp.launches(1)} launches", flush=True)


def main():
    for name, text in zoo.ALL.items():
        run(text, 16, 16, 12)
    run(zoo.SEED7_K1, 16, 32, 12, stride=2)
    run(zoo.SEED7_K1, 64, 64, 16)  # tcgen05 fwd / persistent dgrad / wgrad
    run(zoo.IM2COL, 128, 128, 8)
    run(zoo.SEED7_K1, 256, 256, 8, n=1)
    run(zoo.SEED7_K1, 128, 128, 7)  # K-split small FC (pointwise_ks), padded-quad wgrad
    from paper_2304_07741_b200.dense_conv import TcConv2d

    conv = TcConv2d(3, 64, 7, stride=2, padding=3, bias=False).cuda()
    xx = torch.randn(2, 3, 64, 64, device="cuda", requires_grad=True)
    conv(xx).sum().backward()
    torch.cuda.synchronize()
    print("ok dense stem conv", flush=True)


if __name__ == "__main__":
    main()
