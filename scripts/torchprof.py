"""Top CUDA kernels of the bench step under torch.profiler (analysis only — never a bench number)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

import bench  # noqa: E402

kernel = sys.argv[1] if len(sys.argv) > 1 else "seed7_k1"
torch.backends.cudnn.allow_tf32 = False
torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.benchmark = True
dev = torch.device("cuda:0")
m = bench.build_model(kernel, dev) if kernel != "none" else __import__("torchvision").models.resnet18().to(dev)
opt = torch.optim.SGD(m.parameters(), lr=0.01, momentum=0.9)
x = torch.randn(256, 3, 224, 224, device=dev)
y = torch.randint(0, 1000, (256,), device=dev)


def step():
    opt.zero_grad(set_to_none=True)
    F.cross_entropy(m(x), y).backward()
    opt.step()


for _ in range(4):
    step()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        step()
    torch.cuda.synchronize()
ev = prof.key_averages()
rows = sorted(ev, key=lambda e: -e.device_time_total)
tot = sum(e.device_time_total for e in ev)
print(f"total device time per step: {tot / 2 / 1000:.2f} ms")
for e in rows[:30]:
    print(f"{e.device_time_total / 2 / 1000:8.3f} ms/step {100 * e.device_time_total / tot:5.1f}%  x{e.count // 2:4d}  {e.key[:110]}")
