"""Print GPU-vs-oracle parity ratios (<=1 passes) for the pinned kernels — a debug aid."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import numpy as np  # noqa: E402

from paper_2304_07741_b200 import zoo  # noqa: E402
from parity import elementwise_ratio, normwise_ratio, reference  # noqa: E402
from test_gpu_parity import run_gpu  # noqa: E402

for name in sys.argv[1:] or ["im2col", "seed7_k1"]:
    case = reference(zoo.ALL[name], 64, 64, 20, 20, n=2)
    y, dx, dws = run_gpu(case)
    r = {"y": elementwise_ratio(y, case.y.numpy()), "dx": elementwise_ratio(dx, case.dx.numpy())}
    for i, (a, b) in enumerate(zip(dws, case.dw)):
        r[f"dw{i}"] = normwise_ratio(a, b.numpy())
    bad = np.abs(y - case.y.numpy()) > 1e-5 + 1e-4 * np.abs(case.y.numpy())
    idx = np.argwhere(bad)[:8]
    print(name, {k: round(v, 3) for k, v in r.items()}, "bad y:", int(bad.sum()), idx.tolist())
