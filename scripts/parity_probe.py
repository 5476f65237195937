"""Print GPU-vs-oracle parity ratios (<=1 passes) — a debug aid.
    python scripts/parity_probe.py name[:cin:cout:hw:stride] ..."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import numpy as np  # noqa: E402

from paper_2304_07741_b200 import zoo  # noqa: E402
from parity import elementwise_ratio, normwise_ratio, reference  # noqa: E402
from test_gpu_parity import run_gpu  # noqa: E402

for spec in sys.argv[1:] or ["im2col", "seed7_k1"]:
    name, *dims = spec.split(":")
    cin, cout, hw, stride = (list(map(int, dims)) + [64, 64, 20, 1][len(dims):]) if dims else (64, 64, 20, 1)
    case = reference(zoo.ALL[name], cin, cout, hw, hw, stride=stride, n=2)
    y, dx, dws = run_gpu(case)
    r = {"y": elementwise_ratio(y, case.y.numpy()), "dx": elementwise_ratio(dx, case.dx.numpy())}
    for i, (a, b) in enumerate(zip(dws, case.dw)):
        r[f"dw{i}"] = normwise_ratio(a, b.numpy())
    print(spec, {k: round(v, 3) for k, v in r.items()}, [L.what for L in case.plan.launches])
    for key, got, want in [("y", y, case.y.numpy()), ("dx", dx, case.dx.numpy())]:
        bad = np.abs(got - want) > 1e-5 + 1e-4 * np.abs(want)
        if bad.any():
            idx = np.argwhere(bad)
            print(f"  {key}: {int(bad.sum())} bad of {bad.size}; first {idx[:6].tolist()}; channels {sorted(set(idx[:, 1].tolist()))[:20]}")
    for i, (a, b) in enumerate(zip(dws, case.dw)):
        b = b.numpy()
        err = np.abs(a - b)
        print(f"  dw{i} shape {a.shape} max err {err.max():.3g} at {np.unravel_index(err.argmax(), err.shape)}, |b|max {np.abs(b).max():.3g}")
