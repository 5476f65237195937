import sys, os
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
from parity import reference
from test_gpu_parity import run_gpu
from paper_2304_07741_b200 import zoo
for (ci, co, hw, st, n) in [(256, 512, 14, 2, 2), (256, 256, 7, 1, 2), (64, 64, 7, 1, 2), (32, 32, 7, 1, 2), (512, 512, 7, 1, 3)]:
    case = reference(zoo.SEED7_K1, ci, co, hw, hw, stride=st, n=n)
    y, dx, dws = run_gpu(case)
    ref = [w.numpy() if hasattr(w, "numpy") else w for w in case.dw]
    for i, (g, r) in enumerate(zip(dws, ref)):
        r = np.asarray(r, dtype=np.float64).reshape(g.shape)
        err = np.abs(g - r)
        tol = 1e-5 + 1e-4 * np.abs(r).max()
        if err.max() > tol:
            bad = err > tol
            rows = np.nonzero(bad.any(1))[0]
            cols = np.nonzero(bad.any(0))[0]
            print(ci, co, hw, st, n, f"dw{i}", g.shape, "max", err.max(), "tol", tol, "bad rows", len(rows), rows[:10], "bad cols", len(cols), cols[:10], "nan", np.isnan(g).sum())
        else:
            print(ci, co, hw, st, n, f"dw{i} ok")
