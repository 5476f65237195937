"""Debug: one sampler_20_0_16 kernel (16 -> 32, stride 2, 10x9) on the GPU vs the oracle."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from parity import reference, elementwise_ratio
from test_gpu_parity import run_gpu
texts = ["canvas-ir v1\n" + t for t in open(os.path.join(ROOT, "tests/golden/sampler_20_0_16.cir")).read().split("canvas-ir v1\n")[1:]]
i = int(sys.argv[1]) if len(sys.argv) > 1 else 5
case = reference(texts[i], 16, 32, 10, 9, stride=2, n=2)
y, dx, dws = run_gpu(case)
print("y", elementwise_ratio(y, case.y.numpy()), "dx", elementwise_ratio(dx, case.dx.numpy()))
bad = np.argwhere(np.abs(dx - case.dx.numpy()) > 1e-5 + 1e-4 * np.abs(case.dx.numpy()))
print("bad dx", len(bad), bad[:10].tolist())
print("sample gpu", dx.ravel()[:8], "ref", case.dx.numpy().ravel()[:8])
