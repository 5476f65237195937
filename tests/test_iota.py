"""Index maps and tie rules pinned bit-exactly on the CPU (host emulator of the
generated functors, tests/emu) — see tests/iota.py.  The same sweeps run on the
B200 through the C ABI in tests/test_gpu_pinning.py.

* iota payload, ALL 256 kernels of the reference sweep (nodes=10, seed=7):
  every forward value equal to the fp64 oracle bit-for-bit, every dx entry
  too (they are exact dyadic numbers), dW normwise;
* tie payload (integers in [-2, 2]) over the same 256 kernels: forward equal
  bit-for-bit, the tie-split backward within tolerance;
* both payloads on the pinned kernels with Fig.-2 replication (concat and
  sum) and the stride-2 policy.
"""

import multiprocessing
import os
from concurrent.futures import ProcessPoolExecutor

import pytest

from emu.runner import EmuPlan
from iota import compare, iota_form, iota_reference
from paper_2304_07741_b200 import zoo


def emu_run(case):
    ep = EmuPlan(case.plan)
    flat = [w.float().numpy().copy() for c in case.weights for w in c]
    x = case.x.float().numpy().copy()
    y, saved = ep.forward(x, flat)
    dx, dws = ep.backward(x, flat, saved, case.dy.float().numpy().copy())
    return y, dx, dws


def _texts():
    return ["canvas-ir v1\n" + t for t in open("tests/golden/sampler_10_7_256.cir").read().split("canvas-ir v1\n")[1:]]


def _one(args):
    i, ties = args
    import torch

    torch.set_num_threads(1)
    try:
        case = iota_reference(_texts()[i], 8, 16, 7, 6, n=2, ties=ties)
        compare(case, *emu_run(case), f"sweep #{i} ties={ties}")
    except AssertionError as e:
        return str(e)[:300]
    return None


@pytest.mark.parametrize("ties", [False, True])
def test_sweep256(ties):
    with ProcessPoolExecutor(min(8, os.cpu_count() or 1), mp_context=multiprocessing.get_context("spawn")) as ex:
        errs = [e for e in ex.map(_one, [(i, ties) for i in range(256)]) if e]
    assert not errs, errs[:5]


@pytest.mark.parametrize("ties", [False, True])
@pytest.mark.parametrize("cin,cout,stride", [(8, 16, 2), (16, 8, 1), (16, 8, 2)])
@pytest.mark.parametrize("name", ["seed7_k1", "seed7_k0", "involution", "im2col"])
def test_pinned_replication(name, cin, cout, stride, ties):
    case = iota_reference(zoo.ALL[name], cin, cout, 9, 10, stride=stride, n=2, ties=ties)
    compare(case, *emu_run(case), f"{name} {cin}->{cout} s{stride} ties={ties}")


def test_iota_form_keeps_structure():
    """The iota form changes value ops only: same nodes, shapes, edges and inputs."""
    t = iota_form(zoo.SEED7_K1)
    assert "softmax" not in t and "ew(neg) (0) -> 1" in t
    assert t.count("\n") == zoo.SEED7_K1.count("\n")
    keep = [ln for ln in zoo.SEED7_K1.splitlines() if not ln.startswith("e: ")]
    assert keep == [ln for ln in t.splitlines() if not ln.startswith("e: ")]
    assert iota_form(zoo.SEED7_K0, keep_relu_abs=True).count("ew(abs)") == 1


@pytest.mark.parametrize("lo,hi", [(-1, 1), (-2, 0), (0, 1)])
@pytest.mark.parametrize("name", ["fold_max_abs", "unfold_pad_max_relu", "bcast_min_max_shift"])
def test_constructed_ties_emulated(name, lo, hi):
    """The constructed-tie fixtures of tests/test_gpu_pinning.py on the host emulator."""
    import numpy as np

    from parity import assert_close
    from test_gpu_pinning import TIE_FIXTURES, _tie_case

    case = _tie_case(TIE_FIXTURES[name], lo, hi)
    y, dx, dws = emu_run(case)
    assert np.array_equal(y, case.y.numpy())
    assert_close(case, y, dx, [], f"{name} [{lo},{hi}]")
