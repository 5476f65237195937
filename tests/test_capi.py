"""The C-ABI library loads, exports exactly what include/canvas_b200.h declares,
and validates blobs before touching the driver (no GPU needed)."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_2304_07741_b200 import executor, zoo

HDR = Path(__file__).resolve().parents[1] / "include" / "canvas_b200.h"


def declared():
    text = HDR.read_text()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(canvas_\w+)\(", text, re.M)))


def test_exports_every_declared_symbol():
    lib = executor.load_library()
    names = declared()
    assert len(names) >= 9
    for n in names:
        assert hasattr(lib, n), n


def test_abi_version_matches_blob():
    from paper_2304_07741_b200.lowering import ABI_VERSION

    assert executor.load_library().canvas_abi_version() == ABI_VERSION


def _create(blob):
    lib = executor.load_library()
    h = ctypes.c_void_p()
    rc = lib.canvas_plan_create(blob, len(blob), 0, ctypes.byref(h))
    return rc, lib.canvas_last_error().decode()


def test_bad_blob_rejected():
    rc, msg = _create(b"not a blob at all")
    assert rc == -1 and "magic" in msg


def test_version_rejected():
    p = executor.plan_for(zoo.NEG, c_in=8, c_out=8, h=4, w=4)
    b = bytearray(p.blob())
    b[8] = 99
    rc, msg = _create(bytes(b))
    assert rc == -2


def test_truncated_blob_rejected():
    p = executor.plan_for(zoo.SEED7_K1, c_in=8, c_out=8, h=4, w=4)
    rc, msg = _create(p.blob()[:-7])
    assert rc == -1


def test_valid_blob_reaches_device_check():
    """A well-formed blob parses; without a B200 the call fails loudly (no fallback)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu tests")
    p = executor.plan_for(zoo.SEED7_K1, c_in=16, c_out=32, h=8, w=8, stride=2)
    rc, msg = _create(p.blob())
    assert rc == -4 and ("libcuda" in msg or "cuInit" in msg)


def test_module_refuses_cpu():
    import torch

    from paper_2304_07741_b200.module import CanvasConv2d

    m = CanvasConv2d(zoo.SEED7_K1, 8, 8)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        m(torch.randn(1, 8, 6, 6))


def test_canvas_module_copy_and_pickle_drop_plan_cache():
    """a used CanvasConv2d holds ctypes plan handles; deepcopy / pickle
    must drop that cache instead of failing."""
    import copy
    import io

    import torch

    from paper_2304_07741_b200 import zoo
    from paper_2304_07741_b200.module import CanvasConv2d

    m = CanvasConv2d(zoo.SEED7_K1, 16, 32, 3)
    m._plans[(8, 8, 0)] = object()  # stands in for a DevicePlan (ctypes handle)
    m2 = copy.deepcopy(m)
    assert m2._plans == {} and m._plans
    buf = io.BytesIO()
    torch.save(m, buf)
    buf.seek(0)
    m3 = torch.load(buf, weights_only=False)
    assert m3._plans == {} and all(torch.equal(a, b) for a, b in zip(m3.weights, m.weights))
