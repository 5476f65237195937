"""Lowering correctness on the CPU: generated functors + launch schedule run
through the host emulator (tests/emu) vs the fp64 oracle, same tolerances as
the GPU parity tests.  Covers every pinned kernel, Fig.-2 replication (concat
and sum) with the stride-2 policy, and ALL 256 kernels of the reference
sampler sweep (nodes=10, seed=7; 48 with free variables)."""

import multiprocessing
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np
import pytest

from emu.runner import EmuPlan
from paper_2304_07741_b200 import zoo
from parity import assert_close, reference


def emu_run(case):
    ep = EmuPlan(case.plan)
    flat = [w.float().numpy().copy() for c in case.weights for w in c]
    x = case.x.float().numpy().copy()
    y, saved = ep.forward(x, flat)
    dx, dws = ep.backward(x, flat, saved, case.dy.float().numpy().copy())
    return y, dx, dws


@pytest.mark.parametrize("name", list(zoo.ALL))
def test_pinned(name):
    case = reference(zoo.ALL[name], 16, 16, 10, 9)
    assert_close(case, *emu_run(case), name)


@pytest.mark.parametrize("h,w", [(6, 12), (6, 14), (7, 4)])
@pytest.mark.parametrize("name", ["seed7_k1", "involution", "im2col", "seed7_k0"])
def test_vector_producers(name, h, w):
    """S % 4 == 0: the tcgen05 operand functors are emitted in 4-pixel form (W % 4
    == 0: lane-affine pixel coordinates; W = 14: per-lane (h, w) copies) and the
    emulated GEMMs evaluate them on pixel quads."""
    case = reference(zoo.ALL[name], 16, 16, h, w)
    if name != "seed7_k0":  # seed-7 #0 has no FC
        assert "static constexpr bool VEC = true" in case.plan.source
    assert_close(case, *emu_run(case), f"{name} vec {h}x{w}")


@pytest.mark.parametrize("n", [4, 2])
@pytest.mark.parametrize("name", ["seed7_k1", "im2col", "involution"])
def test_image_quad_wgrad(name, n, monkeypatch):
    """7x7 targets (S % 4 != 0): the wgrad producers take quads of 4 images at one
    pixel (F::NQ, entries pixel-major; CANVAS_VEC_NQ=1, off by default); batch 2
    exercises the scalar fallback."""
    from paper_2304_07741_b200 import executor, lowering

    monkeypatch.setattr(lowering, "VEC_NQ", True)
    executor._plan_cached.cache_clear()
    case = reference(zoo.ALL[name], 32, 32, 7, 7, n=n)
    executor._plan_cached.cache_clear()
    assert "NQ = true" in case.plan.source
    assert_close(case, *emu_run(case), f"{name} NQ n{n}")


@pytest.mark.parametrize("hw,stride,n", [(7, 1, 2), (7, 1, 3), (14, 2, 2), (5, 1, 3)])
@pytest.mark.parametrize("name", ["seed7_k1", "im2col", "involution"])
@pytest.mark.parametrize("fwd", [False, True])
def test_padded_quad_wgrad(name, hw, stride, n, fwd, monkeypatch):
    """Targets with S % 4 != 0 (7x7: 49 pixels): the wgrad producers (and, with
    CANVAS_VEC_PAD_FWD=1, off by default, the FC forward / dgrad producers) run pixel
    quads over a range padded to SP = 52 per image (padding lanes masked, zero on the
    output-channel side; padding columns not stored), odd batches included."""
    from paper_2304_07741_b200 import executor, lowering

    monkeypatch.setattr(lowering, "VEC_PAD_MIN_LOADS", 1)  # every kernel, not only gather-bound ones
    monkeypatch.setattr(lowering, "VEC_PAD_FWD", fwd)
    monkeypatch.setattr(lowering, "TC_TMEMA", "0")  # the quad smem forward (TMEM-A takes K <= 1024 by default)
    executor._plan_cached.cache_clear()
    try:
        case = reference(zoo.ALL[name], 32, 32, hw, hw, stride=stride, n=n)
        ho = -(-hw // stride)
        sp = -(-ho * ho // 4) * 4
        assert f"SP = {sp}," in case.plan.source and "VEC = true" in case.plan.source
        if fwd and name != "involution":  # involution's FCs (K = 32) take the persistent path
            assert f"SP = {sp};" in case.plan.source
        assert_close(case, *emu_run(case), f"{name} pad {hw}^2 s{stride} n{n} fwd={fwd}")
    finally:
        executor._plan_cached.cache_clear()


@pytest.mark.parametrize("cin,cout,hw,k", [(24, 144, 8, 1), (144, 24, 8, 1), (16, 96, 8, 1), (8, 8, 6, 3)])
@pytest.mark.parametrize("name", ["seed7_k1", "im2col", "involution"])
def test_narrow_targets(name, cin, cout, hw, k):
    """Narrow targets (MobileNetV2 1x1, C = 8): tensor-core wgrad with J < 32 rows."""
    case = reference(zoo.ALL[name], cin, cout, hw, hw, k=k, n=2)
    assert_close(case, *emu_run(case), f"{name} {cin}->{cout} k{k}")


@pytest.mark.parametrize("cin,cout,stride", [(32, 32, 1), (32, 64, 2), (64, 32, 1)])
def test_dgrad_bcast_epilogue(cin, cout, stride, monkeypatch):
    """seed-7 #1's K = 9C FC reads bcast(min)(n7, unfold(softmax)): its dgrad epilogue
    writes the rhs edge contribution and the replica-summed lhs gradient (no
    materialised dL/dv, no replica-sum launch).  Off by default (slower on the
    B200); CANVAS_EPI_BC=1 selects it."""
    from paper_2304_07741_b200 import executor, lowering

    monkeypatch.setattr(lowering, "EPI_BC", True)
    executor._plan_cached.cache_clear()
    try:
        case = reference(zoo.SEED7_K1, cin, cout, 6, 8, stride=stride, n=2)
        assert "EPI_BC = true" in case.plan.source
        assert not any(L.what == "grad n7" for L in case.plan.launches)
        assert_close(case, *emu_run(case), f"epi-bc {cin}->{cout} s{stride}")
    finally:
        executor._plan_cached.cache_clear()


def _epi_on():
    from paper_2304_07741_b200 import lowering

    lowering.EPI_BC = True


def _epi_sweep(i):
    import torch

    torch.set_num_threads(1)
    texts = ["canvas-ir v1\n" + t for t in open("tests/golden/sampler_10_7_256.cir").read().split("canvas-ir v1\n")[1:]]
    case = reference(texts[i], 32, 32, 4, 4)
    if "EPI_BC = true" not in case.plan.source:
        return None, False
    try:
        assert_close(case, *emu_run(case), f"sweep #{i} (epi-bc)")
    except AssertionError as e:
        return str(e), True
    return None, True


def test_dgrad_bcast_epilogue_sweep():
    """Every kernel of the first 96 of the 256-kernel sweep whose FC reads a
    broadcast (at C = 32, where its dgrad is a tensor-core GEMM)."""
    with ProcessPoolExecutor(min(8, os.cpu_count() or 1), mp_context=multiprocessing.get_context("spawn"), initializer=_epi_on) as ex:
        res = list(ex.map(_epi_sweep, range(96)))
    errs = [e for e, _ in res if e]
    assert not errs, errs[:5]
    assert sum(used for _, used in res) >= 3


@pytest.mark.parametrize("cin,cout,stride", [(8, 16, 2), (16, 8, 1), (8, 32, 2)])
@pytest.mark.parametrize("name", ["seed7_k1", "involution", "seed7_k0"])
def test_replication(name, cin, cout, stride):
    case = reference(zoo.ALL[name], cin, cout, 9, 10, stride=stride, n=2)
    assert_close(case, *emu_run(case), f"{name} {cin}->{cout} s{stride}")


def _one(i):
    import torch

    torch.set_num_threads(1)
    texts = ["canvas-ir v1\n" + t for t in open("tests/golden/sampler_10_7_256.cir").read().split("canvas-ir v1\n")[1:]]
    case = reference(texts[i], 16, 16, 8, 8)
    try:
        assert_close(case, *emu_run(case), f"sweep #{i}")
    except AssertionError as e:
        return str(e)
    return None


def test_sampler_sweep_256():
    with ProcessPoolExecutor(min(8, os.cpu_count() or 1), mp_context=multiprocessing.get_context("spawn")) as ex:
        errs = [e for e in ex.map(_one, range(256)) if e]
    assert not errs, errs[:5]


def test_blob_roundtrip_fields():
    from paper_2304_07741_b200.executor import plan_for

    p = plan_for(zoo.SEED7_K1, c_in=64, c_out=128, h=56, w=56, stride=2)
    b = p.blob()
    assert b[:8] == b"CNVSBLOB"
    assert p.copies == 2 and p.mode == "concat" and p.y_copy_off == 64 * 28 * 28
    assert np.frombuffer(b[8:16], np.int64)[0] == 1


@pytest.fixture
def planes_everywhere(monkeypatch):
    """Lower with plane-major pointwise launches down to 1-pixel planes."""
    from paper_2304_07741_b200 import executor, lowering

    monkeypatch.setattr(lowering, "PLANES_MIN_S", 1)
    executor._plan_cached.cache_clear()
    yield
    executor._plan_cached.cache_clear()


@pytest.mark.parametrize("name", list(zoo.ALL))
def test_plane_major_pointwise(name, planes_everywhere):
    case = reference(zoo.ALL[name], 16, 32, 10, 9, stride=2)
    assert_close(case, *emu_run(case), f"{name} plane-major")


def test_plane_major_sweep_first40(planes_everywhere):
    """Plane-major functors (every eligible launch, down to 1-pixel planes)
    over the first 40 sweep kernels; at least some launches must use them."""
    from paper_2304_07741_b200.executor import plan_for

    assert "pointwise_planes" in plan_for(zoo.SEED7_K1, c_in=16, c_out=16, h=8, w=7).source
    texts = ["canvas-ir v1\n" + t for t in open("tests/golden/sampler_10_7_256.cir").read().split("canvas-ir v1\n")[1:]]
    for i in range(40):
        case = reference(texts[i], 16, 16, 8, 7)
        assert_close(case, *emu_run(case), f"sweep #{i} plane-major")


@pytest.mark.parametrize("cin,cout,stride", [(32, 32, 1), (32, 64, 2), (64, 32, 1)])
def test_operand_writeback(cin, cout, stride, monkeypatch):
    """seed-7 #1's K=9C FC: the forward GEMM writes its computed operand and the
    wgrad reads it back (SAVE_B), per Fig.-2 copy (optional path, off by default)."""
    from paper_2304_07741_b200 import executor, lowering

    monkeypatch.setattr(lowering, "SAVE_OPERAND", True)
    executor._plan_cached.cache_clear()
    case = reference(zoo.SEED7_K1, cin, cout, 9, 8, stride=stride, n=2)
    executor._plan_cached.cache_clear()
    assert "SAVE_B = true" in case.plan.source
    assert_close(case, *emu_run(case), f"write-back {cin}->{cout} s{stride}")


def _nvcc_plan(i):
    import shutil
    import subprocess
    import tempfile

    from paper_2304_07741_b200.executor import plan_for

    texts = ["canvas-ir v1\n" + t for t in open("tests/golden/sampler_10_7_256.cir").read().split("canvas-ir v1\n")[1:]]
    p = plan_for(texts[i], c_in=64, c_out=64, h=56, w=56, k=3, g=4)
    d = tempfile.mkdtemp()
    try:
        with open(f"{d}/p.cu", "w") as f:
            f.write(p.source)
        r = subprocess.run([os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc"), "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17", "-cubin", "-I", "paper_2304_07741_b200/csrc/kernels", "-diag-suppress", "177", f"{d}/p.cu", "-o", f"{d}/p.cubin"], capture_output=True, text=True)
        return None if r.returncode == 0 else f"#{i}: " + " | ".join(l for l in r.stderr.splitlines() if "error" in l)[:300]
    finally:
        shutil.rmtree(d, ignore_errors=True)


@pytest.mark.skipif(not os.path.exists(os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")), reason="nvcc not present")
def test_sweep_256_plans_compile_for_sm100a():
    """Every kernel of the 256-kernel sweep lowers at config-1 shapes (C=64,
    56x56) to code ptxas accepts for sm_100a (shared-memory limits, register
    budgets) — the build check the GPU's NVRTC would otherwise fail at run time."""
    with ProcessPoolExecutor(min(16, os.cpu_count() or 1), mp_context=multiprocessing.get_context("spawn")) as ex:
        errs = [e for e in ex.map(_nvcc_plan, range(256)) if e]
    assert not errs, errs[:5]


@pytest.mark.parametrize("name", ["seed7_k1", "seed7_k0", "involution"])
def test_gradient_siblings(name, monkeypatch):
    """CANVAS_GRAD_SIBLINGS=1 (off by default): two gradient tensors of one shape in
    one launch when every gradient the second reads is already written."""
    from paper_2304_07741_b200 import executor, lowering

    monkeypatch.setattr(lowering, "GRAD_SIBLINGS", True)
    executor._plan_cached.cache_clear()
    try:
        case = reference(zoo.ALL[name], 16, 16, 10, 9)
        if name == "seed7_k1":
            assert any(L.what == "grad n7 + n1" for L in case.plan.launches)
        assert_close(case, *emu_run(case), f"{name} siblings")
    finally:
        executor._plan_cached.cache_clear()


@pytest.mark.parametrize("cin,hw", [(64, 8), (128, 7), (256, 5)])
def test_ksplit_small_fc(cin, hw):
    """Few pixels, long reduction: fc(G) with its K = C loop split over lanes
    (canvas::pointwise_ks), the partial sums reduced before the store."""
    case = reference(zoo.SEED7_K1, cin, cin, hw, hw, n=2)
    assert any("K split" in L.what for L in case.plan.launches), [L.what for L in case.plan.launches]
    assert_close(case, *emu_run(case), f"seed7_k1 {cin} {hw}x{hw}")
