"""GPU parity: the sm_100a executor (through the C ABI) vs the fp64 CPU oracle.

Covers every pinned kernel, Fig.-2 replication in both
directions with the stride-2 policy, the first 20 kernels of the reference
sampler (nodes=10, seed=7), the im2col calibration against cuDNN-free
F.conv2d semantics, determinism, and the CanvasConv2d module path.
"""

import numpy as np
import pytest
import torch

from paper_2304_07741_b200 import zoo
from parity import assert_close, reference

pytestmark = pytest.mark.gpu


def run_gpu(case):
    from paper_2304_07741_b200.executor import device_plan

    dev = torch.device("cuda:0")
    dp = device_plan(case.plan, 0)
    x = case.x.float().to(dev)
    ws = [w.float().to(dev).contiguous() for c in case.weights for w in c]
    n = x.shape[0]
    saved_b, ws_b = dp.sizes(n)
    y = torch.full(tuple(case.y.shape), float("nan"), device=dev)
    saved = torch.empty(max(saved_b, 1), dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    dp.forward(x, ws, y, saved, st)
    dy = case.dy.float().to(dev)
    dx = torch.full_like(x, float("nan")) if case.plan.stride == 1 else torch.full_like(x, 7.0)
    dws = [torch.full_like(w, float("nan")) for w in ws]
    work = torch.empty(max(ws_b, 1), dtype=torch.uint8, device=dev)
    dp.backward(x, ws, saved, dy, dx, dws, work, st)
    torch.cuda.synchronize()
    return y.cpu().numpy(), dx.cpu().numpy(), [d.cpu().numpy() for d in dws]


@pytest.mark.parametrize("name", list(zoo.ALL))
def test_pinned_config1(name):
    """Config-1 shapes (C=64, 56x56), batch 2."""
    case = reference(zoo.ALL[name], 64, 64, 56, 56, n=2)
    y, dx, dws = run_gpu(case)
    assert_close(case, y, dx, dws, name)


@pytest.mark.parametrize("cin,cout,stride", [(16, 32, 2), (32, 16, 1), (16, 64, 2), (16, 16, 2)])
@pytest.mark.parametrize("name", ["seed7_k1", "im2col", "involution", "seed7_k0"])
def test_replication_and_stride(name, cin, cout, stride):
    case = reference(zoo.ALL[name], cin, cout, 14, 13, stride=stride, n=3)
    y, dx, dws = run_gpu(case)
    assert_close(case, y, dx, dws, f"{name} {cin}->{cout} s{stride}")


def _sweep(path):
    text = open(path).read()
    return ["canvas-ir v1\n" + t for t in text.split("canvas-ir v1\n")[1:]]


@pytest.mark.parametrize("i", range(20))
def test_sampler_sweep_first20(i):
    texts = _sweep("tests/golden/sampler_10_7_20.cir")
    case = reference(texts[i], 32, 32, 12, 12, n=2)
    y, dx, dws = run_gpu(case)
    assert_close(case, y, dx, dws, f"sweep #{i}")


def test_deterministic():
    case = reference(zoo.SEED7_K1, 64, 64, 28, 28, n=4)
    a = run_gpu(case)
    b = run_gpu(case)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert all(np.array_equal(u, v) for u, v in zip(a[2], b[2]))


def test_im2col_is_conv():
    """SPEC.md:509 derived oracle: unfold(h); unfold(w); fc(C) == conv2d(padding=1)."""
    case = reference(zoo.IM2COL, 64, 64, 20, 20, n=2)
    y, _, _ = run_gpu(case)
    w = case.weights[0][0].view(64, 64, 3, 3)
    ref = torch.nn.functional.conv2d(case.x, w, padding=1).numpy()
    assert np.max(np.abs(y - ref)) <= 1e-5 + 1e-4 * np.max(np.abs(ref))


def test_module_autograd():
    from paper_2304_07741_b200.module import CanvasConv2d

    torch.manual_seed(0)
    m = CanvasConv2d(zoo.SEED7_K1, 32, 64, 3, stride=2).cuda()
    x = torch.randn(3, 32, 16, 16, device="cuda", requires_grad=True)
    y = m(x)
    assert y.shape == (3, 64, 8, 8)
    y.square().sum().backward()
    assert x.grad is not None and torch.isfinite(x.grad).all()
    assert all(p.grad is not None and torch.isfinite(p.grad).all() for p in m.weights)


def test_candidate_evaluator_real_worker():
    from paper_2304_07741_b200.evaluator import CandidateEvaluator

    texts = _sweep("tests/golden/sampler_10_7_20.cir")[:3]
    res = CandidateEvaluator([0], shapes={"batch": 2, "h": 16, "w": 16, "c_in": 16, "c_out": 16}).run(texts, timeout_s=600)
    assert [r.status for r in res] == ["ok"] * 3, [r.error for r in res]
    assert all(r.fwd_ms > 0 and r.bwd_ms > 0 for r in res)


@pytest.mark.parametrize("name", ["seed7_k1", "im2col", "involution"])
@pytest.mark.parametrize("cin,cout,hw,stride", [(256, 512, 14, 2), (512, 512, 7, 1), (128, 256, 28, 2)])
def test_wide_channels(name, cin, cout, hw, stride):
    """ResNet-18 stage-3/4 widths: multi-tile N (dgrad N = 9C split over tiles),
    persistent and 16-producer-warp GEMM variants, packed weight images > 1 tile."""
    case = reference(zoo.ALL[name], cin, cout, hw, hw, stride=stride, n=2)
    y, dx, dws = run_gpu(case)
    assert_close(case, y, dx, dws, f"{name} {cin}->{cout} {hw}^2 s{stride}")


@pytest.mark.parametrize("golden,count", [("sampler_16_7_64.cir", 64), ("sampler_20_0_16.cir", 16)])
def test_larger_sampled_kernels(golden, count):
    """Every kernel of the reference's nodes=16 (64 kernels) and nodes=20 (16
    kernels) sweeps, through the C ABI vs the fp64 oracle at a small shape with
    Fig.-2 replication (C_in=16 -> C_out=32, stride 2)."""
    texts = _sweep(f"tests/golden/{golden}")
    assert len(texts) == count
    bad = []
    for i, t in enumerate(texts):
        case = reference(t, 16, 32, 10, 9, stride=2, n=2)
        try:
            assert_close(case, *run_gpu(case), f"{golden} #{i}")
        except AssertionError as e:
            bad.append(str(e)[:200])
    assert not bad, bad[:5]


@pytest.mark.parametrize("name", ["seed7_k1", "im2col"])
def test_wgrad_row_groups(name, monkeypatch):
    """The JG = 2 wgrad variant (two 128-row tiles per CTA sharing the gathered
    output-channel operand; off by default) at a stage-2 width."""
    from paper_2304_07741_b200 import executor, lowering

    monkeypatch.setattr(lowering, "TC_WGRAD_JG_MAX", 2)
    executor._plan_cached.cache_clear()
    try:
        case = reference(zoo.ALL[name], 128, 128, 28, 28, n=2)
        assert ", 16, 2>(a)" in case.plan.source  # tc_gemm_wgrad<F, NT, STAGES, PW, JG = 2>
        y, dx, dws = run_gpu(case)
        assert_close(case, y, dx, dws, f"{name} JG=2")
    finally:
        executor._plan_cached.cache_clear()


@pytest.mark.parametrize("cin,cout,hw,stride", [(64, 64, 16, 1), (64, 128, 16, 2), (128, 128, 8, 1)])
def test_dgrad_bcast_epilogue(cin, cout, hw, stride, monkeypatch):
    """The dgrad whose TMEM epilogue applies the input broadcast's adjoint
    (CANVAS_EPI_BC=1, off by default): seed-7 #1 vs the fp64 oracle."""
    from paper_2304_07741_b200 import executor, lowering

    monkeypatch.setattr(lowering, "EPI_BC", True)
    executor._plan_cached.cache_clear()
    try:
        case = reference(zoo.SEED7_K1, cin, cout, hw, hw, stride=stride, n=2)
        assert "EPI_BC = true" in case.plan.source
        y, dx, dws = run_gpu(case)
        assert_close(case, y, dx, dws, f"epi-bc {cin}->{cout} {hw}^2 s{stride}")
    finally:
        executor._plan_cached.cache_clear()


@pytest.mark.parametrize("cin,cout,hw,k", [(24, 144, 14, 1), (144, 24, 14, 1), (16, 96, 16, 1), (16, 16, 12, 3), (8, 8, 12, 3)])
@pytest.mark.parametrize("name", ["seed7_k1", "im2col", "involution"])
def test_narrow_targets(name, cin, cout, hw, k):
    """MobileNetV2-style narrow 1x1 targets and C = 8/16 3x3 targets: tensor-core
    wgrad with J = 8..24 rows of the 128-row tile and N = 16 columns."""
    case = reference(zoo.ALL[name], cin, cout, hw, hw, k=k, n=2)
    y, dx, dws = run_gpu(case)
    assert_close(case, y, dx, dws, f"{name} {cin}->{cout} {hw}^2 k{k}")


@pytest.mark.parametrize("n", [4, 2])
@pytest.mark.parametrize("name", ["seed7_k1", "im2col", "involution"])
def test_image_quad_wgrad(name, n, monkeypatch):
    """ResNet stage-4 geometry (7x7, S % 4 != 0): image-quad wgrad producers (F::NQ,
    CANVAS_VEC_NQ=1, off by default) at batch 4, the scalar fallback at batch 2."""
    from paper_2304_07741_b200 import executor, lowering

    monkeypatch.setattr(lowering, "VEC_NQ", True)
    executor._plan_cached.cache_clear()
    case = reference(zoo.ALL[name], 128, 128, 7, 7, n=n)
    executor._plan_cached.cache_clear()
    assert "NQ = true" in case.plan.source
    assert_close(case, *run_gpu(case), f"{name} NQ n{n}")


@pytest.mark.parametrize("name,cin,hw", [("seed7_k1", 64, 16), ("im2col", 128, 8), ("seed7_k1", 128, 7), ("im2col", 64, 12), ("seed7_k1", 96, 9)])
def test_fc_forward_tmem_a(name, cin, hw, monkeypatch):
    """FC forward with the computed operand staged in tensor memory (tcgen05.mma
    with A from TMEM, producers writing it with tcgen05.st; CANVAS_TMEMA=1, off by
    default) vs the fp64 oracle."""
    from paper_2304_07741_b200 import executor, lowering

    monkeypatch.setattr(lowering, "TC_TMEMA", True)
    executor._plan_cached.cache_clear()
    try:
        case = reference(zoo.ALL[name], cin, cin, hw, hw, n=2)
        assert "tc_gemm_pix_tmema" in case.plan.source
        assert_close(case, *run_gpu(case), f"{name} tmem-A {cin} {hw}^2")
    finally:
        executor._plan_cached.cache_clear()


@pytest.mark.parametrize("cin,hw,stride,n", [(512, 7, 1, 3), (256, 14, 2, 2), (64, 5, 1, 5)])
@pytest.mark.parametrize("name", ["seed7_k1", "im2col", "involution"])
@pytest.mark.parametrize("fwd", [False, True])
def test_padded_quad_wgrad(name, cin, hw, stride, n, fwd, monkeypatch):
    """S % 4 != 0 (ResNet stage 4, 7x7): wgrad producers (and with CANVAS_VEC_PAD_FWD=1
    the FC forward / dgrad producers) on pixel quads over a per-image range padded to
    a multiple of 4 (padding lanes masked to zero / padding columns not stored)."""
    from paper_2304_07741_b200 import executor, lowering

    monkeypatch.setattr(lowering, "VEC_PAD_MIN_LOADS", 1)
    monkeypatch.setattr(lowering, "VEC_PAD_FWD", fwd)
    if fwd:
        monkeypatch.setattr(lowering, "TC_TMEMA", "0")  # the padded quad smem forward, not TMEM-A
    executor._plan_cached.cache_clear()
    try:
        case = reference(zoo.ALL[name], cin, cin, hw, hw, stride=stride, n=n)
        ho = -(-hw // stride)
        assert f"SP = {-(-ho * ho // 4) * 4}," in case.plan.source
        assert_close(case, *run_gpu(case), f"{name} pad {cin} {hw}^2 s{stride} n{n} fwd={fwd}")
    finally:
        executor._plan_cached.cache_clear()
