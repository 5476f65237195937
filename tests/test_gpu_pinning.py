"""GPU pinning of the parity that the reference leaves unpinned (VERDICT r1
"next" #1), through the C ABI on the B200:

* index maps bit-exact: the iota form of ALL 256 sweep kernels (tests/iota.py)
  — every forward value and every (exact) dx entry equal to the fp64 oracle;
* tie rules: the tie payload over the same 256 kernels, plus constructed-tie
  fixtures for fold-max, bcast min/max, relu/abs at 0 and unfold zero padding
  (App. A.5/A.6/A.8);
* Fig.-2 replication (concat / sum) and the stride-2 policy under both payloads;
* config-1 shapes exactly (N=8, C=64, 56x56) for the pinned kernels;
* the bench's layer shape at the bench's batch (seed-7 #1, 256 x 64 x 56^2),
  checked against the fp64 oracle over every image (chunked);
* a parity sample inside the candidate evaluator (config 4): kernels timed at
  config-1 shapes, the same plan checked at batch 2 by the oracle checker.
"""

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

from iota import compare, iota_reference
from paper_2304_07741_b200 import zoo
from parity import assert_close, oracle_checker, reference

pytestmark = pytest.mark.gpu


def _texts(name="sampler_10_7_256.cir"):
    return ["canvas-ir v1\n" + t for t in open(f"tests/golden/{name}").read().split("canvas-ir v1\n")[1:]]


def run_gpu(case):
    from test_gpu_parity import run_gpu as rg

    return rg(case)


def _compile_all(plans):
    """Create the device plans on host threads (NVRTC runs outside the GIL)."""
    from paper_2304_07741_b200.executor import device_plan

    with ThreadPoolExecutor(16) as ex:
        list(ex.map(lambda p: device_plan(p, 0), plans))


@pytest.mark.parametrize("ties", [False, True], ids=["iota", "ties"])
def test_sweep256_index_maps_and_ties(ties):
    texts = _texts()
    cases = [iota_reference(t, 8, 16, 7, 6, n=2, ties=ties) for t in texts]
    _compile_all([c.plan for c in cases])
    bad, exact_dx = [], 0
    for i, c in enumerate(cases):
        try:
            r = compare(c, *run_gpu(c), f"#{i}")
            exact_dx += r["dx_exact_n"]
        except AssertionError as e:
            bad.append(str(e)[:200])
    assert not bad, (len(bad), bad[:5])
    if not ties:  # nearly every dx entry of the iota payload is exact (1/3 tie splits are not)
        assert exact_dx >= 0.999 * sum(c.dx.numel() for c in cases)


@pytest.mark.parametrize("ties", [False, True], ids=["iota", "ties"])
@pytest.mark.parametrize("cin,cout,stride", [(8, 16, 2), (16, 8, 1), (16, 8, 2), (16, 32, 1)])
def test_replication_stride_payloads(cin, cout, stride, ties):
    names = ["seed7_k1", "seed7_k0", "involution", "im2col", "neg"]
    cases = [iota_reference(zoo.ALL[n], cin, cout, 9, 10, stride=stride, n=2, ties=ties) for n in names]
    cases += [iota_reference(t, cin, cout, 9, 10, stride=stride, n=2, ties=ties) for t in _texts()[:24]]
    _compile_all([c.plan for c in cases])
    for i, c in enumerate(cases):
        compare(c, *run_gpu(c), f"case {i} {cin}->{cout} s{stride} ties={ties}")


# Constructed-tie fixtures: each isolates one tie rule on integer payloads.
TIE_FIXTURES = {
    # fold-max ties (even split, A.6) after abs (abs'(0) = 0, A.5)
    "fold_max_abs": """canvas-ir v1
n0: shape=[C; H, W]
n1: shape=[C; H, W]
n2: shape=[C; W]
n3: shape=[C; H, W]
e: ew(abs) (0) -> 1
e: fold(dim=1,max) (1) -> 2
e: bcast(mul) (2,0) -> 3
# bcast@3: prefix=[C] suffix=[W] M=H subs={}
""",
    # unfold zero padding ties with x <= 0 in a max over the unfold dim (A.3 + A.6), relu'(0) = 0
    "unfold_pad_max_relu": """canvas-ir v1
n0: shape=[C; H, W]
n1: shape=[C, KH; H, W]
n2: shape=[C; H, W]
n3: shape=[C; H, W]
n4: shape=[C; H, W]
e: unfold(h) (0) -> 1
e: fold(dim=1,max) (1) -> 2
e: ew(relu) (0) -> 3
e: bcast(mul) (2,3) -> 4
# bcast@4: prefix=[] suffix=[H, W] M=1 subs={}
""",
    # bcast min / max ties (1/2 - 1/2 split, A.8) between x and its shifted copy
    "bcast_min_max_shift": """canvas-ir v1
n0: shape=[C; H, W]
n1: shape=[C; H, W]
n2: shape=[C; H, W]
n3: shape=[C; H, W]
e: shift(h,+1) (0) -> 1
e: bcast(min) (1,0) -> 2
# bcast@2: prefix=[] suffix=[H, W] M=1 subs={}
e: bcast(max) (2,0) -> 3
# bcast@3: prefix=[] suffix=[H, W] M=1 subs={}
""",
}


def _tie_case(text, lo, hi, n=2, cin=8, cout=8, h=9, w=10):
    """Integer payload in [lo, hi]: forward values exact on both sides, so both
    take the same tie branches; gradients compared at the fp32 tolerance."""
    from oracle import torch_ref as R
    from paper_2304_07741_b200.executor import plan_for, solve_target

    p = plan_for(text, c_in=cin, c_out=cout, h=h, w=w)
    t, a = solve_target(text, c_in=cin, c_out=cout, h=h, w=w)
    ck = R.concretize(t, a)
    x = torch.randint(lo, hi + 1, (n, cin, h, w), generator=torch.Generator().manual_seed(0)).double()
    wts = [[] for _ in range(p.copies)]
    xr = x.clone().requires_grad_(True)
    y = R.conv_replacement(ck, xr, wts, cin, cout, 1)
    dy = torch.randint(-3, 4, tuple(y.shape), generator=torch.Generator().manual_seed(1)).double()
    y.backward(dy)
    from parity import Case

    return Case(x, wts, dy, y.detach(), xr.grad, [], p)


@pytest.mark.parametrize("lo,hi", [(-1, 1), (-2, 0), (0, 1)])
@pytest.mark.parametrize("name", list(TIE_FIXTURES))
def test_constructed_ties(name, lo, hi):
    case = _tie_case(TIE_FIXTURES[name], lo, hi)
    y, dx, _ = run_gpu(case)
    assert np.array_equal(y, case.y.numpy()), f"{name}: forward must be exact on integers"
    assert_close(case, y, dx, [], f"{name} ties [{lo},{hi}]")
    # the fixture really exercises ties: some gradient entry is a fraction
    frac = np.abs(case.dx.numpy() * 2 - np.round(case.dx.numpy() * 2)) > 0
    half = np.abs(case.dx.numpy() - np.round(case.dx.numpy())) > 0
    assert half.any() or frac.any() or name == "unfold_pad_max_relu"


@pytest.mark.parametrize("name", ["seed7_k1", "seed7_k0", "im2col", "involution"])
def test_config1_exact_shape(name):
    """Config 1 exactly: N=8, C=64, H=W=56, G=4, K=3."""
    case = reference(zoo.ALL[name], 64, 64, 56, 56, n=8)
    assert_close(case, *run_gpu(case), f"{name} config 1")


def test_bench_layer_batch256():
    """The bench's dominant layer at the bench's batch: seed-7 #1 replacing a
    layer1 conv, 256 x 64 x 56 x 56, against the fp64 oracle over all 256
    images (16-image chunks; dW summed over the chunks in fp64).

    At this size a few of the ~10^9 forward min/max decisions compare values
    that differ by less than the device's rounding of them (measured: 7
    pixels of 802,816 flip at batch 256); the fp64 oracle and the fp32 device
    order those pairs differently and route a whole gradient term to the other
    operand.  The oracle flags such decisions (``NearTies``: nonzero gaps below
    3e-5 relative + 1e-6 absolute; 1.4% of pixels after a 3x3 dilation, which
    covers all 7 measured flips); dy is zeroed there on both sides so no gradient goes through
    them, and y, dx of every image and the batch dW are compared at the
    north-star tolerances."""
    from oracle import torch_ref as R
    from paper_2304_07741_b200.executor import device_plan, plan_for, solve_target

    n, c, hw, chunk = 256, 64, 56, 16
    text = zoo.SEED7_K1
    plan = plan_for(text, c_in=c, c_out=c, h=hw, w=hw)
    t, a = solve_target(text, c_in=c, c_out=c, h=hw, w=hw)
    ck = R.concretize(t, a)
    x = torch.randn(n, c, hw, hw, generator=torch.Generator().manual_seed(0), dtype=torch.float32)
    dy = torch.randn(n, c, hw, hw, generator=torch.Generator().manual_seed(1), dtype=torch.float32)
    wts = R.init_weights(ck, copies=1, seed=2, dtype=torch.float32)[0]
    w64 = [w.double() for w in wts]
    pix = []
    with torch.no_grad():
        for c0 in range(0, n, chunk):
            with R.NearTies(rel=3e-5, abs_tol=1e-6, hw=(hw, hw)) as nt:
                R.conv_replacement(ck, x[c0 : c0 + chunk].double(), [w64], c, c, 1)
            pix.append(nt.pixels)
    # the decisions of seed-7 #1 sit at the output pixel (n7, n8 = min(n7, unfold(n1))):
    # dy = 0 there (dilated by the 3x3 unfold) removes every gradient they route
    flagged = torch.nn.functional.max_pool2d(torch.cat(pix).view(n, 1, hw, hw).float(), 3, 1, 1) > 0
    frac = float(flagged.float().mean())
    assert frac < 0.03, f"{frac:.2%} of pixels near-tied"  # measured 1.4%
    dy = dy * (~flagged).float()
    dev = torch.device("cuda:0")
    dp = device_plan(plan, 0)
    xd, dyd = x.to(dev), dy.to(dev)
    wd = [w.to(dev) for w in wts]
    sb, wb = dp.sizes(n)
    saved = torch.empty(max(sb, 1), dtype=torch.uint8, device=dev)
    work = torch.empty(max(wb, 1), dtype=torch.uint8, device=dev)
    y = torch.full((n, c, hw, hw), float("nan"), device=dev)
    dx = torch.full_like(xd, float("nan"))
    dws = [torch.full_like(w, float("nan")) for w in wd]
    st = torch.cuda.current_stream().cuda_stream
    dp.forward(xd, wd, y, saved, st)
    dp.backward(xd, wd, saved, dyd, dx, dws, work, st)
    torch.cuda.synchronize()
    y, dx, dws = y.cpu().numpy(), dx.cpu().numpy(), [d.cpu().numpy() for d in dws]
    wr = [w.clone().requires_grad_(True) for w in w64]
    worst = {"y": 0.0, "dx": 0.0}
    for c0 in range(0, n, chunk):
        xr = x[c0 : c0 + chunk].double().requires_grad_(True)
        yr = R.conv_replacement(ck, xr, [wr], c, c, 1)
        yr.backward(dy[c0 : c0 + chunk].double())
        for k, a_, b_ in (("y", y[c0 : c0 + chunk], yr.detach().numpy()), ("dx", dx[c0 : c0 + chunk], xr.grad.numpy())):
            r = float(np.max(np.abs(a_ - b_) / (1e-5 + 1e-4 * np.abs(b_))))
            worst[k] = max(worst[k], r)
    for i, w in enumerate(wr):
        b = w.grad.numpy()
        worst[f"dw{i}"] = float(np.max(np.abs(dws[i] - b)) / (1e-5 + 1e-4 * np.max(np.abs(b))))
    assert all(v <= 1.0 for v in worst.values()), (worst, frac)
    print("batch-256 layer parity (ratio to tolerance):", worst, f"near-tie pixels (dy zeroed): {frac:.2%}")


def test_evaluator_parity_sample():
    """Config 4 with a parity sample: the first 32 kernels of the 256 sweep are
    timed at config-1 shapes and the same plans checked at batch 2 against the
    fp64 oracle (checker injected; the evaluator never imports the oracle)."""
    from paper_2304_07741_b200.evaluator import CandidateEvaluator

    texts = _texts()[:32]
    res = CandidateEvaluator([0], prefetch=8, parity_batch=2, checker=oracle_checker).run(texts, timeout_s=1500)
    st = [r.status for r in res]
    assert all(s in ("ok", "nonfinite") for s in st), [(r.task_id, r.status, r.error, r.extra.get("parity")) for r in res if r.status not in ("ok", "nonfinite")]
    checked = [r for r in res if r.status == "ok"]
    assert len(checked) >= 30 and all(r.extra["parity"]["ok"] for r in checked)
