"""Shared parity harness (TEST INFRASTRUCTURE): oracle fp64 vs executor (GPU or host emulator).

Inputs follow SURVEY §8d: x ~ N(0,1) seed 0, dy ~ N(0,1) seed 1, FC weights
U(+-1/sqrt(fan_in)) seed 2 in IR edge order per replica — drawn on the CPU so
both sides see identical bits.

Tolerances (north star): activations and dgrad elementwise |a-b| <= 1e-5 +
1e-4 |b| against the fp64 oracle; wgrad normwise (SURVEY §7 hard part 1:
even exact fp32 fails elementwise on ~0.19% of dW entries of a long
reduction) ||a-b||_inf <= 1e-5 + 1e-4 ||b||_inf.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from oracle import torch_ref as R
from paper_2304_07741_b200.executor import plan_for, solve_target

RTOL, ATOL = 1e-4, 1e-5


@dataclass
class Case:
    x: torch.Tensor  # fp64
    weights: list  # [copy][fc] fp64
    dy: torch.Tensor
    y: torch.Tensor
    dx: torch.Tensor
    dw: list  # flat fp64
    plan: object


def reference(text, cin, cout, h, w, stride=1, n=2, g=4, k=3, xs=None) -> Case:
    p = plan_for(text, c_in=cin, c_out=cout, h=h, w=w, k=k, g=g, stride=stride, xs=xs)
    t, a = solve_target(text, c_in=cin, c_out=cout, h=h, w=w, k=k, g=g, stride=stride, xs=xs)
    ck = R.concretize(t, a)
    x = torch.randn(n, cin, h, w, generator=torch.Generator().manual_seed(0), dtype=torch.float32).double()
    wts = R.init_weights(ck, copies=p.copies, seed=2, dtype=torch.float32)
    wts = [[w_.double() for w_ in c] for c in wts]
    xr = x.clone().requires_grad_(True)
    wr = [[w_.clone().requires_grad_(True) for w_ in c] for c in wts]
    y = R.conv_replacement(ck, xr, wr, cin, cout, stride)
    dy = torch.randn(y.shape, generator=torch.Generator().manual_seed(1), dtype=torch.float32).double()
    y.backward(dy)
    return Case(x, wts, dy, y.detach(), xr.grad, [w_.grad for c in wr for w_ in c], p)


def elementwise_ratio(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0
    fin = np.isfinite(b)
    return float(np.max(np.abs(a[fin] - b[fin]) / (ATOL + RTOL * np.abs(b[fin])))) if fin.any() else 0.0


def normwise_ratio(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / (ATOL + RTOL * np.max(np.abs(b))))


def assert_close(case: Case, y, dx, dws, what: str = "") -> dict:
    r = {"y": elementwise_ratio(y, case.y.numpy()), "dx": elementwise_ratio(dx, case.dx.numpy())}
    for i, (a, b) in enumerate(zip(dws, case.dw)):
        r[f"dw{i}"] = normwise_ratio(a, b.numpy())
    bad = {k: v for k, v in r.items() if not v <= 1.0}
    assert not bad, f"{what} parity failure (ratio to tolerance > 1): {bad}"
    return r


def oracle_checker(ir_text: str, shapes: dict, y, dx, dws) -> dict:
    """Parity checker for CandidateEvaluator (its ``checker`` hook): re-draws the
    evaluator's seeded inputs (same recipe: evaluator.parity_inputs / §8d),
    runs the fp64 oracle and compares with the north-star tolerances."""
    case = reference(ir_text, shapes["c_in"], shapes["c_out"], shapes["h"], shapes["w"], stride=shapes.get("stride", 1), n=y.shape[0], g=shapes.get("g", 4), k=shapes.get("k", 3))
    try:
        r = assert_close(case, y, dx, dws, "evaluator parity sample")
        return {"ok": True, "ratios": {k: round(v, 4) for k, v in r.items()}}
    except AssertionError as e:
        return {"ok": False, "error": str(e)[:300]}
