"""Index-map pinning with an iota payload (TEST INFRASTRUCTURE).

SURVEY §8c item 2 / north star "all Unfold/Shift/Group index maps must be
bit-exact".  A kernel's *index maps* — Group reshapes, Shift/Unfold affine
maps with their per-stage zero predicates (App. A.2-A.3), Broadcast tile
order r mod L (A.8), FC flat channel index (A.4), Fig.-2 copy offsets and
the stride-2 subsample (A.10) — are checked bit-for-bit by running the
kernel's *iota form*:

* every value op is swapped for one that is exact on integers while the
  graph, its shapes and every rearrangement / broadcast edge stay as they
  are: ``ew(*)`` and ``softmax`` -> ``ew(neg)``, ``fold(avg)`` ->
  ``fold(max)``, ``bcast(mul)`` -> ``bcast(add)`` (add/sub/min/max kept);
* x and dy are iotas (distinct integers 1..numel, < 2^22 after every add so
  3xTF32 carries them exactly), FC weights are one-hot selection matrices
  W[o, (7o+3) mod K] = 1, so an FC output *is* its input at one flat channel
  index.

Every forward value is then an exact integer computed purely from source
positions: a wrong index map, a dropped or misplaced zero predicate, a wrong
broadcast replica or copy offset changes the bits.  The oracle runs the same
iota form in fp64 (exact) and the device (or host emulator) result must be
*equal* to it.  Backward values are gathers/sums of dy integers with tie
splits by 1/2 or 1/count; they are compared bit-exactly where the oracle's
value is an fp32 number whose every partial sum is exact (checked by
``exact_fp32``), within the fp32 tolerance otherwise.
"""

from __future__ import annotations

import re
from dataclasses import dataclass

import numpy as np
import torch

from oracle import torch_ref as R
from paper_2304_07741_b200.executor import plan_for, solve_target

_EDGE = re.compile(r"^(e: )(\w+)\(([^)]*)\)(.*)$")


def iota_form(text: str, keep_relu_abs: bool = False) -> str:
    """The kernel with every value op replaced by an integer-exact one (module
    doc); ``keep_relu_abs`` keeps relu / abs (exact on integers, and the ops
    whose sub-gradient at 0 the tie payload exercises, App. A.5)."""
    out = []
    for line in text.splitlines():
        m = _EDGE.match(line)
        if m:
            head, op, arg, rest = m.groups()
            if op == "softmax" or (op == "ew" and not (keep_relu_abs and arg in ("relu", "abs"))):
                op, arg = "ew", "neg"
            elif op == "fold":
                arg = arg.replace("avg", "max")
            elif op == "bcast" and arg == "mul":
                arg = "add"
            line = f"{head}{op}({arg}){rest}"
        out.append(line)
    return "\n".join(out) + "\n"


def one_hot_weights(ck, copies: int) -> list[list[torch.Tensor]]:
    out = []
    for j in range(copies):
        ws = []
        for o, k in R.fc_weight_shapes(ck):
            w = torch.zeros(o, k, dtype=torch.float64)
            w[torch.arange(o), (7 * torch.arange(o) + 3 + j) % k] = 1.0
            ws.append(w)
        out.append(ws)
    return out


@dataclass
class IotaCase:
    x: torch.Tensor
    weights: list
    dy: torch.Tensor
    y: torch.Tensor
    dx: torch.Tensor
    dw: list
    plan: object
    text: str
    ties: bool = False


def iota_reference(text: str, cin, cout, h, w, stride=1, n=2, g=4, k=3, xs=None, ties: bool = False) -> IotaCase:
    """``ties=False``: iota payload (distinct values: index maps).  ``ties=True``:
    small integers in [-2, 2] (x) / [-3, 3] (dy), seed 0 / 1, so that nearly
    every max / min / fold-max / relu / abs sees exact ties and zeros — the
    App. A.5/A.6/A.8 tie rules decide the backward (both sides take the same
    branch: every forward value is an exact integer on both)."""
    t_iota = iota_form(text, keep_relu_abs=ties)
    p = plan_for(t_iota, c_in=cin, c_out=cout, h=h, w=w, k=k, g=g, stride=stride, xs=xs)
    t, a = solve_target(t_iota, c_in=cin, c_out=cout, h=h, w=w, k=k, g=g, stride=stride, xs=xs)
    ck = R.concretize(t, a)
    if ties:
        x = torch.randint(-2, 3, (n, cin, h, w), generator=torch.Generator().manual_seed(0)).double()
    else:
        x = torch.arange(1, n * cin * h * w + 1, dtype=torch.float64).reshape(n, cin, h, w)
    wts = one_hot_weights(ck, p.copies)
    xr = x.clone().requires_grad_(True)
    wr = [[w_.clone().requires_grad_(True) for w_ in c] for c in wts]
    y = R.conv_replacement(ck, xr, wr, cin, cout, stride)
    if ties:
        dy = torch.randint(-3, 4, tuple(y.shape), generator=torch.Generator().manual_seed(1)).double()
    else:
        dy = torch.arange(1, y.numel() + 1, dtype=torch.float64).reshape(y.shape)
    y.backward(dy)
    assert float(y.detach().abs().max()) < 2**22, "iota payload too large for exact 3xTF32"
    return IotaCase(x, wts, dy, y.detach(), xr.grad, [w_.grad for c in wr for w_ in c], p, t_iota, ties)


def exact_fp32(b: np.ndarray) -> np.ndarray:
    """Mask of oracle values that are exact small dyadic numbers (integers or
    halves / quarters of integers below 2^20): every fp32 evaluation order of
    their sums is then exact, so the device must reproduce them bit-for-bit."""
    b = np.asarray(b, np.float64)
    return (np.abs(b) < 2**20) & (np.round(b * 4) == b * 4)


def compare(case: IotaCase, y, dx, dws, what: str = "") -> dict:
    """y must equal the oracle bit-for-bit; dx bit-for-bit on exact entries and
    within 1e-4 rel / 1e-5 abs elsewhere; dW normwise (SURVEY §7 hard part 1).
    Tie payloads compare every dx entry within the tolerance: a tie split by
    1/3 is inexact in fp32 even where the fp64 sum of the splits is an
    integer, while a wrong tie rule is off by >= 1/2 of a gradient term."""
    yb = case.y.numpy()
    y = np.asarray(y, np.float64)
    bad_y = int(np.count_nonzero(y != yb))
    dxb = case.dx.numpy()
    dx = np.asarray(dx, np.float64)
    ex = exact_fp32(dxb) if not case.ties else np.zeros(dxb.shape, bool)
    bad_dx = int(np.count_nonzero(dx[ex] != dxb[ex]))
    tol = np.abs(dx[~ex] - dxb[~ex]) > 1e-5 + 1e-4 * np.abs(dxb[~ex])
    bad_dx_tol = int(np.count_nonzero(tol))
    bad_dw = []
    for i, (a, b) in enumerate(zip(dws, case.dw)):
        b = b.numpy()
        if np.max(np.abs(np.asarray(a, np.float64) - b)) > 1e-5 + 1e-4 * np.max(np.abs(b)):
            bad_dw.append(i)
    r = {"y_mismatch": bad_y, "y_n": int(yb.size), "dx_exact_mismatch": bad_dx, "dx_exact_n": int(ex.sum()), "dx_tol_fail": bad_dx_tol, "dw_fail": bad_dw}
    assert bad_y == 0 and bad_dx == 0 and bad_dx_tol == 0 and not bad_dw, f"{what} iota mismatch: {r}"
    return r
