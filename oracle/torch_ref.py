"""Torch-on-CPU restatement of Canvas kernel numerics (TEST INFRASTRUCTURE).

``run_kernel`` executes one concrete kernel graph in topological order with
plain torch ops (fp64 for parity, fp32 for the CPU baseline timing), autograd
providing the backward pass.  Each primitive cites the semantic source it
follows; conventions the reference leaves open follow SURVEY.md App. A.

``CanvasConvRef`` wraps a kernel as a conv replacement (Fig.-2 replication,
stride policy) — the CPU "reference path" that bench.py's reference arm
times and that the GPU module is compared against.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.nn.functional as F

from paper_2304_07741_b200.canvas import ir as cir
from paper_2304_07741_b200.canvas.constraint_solver import proportional_values
from paper_2304_07741_b200.canvas.primitives import (
    Broadcast,
    ElementWise,
    Fold,
    FullyConnected,
    Group,
    Shift,
    Softmax,
    Unfold,
    spatial_position,
)
from paper_2304_07741_b200.canvas.shape_algebra import Assignment, evaluate
from paper_2304_07741_b200.canvas.shape_solver import match_broadcast


@dataclass
class Concrete:
    """A kernel template evaluated under one assignment."""

    template: object
    assignment: Assignment
    extents: list  # per node: tuple of ints (channels ++ spatials)
    nch: list  # per node: number of channel dims
    fc_edges: list  # edge indices of FCs, in IR edge order

    @property
    def dag(self):
        return self.template.dag


def concretize(template, assignment: Assignment) -> Concrete:
    ext, nch = [], []
    for s in template.dag.nodes:
        ext.append(tuple(evaluate(d, assignment) for d in s.dims()))
        nch.append(len(s.channels))
    fcs = [i for i, e in enumerate(template.dag.edges) if isinstance(e.inst.kind, FullyConnected)]
    return Concrete(template, assignment, ext, nch, fcs)


def from_ir(text: str, consts: dict, xs: dict | None = None) -> Concrete:
    t = cir.parse(text).template
    a = Assignment(dict(consts), dict(xs if xs is not None else proportional_values(t, consts)))
    return concretize(t, a)


def fc_weight_shapes(ck: Concrete) -> list[tuple[int, int]]:
    """[out, prod(in channels)] per FC edge (nn.Linear weight layout, App. A.4)."""
    shapes = []
    for i in ck.fc_edges:
        e = ck.dag.edges[i]
        src = e.inputs[0]
        k = math.prod(ck.extents[src][: ck.nch[src]])
        shapes.append((evaluate(e.inst.kind.out, ck.assignment), k))
    return shapes


def _shift(x: torch.Tensor, axis: int, off: int) -> torch.Tensor:
    """out[..., h, ...] = x[..., h+off, ...], zero outside."""
    n = x.shape[axis]
    out = torch.zeros_like(x)
    if abs(off) >= n:
        return out
    if off >= 0:
        out.narrow(axis, 0, n - off).copy_(x.narrow(axis, off, n - off))
    else:
        out.narrow(axis, -off, n + off).copy_(x.narrow(axis, 0, n + off))
    return out


def _shift_ad(x: torch.Tensor, axis: int, off: int) -> torch.Tensor:
    # differentiable formulation of _shift (pad + narrow)
    n = x.shape[axis]
    pad_shape = list(x.shape)
    pad_shape[axis] = abs(off)
    z = x.new_zeros(pad_shape)
    if off >= 0:
        return torch.cat([x, z], dim=axis).narrow(axis, off, n)
    return torch.cat([z, x], dim=axis).narrow(axis, 0, n)


def _unfold(x: torch.Tensor, axis: int, insert_axis: int, k: int) -> torch.Tensor:
    """U[..., kk@insert, ..., h] = x[..., h + kk - k//2, ...], zero padded."""
    parts = [_shift_ad(x, axis, kk - k // 2) for kk in range(k)]
    return torch.stack(parts, dim=insert_axis)


class NearTies:
    """Context manager recording where a max / min decision of the forward pass
    (bcast min/max, fold max) compares two values that differ by a nonzero
    amount below ``rel`` of their magnitude.

    Such a pair is a *branch the oracle cannot pin*: the fp64 oracle and an
    fp32 device (different rounding of the compared values — measured up to
    ~7e-6 relative after an FC's cancellation) may order it differently, and
    the backward then routes a whole gradient term to the other operand
    (App. A.6/A.8).  Exact ties (structural zeros, equal integers) are not
    near-ties: both sides see them exactly.

    ``flags`` [N]: images with any near-tie.  ``pixels`` [N, H*W] (when ``hw``
    is given): the output pixels of decisions whose operands are laid out
    [..., H*W] (bcast with the full spatial suffix); a near-tie that cannot be
    localised (other layouts, fold max) flags every pixel of its image.
    Large-batch parity tests zero dy at flagged pixels so no gradient flows
    through those decisions on either side.
    """

    active: "NearTies | None" = None

    def __init__(self, rel: float = 3e-5, hw: tuple | None = None, abs_tol: float = 0.0):
        self.rel = rel
        self.abs_tol = abs_tol
        self.hw = hw
        self.flags: torch.Tensor | None = None
        self.pixels: torch.Tensor | None = None

    def __enter__(self):
        NearTies.active = self
        return self

    def __exit__(self, *exc):
        NearTies.active = None

    def _add(self, nb: int, img: torch.Tensor, pix: torch.Tensor | None) -> None:
        self.flags = img if self.flags is None else self.flags | img
        if self.hw is not None:
            S = self.hw[0] * self.hw[1]
            if pix is None:
                pix = img[:, None].expand(nb, S)
            self.pixels = pix.clone() if self.pixels is None else self.pixels | pix

    def note(self, a: torch.Tensor, b: torch.Tensor) -> None:
        with torch.no_grad():
            d = (a - b).abs()
            near = (d > 0) & (d <= self.rel * torch.maximum(a.abs(), b.abs()) + self.abs_tol)
            nb = near.shape[0]
            img = near.reshape(nb, -1).any(1)
            pix = None
            if self.hw is not None and near.shape[-1] == self.hw[0] * self.hw[1]:
                pix = near.reshape(nb, -1, near.shape[-1]).any(1)
            self._add(nb, img, pix)

    def note_fold_max(self, x: torch.Tensor, dim: int) -> None:
        if x.shape[dim] < 2:
            return
        with torch.no_grad():
            top = x.topk(2, dim=dim).values
            a, b = top.select(dim, 0), top.select(dim, 1)
            d = (a - b).abs()
            near = (d > 0) & (d <= self.rel * torch.maximum(a.abs(), b.abs()) + self.abs_tol)
            self._add(near.shape[0], near.reshape(near.shape[0], -1).any(1), None)


def run_kernel(ck: Concrete, x: torch.Tensor, weights: list[torch.Tensor]) -> torch.Tensor:
    """Forward of one kernel copy: x [N, *node0 extents] -> output node tensor."""
    vals: dict[int, torch.Tensor] = {0: x}
    fc_iter = iter(weights)
    nb = x.shape[0]
    for e in ck.dag.edges:  # topological by construction (ref ir.py:147-148)
        kind = e.inst.kind
        src = vals[e.inputs[0]]
        sin = e.inputs[0]
        nch_in = ck.nch[sin]
        out_ext = ck.extents[e.out]
        if isinstance(kind, Group):
            y = src.reshape((nb, *out_ext))  # pure view, x = g*(X/G)+j
        elif isinstance(kind, Shift):
            ax = 1 + nch_in + spatial_position(e.inst.inputs[0], kind.axis)
            y = _shift_ad(src, ax, kind.offset)
        elif isinstance(kind, Unfold):
            ax = 1 + nch_in + spatial_position(e.inst.inputs[0], kind.axis)
            at = nch_in if kind.insert is None else kind.insert
            k = ck.assignment.constants["KH" if kind.axis == "h" else "KW"]
            # insertion index in the output tensor; the source axis index is unchanged
            # in the input, and the stacked dim lands at 1+at.
            y = _unfold(src, ax, 1 + at, k)
        elif isinstance(kind, FullyConnected):
            w = next(fc_iter)
            kin = math.prod(ck.extents[sin][:nch_in])
            xs = src.reshape(nb, kin, -1)
            y = torch.einsum("oi,nis->nos", w.to(src.dtype), xs).reshape((nb, *out_ext))
        elif isinstance(kind, ElementWise):
            fn = kind.fn
            y = {
                "relu": torch.relu,
                "abs": torch.abs,
                "sin": torch.sin,
                "exp": torch.exp,
                "neg": torch.neg,
            }[fn](src)
        elif isinstance(kind, Fold):
            ax = 1 + kind.dim
            y = src.mean(dim=ax) if kind.mode == "avg" else src.amax(dim=ax)  # amax: ties split evenly (A.6)
            if kind.mode == "max" and NearTies.active is not None:
                NearTies.active.note_fold_max(src, ax)
        elif isinstance(kind, Softmax):
            lo, hi = 1 + kind.start, 1 + kind.end
            shp = src.shape
            flat = src.reshape(*shp[:lo], -1, *shp[hi + 1 :])
            y = torch.softmax(flat, dim=lo).reshape(shp)
        elif isinstance(kind, Broadcast):
            y = _broadcast(ck, e, vals[e.inputs[0]], vals[e.inputs[1]])
        else:  # pragma: no cover
            raise TypeError(kind)
        vals[e.out] = y
    return vals[ck.template.output_node]


def bcast_axes(ck: Concrete, e) -> tuple[int, int, int, int]:
    """(core start axis, lhs core ndim, rhs core ndim, rhs ndim) in tensor axes (batch = axis 0)."""
    m = match_broadcast(e.inst.inputs[0], e.inst.inputs[1])
    lhs_node, rhs_node = e.inputs
    if m.region == "spatial":
        base_l = 1 + ck.nch[lhs_node] + m.lhs_span[0]
        base_r = 1 + ck.nch[rhs_node] + m.rhs_span[0]
    elif m.region == "channel":
        base_l = 1 + m.lhs_span[0]
        base_r = 1 + m.rhs_span[0]
    else:
        base_l = base_r = 1 + len(m.common_prefix)
    assert base_l == base_r, "prefix must align"
    return base_l, m.lhs_span[1] - m.lhs_span[0], m.rhs_span[1] - m.rhs_span[0], 1 + len(ck.extents[rhs_node])


def _broadcast(ck: Concrete, e, lhs: torch.Tensor, rhs: torch.Tensor) -> torch.Tensor:
    """out[p, r, s] = lhs[p, r mod L, s] (op) rhs[p, r, s]  — tile order (App. A.8)."""
    base, nl, nr, _ = bcast_axes(ck, e)
    nb = lhs.shape[0]
    pre = rhs.shape[1:base]
    suf = rhs.shape[base + nr :]
    P = math.prod(pre)
    S = math.prod(suf)
    L = math.prod(lhs.shape[base : base + nl])
    R = math.prod(rhs.shape[base : base + nr])
    assert R % L == 0
    l3 = lhs.reshape(nb, P, L, S).repeat(1, 1, R // L, 1)  # tile: index r -> r mod L
    r3 = rhs.reshape(nb, P, R, S)
    op = e.inst.kind.op
    if op == "add":
        o = l3 + r3
    elif op == "sub":
        o = l3 - r3  # lhs - rhs in IR operand order (App. A.8)
    elif op == "mul":
        o = l3 * r3
    elif op == "min":
        o = torch.minimum(l3, r3)  # ties: gradient split 1/2 - 1/2
        if NearTies.active is not None:
            NearTies.active.note(l3, r3)
    elif op == "max":
        o = torch.maximum(l3, r3)
        if NearTies.active is not None:
            NearTies.active.note(l3, r3)
    else:  # pragma: no cover
        raise ValueError(op)
    return o.reshape(rhs.shape)


def init_weights(ck: Concrete, copies: int = 1, seed: int = 2, dtype=torch.float32) -> list[list[torch.Tensor]]:
    """U(-1/sqrt(fan_in), 1/sqrt(fan_in)) per FC, IR edge order, per copy (App. A.10)."""
    g = torch.Generator().manual_seed(seed)
    out = []
    for _ in range(copies):
        ws = []
        for o, k in fc_weight_shapes(ck):
            b = 1.0 / math.sqrt(k)
            ws.append((torch.rand((o, k), generator=g, dtype=torch.float64) * 2 - 1).mul_(b).to(dtype))
        out.append(ws)
    return out


def conv_replacement(ck: Concrete, x: torch.Tensor, weights: list[list[torch.Tensor]], c_in: int, c_out: int, stride: int) -> torch.Tensor:
    """Fig.-2 replication + stride policy (App. A.10).

    stride s: x[..., ::s, ::s] first, then the template at output resolution.
    C_out = r*C_in: r copies on the same input, outputs concatenated on channels.
    C_in = r*C_out: input chunk j -> copy j, outputs summed.
    """
    if stride != 1:
        x = x[:, :, ::stride, ::stride]  # subsample first, template at output resolution (A.10)
    c = min(c_in, c_out)
    r = max(c_in, c_out) // c
    if c_out >= c_in:
        return torch.cat([run_kernel(ck, x, weights[j]) for j in range(r)], dim=1)
    out = None
    for j in range(r):
        yj = run_kernel(ck, x[:, j * c : (j + 1) * c], weights[j])
        out = yj if out is None else out + yj
    return out


class CanvasConvRef(torch.nn.Module):
    """CPU torch module computing a Canvas conv replacement (reference path).

    The concrete graph depends on the input resolution (H, W are constants of
    the assignment), so it is rebuilt lazily per input size; the FC weight
    shapes only depend on channel dims and are fixed at construction.
    """

    def __init__(self, ir_text: str, c_in: int, c_out: int, h: int, w: int, kh: int, kw: int, stride: int = 1, g: int = 4, xs: dict | None = None, seed: int | None = 2):
        super().__init__()
        self.text, self.g, self.kh, self.kw, self.xs = ir_text, g, kh, kw, xs
        self.c_in, self.c_out, self.stride = c_in, c_out, stride
        c = min(c_in, c_out)
        self.r = max(c_in, c_out) // c
        ck = self._concrete(max(h, 8 * stride), max(w, 8 * stride))
        if seed is None:
            ws = []
            for _ in range(self.r):
                cw = []
                for o, k in fc_weight_shapes(ck):
                    b = 1.0 / math.sqrt(k)
                    cw.append(torch.empty(o, k).uniform_(-b, b))
                ws.append(cw)
        else:
            ws = init_weights(ck, copies=self.r, seed=seed)
        self.weights = torch.nn.ParameterList([torch.nn.Parameter(w) for copy in ws for w in copy])
        self.nfc = len(ck.fc_edges)
        self._cks: dict = {}

    def _concrete(self, h: int, w: int) -> Concrete:
        c = min(self.c_in, self.c_out)
        t = cir.parse(self.text).template
        consts = {"C": c, "G": self.g, "H": -(-h // self.stride), "W": -(-w // self.stride), "KH": self.kh, "KW": self.kw}
        a = Assignment(consts, dict(self.xs if self.xs is not None else proportional_values(t, consts)))
        return concretize(t, a)

    def forward(self, x):
        key = tuple(x.shape[2:])
        ck = self._cks.get(key)
        if ck is None:
            ck = self._cks[key] = self._concrete(*key)
        ws = [list(self.weights[j * self.nfc : (j + 1) * self.nfc]) for j in range(self.r)]
        return conv_replacement(ck, x, ws, self.c_in, self.c_out, self.stride)
