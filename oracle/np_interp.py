"""Independent numpy-fp64 forward interpreter (TEST INFRASTRUCTURE).

A second restatement of SPEC.md:491-533 ``interpreter.execute`` written with
explicit index formulas (gathers over integer index arrays + validity masks)
instead of torch ops, so that torch_ref.py and this file do not share a
common-mode bug.  Also counts MACs the way SPEC.md:510 prescribes (FC only).
"""

from __future__ import annotations

import math

import numpy as np

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
from paper_2304_07741_b200.canvas.shape_solver import match_broadcast


def _gather_shift(x: np.ndarray, axis: int, off: int) -> np.ndarray:
    n = x.shape[axis]
    src = np.arange(n) + off
    ok = (src >= 0) & (src < n)
    out = np.take(x, np.clip(src, 0, n - 1), axis=axis)
    mask_shape = [1] * x.ndim
    mask_shape[axis] = n
    return out * ok.reshape(mask_shape)


def execute(ck, x: np.ndarray, weights: list[np.ndarray]) -> tuple[np.ndarray, int]:
    """Forward of one kernel copy in fp64; returns (output, MAC count)."""
    vals = {0: np.asarray(x, dtype=np.float64)}
    nb = x.shape[0]
    macs = 0
    wi = 0
    for e in ck.dag.edges:
        kind = e.inst.kind
        s = e.inputs[0]
        a = vals[s]
        nch = ck.nch[s]
        if isinstance(kind, Group):
            y = a.reshape((nb, *ck.extents[e.out]))
        elif isinstance(kind, Shift):
            y = _gather_shift(a, 1 + nch + spatial_position(e.inst.inputs[0], kind.axis), kind.offset)
        elif isinstance(kind, Unfold):
            ax = 1 + nch + spatial_position(e.inst.inputs[0], kind.axis)
            k = ck.assignment.constants["KH" if kind.axis == "h" else "KW"]
            at = nch if kind.insert is None else kind.insert
            planes = [_gather_shift(a, ax, kk - k // 2) for kk in range(k)]
            y = np.stack(planes, axis=1 + at)
        elif isinstance(kind, FullyConnected):
            w = np.asarray(weights[wi], dtype=np.float64)
            wi += 1
            kin = math.prod(ck.extents[s][:nch])
            xs = a.reshape(nb, kin, -1)
            y = np.einsum("oi,nis->nos", w, xs).reshape((nb, *ck.extents[e.out]))
            macs += w.shape[0] * kin * xs.shape[2] * nb
        elif isinstance(kind, ElementWise):
            y = {"relu": lambda v: np.maximum(v, 0.0), "abs": np.abs, "sin": np.sin, "exp": np.exp, "neg": np.negative}[kind.fn](a)
        elif isinstance(kind, Fold):
            y = a.mean(axis=1 + kind.dim) if kind.mode == "avg" else a.max(axis=1 + kind.dim)
        elif isinstance(kind, Softmax):
            lo, hi = 1 + kind.start, 1 + kind.end
            shp = a.shape
            f = a.reshape(*shp[:lo], -1, *shp[hi + 1 :])
            m = f.max(axis=lo, keepdims=True)
            ex = np.exp(f - m)
            y = (ex / ex.sum(axis=lo, keepdims=True)).reshape(shp)
        elif isinstance(kind, Broadcast):
            lhs, rhs = vals[e.inputs[0]], vals[e.inputs[1]]
            m = match_broadcast(e.inst.inputs[0], e.inst.inputs[1])
            r_node = e.inputs[1]
            if m.region == "channel":
                base = 1 + m.rhs_span[0]
            elif m.region == "spatial":
                base = 1 + ck.nch[r_node] + m.rhs_span[0]
            else:
                base = 1 + len(m.common_prefix)
            nr = m.rhs_span[1] - m.rhs_span[0]
            nl = m.lhs_span[1] - m.lhs_span[0]
            P = math.prod(rhs.shape[1:base])
            R = math.prod(rhs.shape[base : base + nr])
            S = math.prod(rhs.shape[base + nr :])
            L = math.prod(lhs.shape[base : base + nl])
            li = np.arange(R) % L  # lhs core index for every rhs core index
            lv = lhs.reshape(nb, P, L, S)[:, :, li, :]
            rv = rhs.reshape(nb, P, R, S)
            op = {"add": np.add, "sub": np.subtract, "mul": np.multiply, "min": np.minimum, "max": np.maximum}[kind.op]
            y = op(lv, rv).reshape(rhs.shape)
        else:  # pragma: no cover
            raise TypeError(kind)
        vals[e.out] = y
    return vals[ck.template.output_node], macs
