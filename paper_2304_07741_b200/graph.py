"""Concrete kernel graph: a solved Canvas kernel with every extent an int.

Input is the reference boundary payload — a ``KernelTemplate`` (ref
micro_dag.py:224-230, produced by ``ir.parse``, ref ir.py:97-169) plus an
``Assignment`` (ref shape_algebra.py:381-404, from ``TargetSolution.assignment``,
ref ir.py:48-53).  Output is a list of :class:`CNode` whose extents, spans and
replication ratios are plain integers: the only thing the lowering and the
device kernels ever look at.

Layout: a node with shape ``[d0..dk-1; spatials]`` is the
row-major tensor ``[N, d0, .., dk-1, spatials..]``; spatial dims are H and/or W
in that order (ref primitives.py:111-116).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

from .canvas.primitives import (
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
from .canvas.shape_algebra import D_H, D_W, Assignment, evaluate
from .canvas.shape_solver import match_broadcast

#: primitive classes that are pure index maps (never materialised, App. A.1-A.3)
VIEW_OPS = ("group", "shift", "unfold")


class LoweringError(ValueError):
    """The kernel cannot be lowered under this assignment."""


@dataclass
class CNode:
    id: int
    ext: tuple  # channel extents ++ spatial extents
    nch: int
    sp: tuple  # spatial axis names in order, subset of ("h", "w")
    op: str  # "input" | group | shift | unfold | fc | ew | fold | softmax | bcast
    ins: tuple = ()
    attr: dict = field(default_factory=dict)
    consumers: list = field(default_factory=list)  # [(consumer node id, input position)]

    @property
    def numel(self) -> int:
        return math.prod(self.ext)

    @property
    def ch_ext(self) -> tuple:
        return self.ext[: self.nch]

    @property
    def sp_ext(self) -> tuple:
        return self.ext[self.nch :]


@dataclass
class ConcreteGraph:
    nodes: list
    output: int
    fc_nodes: list  # node ids of FC outputs, in IR edge order (= weight order, App. A.10)
    consts: dict

    def fc_shape(self, v: int) -> tuple[int, int]:
        """(out, K) of the FC producing node ``v``: nn.Linear weight layout [out, prod(in ch)] (App. A.4)."""
        nd = self.nodes[v]
        src = self.nodes[nd.ins[0]]
        return nd.attr["O"], math.prod(src.ch_ext)

    def fc_macs_per_image(self) -> int:
        """Σ_FC out*K*spatial — ref primitives.cost FLOPs for FC edges (primitives.py:260-264)."""
        tot = 0
        for v in self.fc_nodes:
            o, k = self.fc_shape(v)
            tot += o * k * math.prod(self.nodes[v].sp_ext)
        return tot


def _sp_names(shape) -> tuple:
    out = []
    for d in shape.spatials:
        if d == D_H:
            out.append("h")
        elif d == D_W:
            out.append("w")
        else:  # pragma: no cover - the reference never builds other spatial dims
            raise LoweringError(f"unknown spatial dim {d}")
    return tuple(out)


def build_graph(template, assignment: Assignment) -> ConcreteGraph:
    """Evaluate every node/edge of ``template`` under ``assignment``."""
    dag = template.dag
    nodes: list[CNode] = []
    for i, s in enumerate(dag.nodes):
        try:
            ext = tuple(evaluate(d, assignment) for d in s.dims())
        except ValueError as err:
            raise LoweringError(f"node {i} {s}: {err}") from err
        nodes.append(CNode(i, ext, len(s.channels), _sp_names(s), "input" if i == 0 else "?"))
    k_of = {"h": assignment.constants["KH"], "w": assignment.constants["KW"]}
    fcs = []
    for e in dag.edges:
        kind = e.inst.kind
        nd = nodes[e.out]
        nd.ins = tuple(e.inputs)
        src = nodes[e.inputs[0]]
        if isinstance(kind, Group):
            nd.op = "group"
            a, b = nd.ext[kind.dim], nd.ext[kind.dim + 1]
            if a * b != src.ext[kind.dim]:
                raise LoweringError(f"group on node {e.out}: {a}*{b} != {src.ext[kind.dim]}")
            nd.attr = {"dim": kind.dim, "B": b}
        elif isinstance(kind, Shift):
            nd.op = "shift"
            nd.attr = {"ax": src.nch + spatial_position(e.inst.inputs[0], kind.axis), "off": kind.offset}
        elif isinstance(kind, Unfold):
            nd.op = "unfold"
            at = src.nch if kind.insert is None else kind.insert
            k = k_of[kind.axis]
            # spatial axis index in the *output* tensor (one more channel dim than the input)
            ax_in = src.nch + spatial_position(e.inst.inputs[0], kind.axis)
            nd.attr = {"at": at, "K": k, "ax_in": ax_in, "ax_out": ax_in + 1}
            if nd.ext[at] != k:
                raise LoweringError(f"unfold on node {e.out}: K extent {nd.ext[at]} != {k}")
        elif isinstance(kind, FullyConnected):
            nd.op = "fc"
            nd.attr = {"O": nd.ext[0], "K": math.prod(src.ch_ext), "fc_index": len(fcs)}
            fcs.append(e.out)
        elif isinstance(kind, ElementWise):
            nd.op = "ew"
            nd.attr = {"fn": kind.fn}
        elif isinstance(kind, Fold):
            nd.op = "fold"
            nd.attr = {"dim": kind.dim, "mode": kind.mode, "D": src.ext[kind.dim]}
        elif isinstance(kind, Softmax):
            nd.op = "softmax"
            nd.attr = {"start": kind.start, "end": kind.end}
        elif isinstance(kind, Broadcast):
            nd.op = "bcast"
            nd.attr = _bcast_attr(e, nodes)
        else:  # pragma: no cover
            raise LoweringError(f"unknown primitive {kind!r}")
        for pos, i in enumerate(e.inputs):
            nodes[i].consumers.append((e.out, pos))
    return ConcreteGraph(nodes, template.output_node, fcs, dict(assignment.constants))


def _bcast_attr(e, nodes) -> dict:
    """Concrete broadcast spans: out[p, r, s] = lhs[p, r mod L, s] (op) rhs[p, r, s] (App. A.8).

    ``cs`` is the first core axis (same in lhs and rhs, the prefix being
    structurally equal — ref shape_solver.py:76-87); ``nl``/``nr`` the core
    ranks; ``L``/``R`` the core sizes, ``R % L == 0``.
    """
    m = match_broadcast(e.inst.inputs[0], e.inst.inputs[1])
    if m is None or m.ratio is None:
        raise LoweringError(f"broadcast into node {e.out} has no solved matching")
    lhs, rhs = nodes[e.inputs[0]], nodes[e.inputs[1]]
    if m.region == "channel":
        cs = m.rhs_span[0]
        cs_l = m.lhs_span[0]
    elif m.region == "spatial":
        cs = rhs.nch + m.rhs_span[0]
        cs_l = lhs.nch + m.lhs_span[0]
    else:
        cs = cs_l = len(m.common_prefix)
    if cs != cs_l:
        raise LoweringError(f"broadcast into node {e.out}: prefix misaligned")
    nl = m.lhs_span[1] - m.lhs_span[0]
    nr = m.rhs_span[1] - m.rhs_span[0]
    lcore = lhs.ext[cs : cs + nl]
    rcore = rhs.ext[cs : cs + nr]
    L, R = math.prod(lcore), math.prod(rcore)
    if R % L or lhs.ext[:cs] != rhs.ext[:cs] or lhs.ext[cs + nl :] != rhs.ext[cs + nr :]:
        raise LoweringError(f"broadcast into node {e.out}: {lhs.ext} onto {rhs.ext} not integral")
    return {"op": e.inst.kind.op, "cs": cs, "nl": nl, "nr": nr, "L": L, "R": R, "M": R // L, "lcore": lcore, "rcore": rcore}
