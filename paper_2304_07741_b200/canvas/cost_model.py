"""Analytical FLOPs / parameter accounting.

MAC = 1 FLOP for FC; 1 per output element for ew/fold/bcast, 3 for softmax, 0
for rearrangements — the per-primitive ``cost`` (ref primitives.py:253-268)
summed over a kernel and multiplied by the Fig.-2 replication factor r
(SPEC.md:480).  ``conv_baseline`` is the K_H x K_W convolution being replaced.
"""

from __future__ import annotations

from .constraint_solver import BackboneSpec, NotReplaceable, Target, _consts
from .micro_dag import KernelTemplate
from .primitives import cost
from .shape_algebra import Assignment


def kernel_cost(tmpl: KernelTemplate, a: Assignment, copies: int = 1) -> tuple[int, int]:
    """(flops, params) of one replacement: Σ_edges cost x r."""
    f = p = 0
    for e in tmpl.dag.edges:
        ef, ep = cost(e.inst, a)
        f += ef
        p += ep
    return f * copies, p * copies


def target_cost(tmpl: KernelTemplate, t: Target, g: int, xs: dict) -> tuple[int, int]:
    if not t.replaceable:
        raise NotReplaceable(f"{t.name}: {t.c_in} -> {t.c_out}")
    return kernel_cost(tmpl, Assignment(_consts(t, g), dict(xs)), t.copies)


def network_cost(spec: BackboneSpec, tmpl: KernelTemplate, g: int, x: dict) -> tuple[int, int]:
    """Σ target kernel costs + non-replaced totals."""
    f, p = spec.non_replaced_flops, spec.non_replaced_params
    for i, t in enumerate(spec.targets):
        if t.replaceable:
            tf, tp = target_cost(tmpl, t, g, {v: xv for (ti, v), xv in x.items() if ti == i})
        else:
            tf, tp = t.original_flops, t.original_params
        f += tf
        p += tp
    return f, p


def conv_baseline(t: Target) -> tuple[int, int]:
    """params = C_in C_out K_H K_W, flops = params H W (MAC = 1 FLOP)."""
    params = t.c_in * t.c_out * t.kh * t.kw
    return params * t.h * t.w, params


def original_cost(spec: BackboneSpec) -> tuple[int, int]:
    f, p = spec.non_replaced_flops, spec.non_replaced_params
    for t in spec.targets:
        bf, bp = conv_baseline(t)
        f += bf
        p += bp
    return f, p


def ideal_speedup(spec: BackboneSpec, tmpl: KernelTemplate, g: int, x: dict) -> float:
    """1 / (1 - replaceable_frac (1 - kernel_frac)) on FLOPs (§8.2)."""
    of, _ = original_cost(spec)
    rep = sum(conv_baseline(t)[0] for t in spec.targets if t.replaceable)
    kf = sum(target_cost(tmpl, t, g, {v: xv for (ti, v), xv in x.items() if ti == i})[0] for i, t in enumerate(spec.targets) if t.replaceable)
    frac = rep / of if of else 0.0
    kfrac = kf / rep if rep else 1.0
    return 1.0 / (1.0 - frac * (1.0 - kfrac)) if frac * (1.0 - kfrac) < 1.0 else float("inf")
