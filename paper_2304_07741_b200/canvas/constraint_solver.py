"""Level-2 (analytical) variable solving — the integrality part.

SPEC.md:372-447 / PAPER.md §6.3: after the level-1 matcher every remaining
dynamic variable ``x`` appears only in numerators, as ``x * p / q`` (node
dims) or inside a broadcast ratio ``M = x * p / q``.  Under a concrete target
assignment each such expression is an integer iff ``x`` is a multiple of
``q / gcd(p, q)``; the lcm of those moduli is the variable's base value
("x_{i,j} = k_{i,j} * lcm(q1, q2, ...)", §6.3).

This module provides exactly that integrality step plus the proportional
choice the executor uses when no budget is given: the smallest multiple of
the modulus that is >= C (so ``x`` tracks the channel count, the SPEC's
base_values rule with target 1 = the target itself).  Budget maximisation
(Δ-ordered doubling) is out of the hot path.
"""

from __future__ import annotations

import math

from .micro_dag import KernelTemplate
from .primitives import Broadcast
from .shape_algebra import Assignment, Dimension, NonIntegral
from .shape_solver import match_broadcast

_VAR = 0


def _split(d: Dimension, consts: dict) -> tuple[int | None, int, int]:
    """(var id or None, numeric numerator without the var, numeric denominator)."""
    a = Assignment(consts)
    var = None
    num = 1
    for atom in d.num:
        if atom[0] == _VAR:
            var = atom[1]
        else:
            num *= a.atom_value(*atom)
    den = math.prod(a.atom_value(*atom) for atom in d.den)
    return var, num, den


def variable_moduli(t: KernelTemplate, consts: dict) -> dict[int, int]:
    """For every free variable the modulus its value must be a multiple of."""
    mod = {v: 1 for v in t.free_vars}

    def need(d: Dimension) -> None:
        var, p, q = _split(d, consts)
        if var is None:
            if p % q:
                raise NonIntegral(f"{d} is not integral under {consts}")
            return
        mod[var] = math.lcm(mod[var], q // math.gcd(p, q))

    for s in t.dag.nodes:
        for d in s.dims():
            need(d)
    for e in t.dag.edges:
        if isinstance(e.inst.kind, Broadcast):
            m = match_broadcast(e.inst.inputs[0], e.inst.inputs[1])
            if m.ratio is None:
                raise NonIntegral("broadcast still needs a level-1 substitution")
            need(m.ratio)
    return mod


def base_values(t: KernelTemplate, consts: dict) -> dict[int, int]:
    """Smallest legal value of every free variable."""
    return variable_moduli(t, consts)


def proportional_values(t: KernelTemplate, consts: dict, scale: int | None = None) -> dict[int, int]:
    """Smallest legal value >= ``scale`` (default C) for every free variable."""
    target = consts["C"] if scale is None else scale
    return {v: q * max(1, -(-target // q)) for v, q in variable_moduli(t, consts).items()}
