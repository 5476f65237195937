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


# ---------------------------------------------------------------------------
# Network-level solve (§6.3): global G, base values by
# the lcm / channel-ratio rule, then budget maximisation by Δ-ordered doubling.
# ---------------------------------------------------------------------------
from dataclasses import dataclass, field  # noqa: E402


class NotReplaceable(ValueError):
    """Target with neither C_in | C_out nor C_out | C_in."""


@dataclass(frozen=True)
class Target:
    name: str
    c_in: int
    c_out: int
    h: int  # output resolution of the replaced conv
    w: int
    kh: int = 3
    kw: int = 3
    original_flops: int = 0
    original_params: int = 0

    @property
    def replaceable(self) -> bool:
        return max(self.c_in, self.c_out) % min(self.c_in, self.c_out) == 0

    @property
    def c(self) -> int:
        return min(self.c_in, self.c_out)

    @property
    def copies(self) -> int:
        return max(self.c_in, self.c_out) // self.c


@dataclass(frozen=True)
class BackboneSpec:
    targets: tuple
    non_replaced_flops: int = 0
    non_replaced_params: int = 0


@dataclass(frozen=True)
class Budget:
    max_flops: int | None = None
    max_params: int | None = None

    def admits(self, cost: tuple[int, int]) -> bool:
        f, p = cost
        return (self.max_flops is None or f <= self.max_flops) and (self.max_params is None or p <= self.max_params)


@dataclass
class Solution:
    g: int
    x: dict  # (target index, var id) -> int
    achieved_flops: int = 0
    achieved_params: int = 0
    saturated: bool = True  # False when the doubling cap stopped the search
    doublings: int = 0
    notes: list = field(default_factory=list)

    def target_xs(self, i: int) -> dict:
        return {v: x for (t, v), x in self.x.items() if t == i}


def candidate_G(spec: BackboneSpec) -> list[int]:
    """Factors (> 1) of gcd of the replaceable targets' channel numbers C_i."""
    cs = [t.c for t in spec.targets if t.replaceable]
    if not cs:
        return []
    g = 0
    for c in cs:
        g = math.gcd(g, c)
    return [f for f in range(2, g + 1) if g % f == 0]


def _consts(t: Target, g: int) -> dict:
    return {"C": t.c, "G": g, "H": t.h, "W": t.w, "KH": t.kh, "KW": t.kw}


def base_values(tmpl: KernelTemplate, spec: BackboneSpec, g: int) -> dict:
    """x_{i,j} = k_{i,j} lcm_{i,j} with target 1 = argmin C_i, k_{1,j} = 1 and
    k_{i,j} = ceil(C_i lcm_{1,j} / (C_1 lcm_{i,j})) (§6.3)."""
    idx = [i for i, t in enumerate(spec.targets) if t.replaceable]
    mods = {i: variable_moduli(tmpl, _consts(spec.targets[i], g)) for i in idx}
    first = min(idx, key=lambda i: (spec.targets[i].c, i))
    c1 = spec.targets[first].c
    out = {}
    for i in idx:
        ci = spec.targets[i].c
        for v in tmpl.free_vars:
            l1, li = mods[first][v], mods[i][v]
            k = -(-(ci * l1) // (c1 * li))
            out[(i, v)] = max(1, k) * li
    return out


def maximize(tmpl: KernelTemplate, spec: BackboneSpec, g: int, base: dict, budget: Budget, cost_fn, cap: int = 32) -> Solution | None:
    """Δ-ordered doubling.  ``cost_fn(x) -> (flops, params)`` of
    the whole network.  Returns None (Discard) when the base already exceeds the
    budget.  Each iteration recomputes Δ_{i,j} = cost(2x_{i,j}) - cost(x) (FLOPs,
    then params), visits variables in ascending (Δ, i, j) order and doubles each
    one whose doubled configuration stays within every bound."""
    x = dict(base)
    cur = cost_fn(x)
    if not budget.admits(cur):
        return None
    doublings = 0
    saturated = True
    for _ in range(cap):
        deltas = []
        for key in sorted(x):
            trial = dict(x)
            trial[key] *= 2
            c = cost_fn(trial)
            deltas.append(((c[0] - cur[0], c[1] - cur[1]), key))
        changed = False
        for _, key in sorted(deltas):
            trial = dict(x)
            trial[key] *= 2
            c = cost_fn(trial)
            if budget.admits(c):
                x, cur, changed = trial, c, True
                doublings += 1
        if not changed:
            break
    else:
        saturated = False
    return Solution(g, x, cur[0], cur[1], saturated, doublings)


def solve_network(tmpl: KernelTemplate, spec: BackboneSpec, budget: Budget, g: int | None = None, cap: int = 32) -> Solution | None:
    """candidate_G -> base_values -> maximize with the network cost model (cost_model.network_cost)."""
    from .cost_model import network_cost

    gs = [g] if g is not None else candidate_G(spec)
    if not gs:
        raise NotReplaceable("no global G divides every replaceable target's channels")
    gg = 4 if g is None and 4 in gs else gs[0]
    base = base_values(tmpl, spec, gg)
    return maximize(tmpl, spec, gg, base, budget, lambda xx: network_cost(spec, tmpl, gg, xx), cap)
