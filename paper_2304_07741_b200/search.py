"""The paper-level entry point ``canvas.sample(nn, budget)``.

Draws kernels with the sampler mirror (canvas/sampler.py, bit-identical to
the reference sampler), solves each one over the network's replacement
targets under a FLOPs / parameter budget with the level-2 solver
(canvas/constraint_solver.py), and returns the kernels that
fit, best analytical speed-up first.  ``apply`` then swaps the network's
standard convs for the chosen kernel (module.replace) so it trains on the
B200 executor.  Accuracy-driven selection (training each candidate, the
harness of SPEC.md:535-596) is the caller's loop over the returned list,
e.g. with evaluator.CandidateEvaluator for latency.
"""

from __future__ import annotations

from dataclasses import dataclass

from torch import nn

from .canvas import ir
from .canvas.constraint_solver import Solution
from .canvas.cost_model import ideal_speedup
from .canvas.sampler import DedupStore, Sampler, SamplerConfig
from .module import replace, solve_for_model


@dataclass
class Candidate:
    ir_text: str
    solution: Solution
    xs_by_name: dict
    ideal_speedup: float


def sample(model: nn.Module, *, flops_frac: float | None = None, params_frac: float | None = None, count: int = 8, nodes: int = 10, seed: int | None = None, g: int | None = None, input_shape=(1, 3, 224, 224), max_draws: int | None = None, store: DedupStore | None = None) -> list[Candidate]:
    """Up to ``count`` sampled kernels that fit the budget on ``model``."""
    smp = Sampler(SamplerConfig(nodes=nodes, seed=seed), store)
    out: list[Candidate] = []
    draws = 0
    limit = max_draws if max_draws is not None else 16 * count
    while len(out) < count and draws < limit:
        draws += 1
        text = ir.emit(smp.sample_kernel())
        try:
            sol, spec, xs_by_name = solve_for_model(model, text, flops_frac=flops_frac, params_frac=params_frac, g=g, input_shape=input_shape)
        except ValueError:  # NonIntegral / NotReplaceable: no legal sizes for this kernel here
            continue
        if sol is None:
            continue
        out.append(Candidate(text, sol, xs_by_name, ideal_speedup(spec, ir.parse(text).template, sol.g, sol.x)))
    return sorted(out, key=lambda c: -c.ideal_speedup)


def apply(model: nn.Module, cand: Candidate) -> list[str]:
    """Replace the model's targets with ``cand`` (its solved G and free variables)."""
    return replace(model, cand.ir_text, g=cand.solution.g, xs_by_name=cand.xs_by_name)
