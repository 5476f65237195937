"""Level-2 solver and network cost model — the SPEC's examples."""

import pytest
import torchvision

from paper_2304_07741_b200 import zoo
from paper_2304_07741_b200.canvas import ir
from paper_2304_07741_b200.canvas.constraint_solver import BackboneSpec, Budget, Target, base_values, candidate_G, maximize, solve_network
from paper_2304_07741_b200.canvas.cost_model import conv_baseline, kernel_cost, network_cost, original_cost
from paper_2304_07741_b200.canvas.shape_algebra import Assignment
from paper_2304_07741_b200.module import backbone_spec, solve_for_model


def spec_of(*cs):
    return BackboneSpec(tuple(Target(f"t{i}", c, c, 8, 8) for i, c in enumerate(cs)))


def test_candidate_G_examples():
    assert candidate_G(spec_of(32, 48)) == [2, 4, 8, 16]  # PAPER §6.3
    assert candidate_G(spec_of(7, 13)) == []
    assert candidate_G(spec_of(64, 64)) == [2, 4, 8, 16, 32, 64]


def test_base_values_fig6_formula(monkeypatch):
    """lcm_{1,1} = 12, lcm_{i,1} = 20, C_i/C_1 = 5 -> x_{1,1} = 12, x_{i,1} = 60 (PAPER §6.3 / Fig. 6)."""
    import paper_2304_07741_b200.canvas.constraint_solver as cs

    spec = BackboneSpec((Target("t1", 16, 16, 8, 8, 3, 3), Target("ti", 80, 80, 8, 8, 5, 5)))
    tmpl = ir.parse(zoo.INVOLUTION).template
    monkeypatch.setattr(cs, "variable_moduli", lambda t, consts: {v: consts["G"] * consts["KH"] for v in t.free_vars})
    b = base_values(tmpl, spec, 4)
    assert b == {(0, 1): 12, (1, 1): 60}


def test_maximize_fig6_two_doublings():
    base = {(0, 1): 12, (1, 1): 60}
    sol = maximize(None, None, 4, base, Budget(max_flops=300), lambda x: (x[(0, 1)] + x[(1, 1)], 0))
    assert sol.x == {(0, 1): 48, (1, 1): 240} and sol.doublings == 4 and sol.saturated


def test_maximize_discard_below_base():
    assert maximize(None, None, 4, {(0, 1): 12}, Budget(max_flops=5), lambda x: (x[(0, 1)], 0)) is None


def test_maximize_cap_unsaturated():
    sol = maximize(None, None, 4, {(0, 1): 1}, Budget(max_flops=10**30), lambda x: (x[(0, 1)], 0), cap=5)
    assert sol.x[(0, 1)] == 32 and not sol.saturated


def test_conv_baseline_golden():
    assert conv_baseline(Target("c", 64, 64, 56, 56, 3, 3)) == (115_605_504, 36_864)
    assert conv_baseline(Target("u", 1, 1, 1, 1, 3, 3)) == (9, 9)


def test_im2col_network_cost_equals_original():
    """im2col at output resolution has exactly the conv's MACs and params."""
    m = torchvision.models.resnet18()
    spec = backbone_spec(m)
    assert len(spec.targets) == 16
    tmpl = ir.parse(zoo.IM2COL).template
    assert network_cost(spec, tmpl, 4, {}) == original_cost(spec)
    assert sum(t.original_flops for t in spec.targets) == 1_676_279_808


def test_solve_resnet18_involution_budget():
    m = torchvision.models.resnet18()
    sol, spec, xs = solve_for_model(m, zoo.INVOLUTION, flops_frac=0.5)
    assert sol is not None and sol.saturated
    of, _ = original_cost(spec)
    assert sol.achieved_flops <= of * 0.5
    tmpl = ir.parse(zoo.INVOLUTION).template
    # maximality: doubling any variable breaks the budget
    for key in sol.x:
        trial = dict(sol.x)
        trial[key] *= 2
        assert network_cost(spec, tmpl, sol.g, trial)[0] > of * 0.5
    assert set(xs) == {t.name for t in spec.targets}


def test_kernel_cost_rearrangement_only_is_free():
    t = ir.parse("canvas-ir v1\nn0: shape=[C; H, W]\nn1: shape=[C; H, W]\ne: shift(h,+1) (0) -> 1\n").template
    assert kernel_cost(t, Assignment({"C": 8, "G": 4, "H": 5, "W": 5, "KH": 3, "KW": 3})) == (0, 0)


def test_solve_requires_common_G():
    with pytest.raises(ValueError):
        solve_network(ir.parse(zoo.INVOLUTION).template, spec_of(7, 13), Budget(max_flops=1))
