"""The CPU oracle (test infrastructure) pinned by derived goldens.

The reference pins no numeric value of any primitive, so the
oracle is pinned by: im2col template == F.conv2d, two
independent restatements agreeing (torch fp64 vs numpy-fp64 index loops),
Involution semantics, linearity / zero-input invariants
 and fp64 gradcheck.
"""

import numpy as np
import pytest
import torch

from oracle import np_interp, torch_ref as R
from paper_2304_07741_b200 import zoo
from paper_2304_07741_b200.executor import solve_target


def concrete(text, c=8, h=6, w=5, g=4):
    t, a = solve_target(text, c_in=c, c_out=c, h=h, w=w, g=g)
    return R.concretize(t, a)


def sweep(path="tests/golden/sampler_10_7_20.cir"):
    return ["canvas-ir v1\n" + t for t in open(path).read().split("canvas-ir v1\n")[1:]]


def test_im2col_equals_conv2d():
    ck = concrete(zoo.IM2COL, c=16, h=9, w=7)
    x = torch.randn(2, 16, 9, 7, dtype=torch.float64)
    w = torch.randn(16, 16 * 9, dtype=torch.float64)
    y = R.run_kernel(ck, x, [w])
    ref = torch.nn.functional.conv2d(x, w.view(16, 16, 3, 3), padding=1)
    assert torch.equal(y, ref) or (y - ref).abs().max() < 1e-12


@pytest.mark.parametrize("text", list(zoo.ALL.values()) + sweep())
def test_two_restatements_agree(text):
    ck = concrete(text)
    g = torch.Generator().manual_seed(0)
    x = torch.randn(2, *ck.extents[0], generator=g, dtype=torch.float64)
    ws = R.init_weights(ck, seed=2, dtype=torch.float64)[0]
    a = R.run_kernel(ck, x, ws).numpy()
    b, macs = np_interp.execute(ck, x.numpy(), [w.numpy() for w in ws])
    assert a.shape == b.shape
    assert np.allclose(a, b, rtol=1e-12, atol=1e-12, equal_nan=True)
    assert macs == 2 * sum(o * k * int(np.prod(ck.extents[v][ck.nch[v]:])) for v, (o, k) in zip([ck.dag.edges[i].out for i in ck.fc_edges], R.fc_weight_shapes(ck)))


def test_involution_semantics():
    """y = x + avg_{kh,kw} ( W2 W1 x )[g, kh*KW+kw] * x_unf[g, c, kh, kw]."""
    c, h, w, g = 8, 5, 6, 4
    ck = concrete(zoo.INVOLUTION, c=c, h=h, w=w, g=g)
    x = torch.randn(1, c, h, w, dtype=torch.float64)
    ws = R.init_weights(ck, seed=3, dtype=torch.float64)[0]
    y = R.run_kernel(ck, x, ws)
    k = torch.einsum("oi,nihw->nohw", ws[1], torch.einsum("oi,nihw->nohw", ws[0], x)).view(1, g, 9, h, w)
    xu = torch.nn.functional.unfold(x, 3, padding=1).view(1, g, c // g, 9, h, w)
    ref = x + (k.unsqueeze(2) * xu).mean(dim=3).reshape(1, c, h, w)
    assert (y - ref).abs().max() < 1e-12


@pytest.mark.parametrize("text", [zoo.IM2COL, zoo.INVOLUTION])
def test_linearity_and_zero(text):
    ck = concrete(text)
    ws = R.init_weights(ck, seed=2, dtype=torch.float64)[0]
    x1 = torch.randn(1, *ck.extents[0], dtype=torch.float64)
    x2 = torch.randn(1, *ck.extents[0], dtype=torch.float64)
    z = R.run_kernel(ck, torch.zeros_like(x1), ws)
    assert z.abs().max() == 0
    if text == zoo.IM2COL:
        lhs = R.run_kernel(ck, 2 * x1 + 3 * x2, ws)
        rhs = 2 * R.run_kernel(ck, x1, ws) + 3 * R.run_kernel(ck, x2, ws)
        assert (lhs - rhs).abs().max() < 1e-10


@pytest.mark.parametrize("name", ["seed7_k1", "involution", "im2col", "seed7_k0"])
def test_gradcheck(name):
    ck = concrete(zoo.ALL[name], c=4, h=3, w=4, g=2)
    x = torch.randn(1, *ck.extents[0], dtype=torch.float64, requires_grad=True)
    ws = [w.requires_grad_(True) for w in R.init_weights(ck, seed=2, dtype=torch.float64)[0]]
    # max/min kinks: perturbation stays away from ties with random inputs
    assert torch.autograd.gradcheck(lambda x_, *w_: R.run_kernel(ck, x_, list(w_)), (x, *ws), eps=1e-6, atol=1e-5)
