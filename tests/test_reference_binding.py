"""The reference package itself on the boundary.

The drop-in boundary is the reference's own payload: ``canvas-ir v1`` text with
a ``solve:`` record (ref ir.py:68-89, TargetSolution ir.py:35-53).  The
reference sampler produces kernels and the reference ``ir.emit`` writes them
with a solve record for a ResNet-18 layer1 target; this package then parses
that text (mirror ``ir.parse``), takes the reference's TargetSolution
constants, lowers it and builds the plan blob — which must be byte-identical to
the blob built from the mirror's own sampler output for the same seed.  The
reference runs in a subprocess (its package is ``canvas``; nothing here imports
it).  Skipped where /root/reference is absent (GPU boxes)."""

import json
import os
import subprocess
import sys

import pytest

from paper_2304_07741_b200.canvas import ir as mir
from paper_2304_07741_b200.canvas.sampler import Sampler, SamplerConfig
from paper_2304_07741_b200.graph import build_graph
from paper_2304_07741_b200.lowering import lower

REF_SRC = "/root/reference/pkg/src"

EMIT = r'''
import json, sys
sys.path.insert(0, sys.argv[1])
from canvas import ir
from canvas.sampler import Sampler, SamplerConfig
out = []
for k in Sampler(SamplerConfig(nodes=10, seed=7)).sample_many(24):
    tg = ir.TargetSolution("layer1.0.conv1", 64, 64, 56, 56, 3, 3, {v: 64 for v in k.free_vars})
    out.append(ir.emit(k, ir.SolveRecord(4, (tg,))))
print(json.dumps(out))
'''


def _blob(text: str) -> bytes:
    parsed = mir.parse(text)
    tg = parsed.solve.targets[0]
    g = build_graph(parsed.template, tg.assignment(parsed.solve.g))
    return lower(g, c_in=tg.c_in, c_out=tg.c_out, stride=1, h_in=tg.h, w_in=tg.w).blob()


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference tree not present")
def test_reference_emitted_ir_lowers_to_identical_blobs():
    r = subprocess.run([sys.executable, "-c", EMIT, REF_SRC], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    ref_texts = json.loads(r.stdout)
    mine = Sampler(SamplerConfig(nodes=10, seed=7)).sample_many(24)
    assert len(ref_texts) == len(mine) == 24
    for i, (rt, k) in enumerate(zip(ref_texts, mine)):
        tg = mir.TargetSolution("layer1.0.conv1", 64, 64, 56, 56, 3, 3, {v: 64 for v in k.free_vars})
        mt = mir.emit(k, mir.SolveRecord(4, (tg,)))
        assert rt == mt, f"kernel {i}: reference and mirror IR text differ"
        assert _blob(rt) == _blob(mt), f"kernel {i}: plan blobs differ"
        parsed = mir.parse(rt)
        assert parsed.solve.targets[0].assignment(4).constants["C"] == 64
