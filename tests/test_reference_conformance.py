"""The reference's own 45 front-end tests, run against this package's mirror.

/root/reference/pkg/tests imports ``canvas.*``; the tests are copied to a
temp dir whose conftest aliases ``canvas`` to ``paper_2304_07741_b200.canvas``.
Skipped where the reference tree is absent (GPU boxes).
"""

import os
import shutil
import subprocess
import sys

import pytest

REF_TESTS = "/root/reference/pkg/tests"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CONFTEST = f'''
import sys
sys.path.insert(0, {ROOT!r})
import paper_2304_07741_b200.canvas as c
from paper_2304_07741_b200.canvas import ir, micro_dag, primitives, shape_algebra, shape_solver
sys.modules["canvas"] = c
for n, m in dict(ir=ir, micro_dag=micro_dag, primitives=primitives, shape_algebra=shape_algebra, shape_solver=shape_solver).items():
    sys.modules["canvas." + n] = m
'''


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference tree not present")
def test_reference_suite_against_mirror(tmp_path):
    for f in os.listdir(REF_TESTS):
        if f.endswith(".py"):
            shutil.copy(os.path.join(REF_TESTS, f), tmp_path / f)
    (tmp_path / "conftest.py").write_text(CONFTEST)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", str(tmp_path)], capture_output=True, text=True, cwd=tmp_path)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "45 passed" in r.stdout, r.stdout[-500:]


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference tree not present")
def test_sampler_mirror_matches_reference_sampler():
    """Beyond the golden sweeps: mirror vs the reference sampler itself over a
    grid of node budgets, seeds, type weights, width caps and prune rules."""
    code = f'''
import sys
sys.path.insert(0, {ROOT!r})
from paper_2304_07741_b200.canvas import ir as mir
from paper_2304_07741_b200.canvas.sampler import Sampler as MS, SamplerConfig as MC
sys.path.insert(0, "/root/reference/pkg/src")
from canvas import ir as rir
from canvas.sampler import Sampler as RS, SamplerConfig as RC
from canvas.micro_dag import DEFAULT_PRUNE_RULES
bad = []
for nodes in (3, 6, 9, 13):
    for seed in (0, 5):
        for tw in ({{}}, {{"bcast": 3.0, "fc": 0.5}}, {{"unfold": 0.0}}):
            for mw, rules in ((3, DEFAULT_PRUNE_RULES), (4, DEFAULT_PRUNE_RULES), (3, frozenset()), (3, frozenset({{"self-subtraction"}}))):
                a = "".join(rir.emit(k) for k in RS(RC(nodes=nodes, seed=seed, type_weights=tw, max_width=mw, prune_rules=rules)).sample_many(4))
                b = "".join(mir.emit(k) for k in MS(MC(nodes=nodes, seed=seed, type_weights=tw, max_width=mw, prune_rules=rules)).sample_many(4))
                if a != b:
                    bad.append((nodes, seed, tw, mw, sorted(rules)))
print("BAD", bad)
'''
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "BAD []" in r.stdout, r.stdout[-2000:]
