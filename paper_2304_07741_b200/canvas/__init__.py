"""Host-side mirror of the reference ``canvas`` search API.

Module names, public names, argument meanings and exception types follow
/root/reference/pkg/src/canvas/ so a user of the reference front end can
switch imports (``from paper_2304_07741_b200.canvas import ir``) and get
bit-identical symbolic results; the reference's own 45 tests run against this
package (tests/test_reference_conformance.py).
"""

from . import ir, micro_dag, primitives, sampler, shape_algebra, shape_solver  # noqa: F401
