"""B200-native executor for Canvas (arXiv 2304.07741) kernel graphs.

Layers:
  canvas/     host-side mirror of the reference search API (shape algebra,
              primitives, level-1 solver, micro-DAG, canvas-ir v1)
  lowering    concrete kernel graph -> tensor-expression graph (+ its adjoint)
  codegen     fusion planning + CUDA C++ for sm_100a from hand-written templates
  runtime     ctypes binding of the C-ABI library libcanvas_b200.so
  module      CanvasKernel nn.Module / autograd Function, conv replacement
"""

__version__ = "0.1.0"
