"""Pinned Canvas kernels (canvas-ir v1 text) used by bench.py, smoke() and tests.

These are *data*: IR texts emitted by the reference sampler / front end
(SURVEY App. B), so bench and the GPU box never need /root/reference:

* ``SEED7_K1`` — first+1 kernel of ``Sampler(SamplerConfig(nodes=10, seed=7))``:
  ends in a dense Unfold+FC (K = 9C), the tensor-core case.  Primary bench kernel.
* ``SEED7_K0`` — kernel #0 of the same sampler: memory-bound, no FC.
* ``IM2COL`` — ``unfold(h); unfold(w); fc(C)`` == ``F.conv2d(padding=1)``.
* ``INVOLUTION`` — PAPER.md:245-249 built through the reference API (free var x1).
* ``NEG`` — ``Sampler(nodes=2, seed=7)``: the trivial ``ew(neg)`` smoke kernel.
"""

IM2COL = """\
canvas-ir v1
n0: shape=[C; H, W]
n1: shape=[C, KH; H, W]
n2: shape=[C, KH, KW; H, W]
n3: shape=[C; H, W]
e: unfold(h) (0) -> 1
e: unfold(w) (1) -> 2
e: fc(C) (2) -> 3
"""

INVOLUTION = """\
canvas-ir v1
n0: shape=[C; H, W]
n1: shape=[x1; H, W]
n2: shape=[G*KH*KW; H, W]
n3: shape=[G, KH*KW; H, W]
n4: shape=[G, C/G; H, W]
n5: shape=[G, C/G, KH; H, W]
n6: shape=[G, C/G, KH, KW; H, W]
n7: shape=[G, C/G, KH, KW; H, W]
n8: shape=[G, C/G, KH; H, W]
n9: shape=[G, C/G; H, W]
n10: shape=[C; H, W]
e: fc(x1) (0) -> 1
e: fc(G*KH*KW) (1) -> 2
e: group(G) (2) -> 3
e: group(G) (0) -> 4
e: unfold(h) (4) -> 5
e: unfold(w) (5) -> 6
e: bcast(mul) (3,6) -> 7
# bcast@7: prefix=[G] suffix=[H, W] M=C/G subs={}
e: fold(dim=3,avg) (7) -> 8
e: fold(dim=2,avg) (8) -> 9
e: bcast(add) (9,0) -> 10
# bcast@10: prefix=[] suffix=[H, W] M=1 subs={}
vars: x1
"""

SEED7_K0 = """\
canvas-ir v1
n0: shape=[C; H, W]
n1: shape=[C; H, W]
n2: shape=[C; W]
n3: shape=[G, C/G; H, W]
n4: shape=[C; H, W]
n5: shape=[KW, C; H, W]
n6: shape=[C; W]
n7: shape=[C; H, W]
n8: shape=[C; H, W]
n9: shape=[C; H, W]
e: ew(neg) (0) -> 1
e: fold(dim=1,max) (0) -> 2
e: group(G) (1) -> 3
e: ew(abs) (1) -> 4
e: unfold(w,at=0) (4) -> 5
e: softmax(0..0) (2) -> 6
e: fold(dim=0,max) (5) -> 7
e: bcast(max) (6,7) -> 8
# bcast@8: prefix=[C] suffix=[W] M=H subs={}
e: bcast(sub) (3,8) -> 9
# bcast@9: prefix=[] suffix=[H, W] M=1 subs={}
"""

SEED7_K1 = """\
canvas-ir v1
n0: shape=[C; H, W]
n1: shape=[C; H, W]
n2: shape=[C, KH; H, W]
n3: shape=[C, KW, KH; H, W]
n4: shape=[G; H, W]
n5: shape=[G, C/G; H, W]
n6: shape=[G, 1, C/G; H, W]
n7: shape=[G, 1, C/G; H, W]
n8: shape=[C, KW, KH; H, W]
n9: shape=[C; H, W]
e: softmax(0..0) (0) -> 1
e: unfold(h) (1) -> 2
e: unfold(w,at=1) (2) -> 3
e: fc(G) (0) -> 4
e: group(G) (0) -> 5
e: group(G) (5) -> 6
e: bcast(min) (4,6) -> 7
# bcast@7: prefix=[G] suffix=[H, W] M=C/G subs={}
e: bcast(min) (7,3) -> 8
# bcast@8: prefix=[] suffix=[H, W] M=KH*KW subs={}
e: fc(C) (8) -> 9
"""

NEG = """\
canvas-ir v1
n0: shape=[C; H, W]
n1: shape=[C; H, W]
e: ew(neg) (0) -> 1
"""

ALL = {"seed7_k1": SEED7_K1, "seed7_k0": SEED7_K0, "im2col": IM2COL, "involution": INVOLUTION, "neg": NEG}
