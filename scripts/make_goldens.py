"""Generate golden fixtures for tests/golden/ FROM THE REFERENCE ITSELF.

Run in the build container only (the reference is not present on GPU boxes):

    PYTHONPATH=/root/reference/pkg/src python scripts/make_goldens.py

Writes:
  tests/golden/sampler_<N>_<seed>_<count>.cir   concatenated ``emit`` texts of
                                                 Sampler(SamplerConfig(nodes=N, seed=S)).sample_many(count)
  tests/golden/frontend.json                    per-kernel iso_hash, per-edge (flops, params), node extents
                                                 at the config-1 assignment, broadcast matchings, sha256
                                                 digests and SampleCounts — all computed by the reference.
                                                 Also the App.-B kernels (seed-7 #0/#1, im2col,
                                                 Involution) re-emitted by the reference ("pinned").

The committed outputs are what the CPU tests pin the host-side mirror
(paper_2304_07741_b200.canvas) against; this script is not imported by any
test or product code.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "..", "tests", "golden")

from canvas import ir, micro_dag, primitives, shape_algebra  # noqa: E402  (reference package)
from canvas.sampler import Sampler, SamplerConfig  # noqa: E402
from canvas.shape_solver import match_broadcast  # noqa: E402

SWEEPS = [(2, 7, 1), (10, 7, 20), (10, 7, 256), (16, 7, 64), (20, 0, 16)]

CONFIG1 = {"C": 64, "G": 4, "H": 56, "W": 56, "KH": 3, "KW": 3}

PINNED = {
    "im2col": """canvas-ir v1
n0: shape=[C; H, W]
n1: shape=[C, KH; H, W]
n2: shape=[C, KH, KW; H, W]
n3: shape=[C; H, W]
e: unfold(h) (0) -> 1
e: unfold(w) (1) -> 2
e: fc(C) (2) -> 3
""",
    "involution": None,  # built through the reference API below
}


def involution_ir() -> str:
    sa = shape_algebra
    g = micro_dag.MicroDag.initial()
    g = micro_dag.grow_kind(g, primitives.FullyConnected(sa.var_dim(1)), (0,))
    g = micro_dag.grow_kind(g, primitives.FullyConnected(sa.var_dim(2)), (1,))
    g = micro_dag.substitute_dag(g, 2, sa.multiply(sa.multiply(sa.D_G, sa.D_KH), sa.D_KW))
    g = micro_dag.grow_kind(g, primitives.Group(0, "G"), (2,))
    g = micro_dag.grow_kind(g, primitives.Group(0, "G"), (0,))
    g = micro_dag.grow_kind(g, primitives.Unfold("h", None), (4,))
    g = micro_dag.grow_kind(g, primitives.Unfold("w", None), (5,))
    g = micro_dag.grow_kind(g, primitives.Broadcast("mul"), (3, 6))
    g = micro_dag.grow_kind(g, primitives.Fold(3, "avg"), (7,))
    g = micro_dag.grow_kind(g, primitives.Fold(2, "avg"), (8,))
    g = micro_dag.grow_kind(g, primitives.Broadcast("add"), (9, 0))
    return ir.emit(micro_dag.finalize(g))


def describe(t, x_value: int = 64) -> dict:
    a = shape_algebra.Assignment(CONFIG1, {v: x_value for v in t.free_vars})
    edges = []
    for e in t.dag.edges:
        rec = {"mn": primitives.mnemonic(e.inst.kind), "in": list(e.inputs), "out": e.out}
        try:
            rec["cost"] = list(primitives.cost(e.inst, a))
        except shape_algebra.NonIntegral:
            rec["cost"] = None
        if isinstance(e.inst.kind, primitives.Broadcast):
            m = match_broadcast(e.inst.inputs[0], e.inst.inputs[1])
            rec["match"] = {
                "region": m.region,
                "lhs_span": list(m.lhs_span),
                "rhs_span": list(m.rhs_span),
                "ratio": None if m.ratio is None else m.ratio.render(),
                "audit": m.audit(),
            }
        edges.append(rec)
    extents = []
    for s in t.dag.nodes:
        try:
            extents.append([shape_algebra.evaluate(d, a) for d in s.dims()])
        except shape_algebra.NonIntegral:
            extents.append(None)
    return {
        "iso_hash": f"{micro_dag.iso_hash(t.dag):016x}",
        "free_vars": list(t.free_vars),
        "edges": edges,
        "extents": extents,
    }


def main() -> None:
    os.makedirs(OUT, exist_ok=True)
    manifest: dict = {"assignment": CONFIG1, "x_value": 64, "sweeps": {}, "pinned": {}}
    for n, seed, count in SWEEPS:
        s = Sampler(SamplerConfig(nodes=n, seed=seed))
        ks = s.sample_many(count)
        texts = [ir.emit(k) for k in ks]
        blob = "".join(texts)
        name = f"sampler_{n}_{seed}_{count}"
        with open(os.path.join(OUT, name + ".cir"), "w") as f:
            f.write(blob)
        manifest["sweeps"][name] = {
            "nodes": n,
            "seed": seed,
            "count": count,
            "sha256": hashlib.sha256(blob.encode()).hexdigest(),
            "counts": s.counts.as_dict(),
            "kernels": [describe(k) for k in ks] if (n, count) in ((10, 256), (2, 1), (10, 20)) else None,
        }
        print(name, manifest["sweeps"][name]["sha256"], s.counts.as_dict(), file=sys.stderr)

    PINNED["involution"] = involution_ir()
    ks10 = [ir.parse("canvas-ir v1\n" + t).template for t in open(os.path.join(OUT, "sampler_10_7_20.cir")).read().split("canvas-ir v1\n")[1:]]
    pinned_texts = {
        "seed7_k0": ir.emit(ks10[0]),
        "seed7_k1": ir.emit(ks10[1]),
        "im2col": ir.emit(ir.parse(PINNED["im2col"]).template),
        "involution": PINNED["involution"],
    }
    for key, text in pinned_texts.items():
        t = ir.parse(text).template
        manifest["pinned"][key] = {"ir": text, **describe(t)}
    # Reference API examples the executor relies on (SPEC/test anchors).
    manifest["anchors"] = {
        "iso_empty": f"{micro_dag.iso_hash(micro_dag.MicroDag((), ())):016x}",
        "iso_input": f"{micro_dag.iso_hash(micro_dag.MicroDag.initial()):016x}",
    }
    with open(os.path.join(OUT, "frontend.json"), "w") as f:
        json.dump(manifest, f, sort_keys=True, separators=(",", ":"))


if __name__ == "__main__":
    main()
