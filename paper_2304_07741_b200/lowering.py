"""Lowering: concrete kernel graph -> fused device-kernel plan (+ its adjoint).

This is the host half of the hot path (SURVEY §3.4 "new build", §7 decisions
2-3).  Given a :class:`~paper_2304_07741_b200.graph.ConcreteGraph` it decides

* which node values are **materialised** in HBM.  Only reductions and
  contractions are: Fold, Softmax, FC outputs, plus the kernel output.  Every
  rearrangement (Group/Shift/Unfold) and every pointwise op (ew, bcast) is
  *inlined* into the loads of its consumer as index arithmetic + zero
  predicates (north star: "rearrangement primitives are never materialised");
* the backward schedule: the adjoint of every primitive is a *pull* (gather)
  expression — col2im-as-gather for Unfold, replica sums for Broadcast LHS,
  tie-split for max/min — so no atomics are needed and results are
  bitwise deterministic (SURVEY §7 decision 5);
* the device kernels: each materialised tensor is produced by one launch of a
  hand-written template from ``csrc/kernels/canvas_kernels.cuh``
  (``pointwise``, ``gemm_nk``, ``gemm_wgrad``/``reduce_partials``), instantiated
  with a *functor* this module emits — straight-line C++ that evaluates the
  node's producer chain at one coordinate with compile-time extents (so every
  index div/mod is a multiply-shift).

The result is a :class:`Plan` whose ``blob()`` is the flat POD payload the
C-ABI ``canvas_plan_create`` consumes (include/canvas_b200.h).

Numeric conventions: unfold U[..k..,h] = I[.., h+k-K//2] zero
padded, per-stage predicates (A.3); shift out[h] = in[h+off] (A.2); bcast tile
order lhs index = r mod L, ``sub`` = lhs - rhs, min/max ties split 1/2 (A.8);
fold max ties split evenly (A.6); relu'(0) = abs'(0) = 0 (A.5); softmax
max-subtracted (A.7); FC dense, bias-free, W[out, prod(in ch)] (A.4).
"""

from __future__ import annotations

import math
import os
import re
import struct
from dataclasses import dataclass, field

from .graph import VIEW_OPS, ConcreteGraph, LoweringError

ABI_VERSION = 1
BLOB_MAGIC = b"CNVSBLOB"
_IDENT = re.compile(r"[A-Za-z_]\w*")
MAX_KSLOTS = 24  # pointers per kernel argument block (csrc/kernels/canvas_kernels.cuh)

# fixed global slots; weights / grads / saved / workspace follow (see Plan.slot_*)
SLOT_X, SLOT_Y, SLOT_DY, SLOT_DX = 0, 1, 2, 3

# beta policies for stores into caller-visible outputs shared by the r copies (Fig.-2)
BETA_NONE, BETA_AFTER_FIRST, BETA_ALWAYS = 0, 1, 2

POINTWISE_BLOCK = 256
POINTWISE_VEC = int(os.environ.get("CANVAS_PW_VEC", "1"))  # elements per thread along the innermost dim
POINTWISE_CAP = 148 * 8 * 4  # grid-stride: 4 waves of 8 x 256-thread CTAs per SM
SAVE_OPERAND = os.environ.get("CANVAS_SAVE_OPERAND", "0") == "1"  # FC forward keeps a computed operand for the wgrad (measured slower: off)
PLANES_MIN_S = int(os.environ.get("CANVAS_PLANES_MIN_S", "128"))  # plane-major launch when H*W >= this (0 = off)
PLANES_CTAS = int(os.environ.get("CANVAS_PLANES_CTAS", str(148 * 64)))  # CTAs of a plane-major launch (planes strided)
GEMM_TILE = 64
SLOT_GUARD = 16384  # bytes of guard zone on each side of every saved / workspace tensor (canvas_runtime.cpp kGuard)
MAX_BATCH = 1024  # images per call; bounds the 32-bit offset arithmetic (canvas_plan_create checks)
REPLICATE_MIN = 4  # materialise a pointwise node re-evaluated this many times per consumer element
FC_SMALL_W4 = os.environ.get("CANVAS_FC_SMALL_W4", "0") == "1"  # per-pixel small FC: 16 B weight rows (measured slower: 0.080 vs 0.070 ms)
FC_SMALL_UNROLL = int(os.environ.get("CANVAS_FC_SMALL_UNROLL", "16"))  # per-pixel small FC input-loop unroll (0: Fn.loop default; 16: 0.070 -> 0.068 ms scalar, needed by the quads)
FC_SMALL_VEC_FILL = int(os.environ.get("CANVAS_FC_SMALL_VEC_FILL", "1024"))  # per-pixel small FC: quads when batch-256 quads >= SMS x this (fc(G) 4x64 at 56^2: 0.070 -> 0.056 ms with unroll 16; at 28^2 quads are slower, 0.081 vs 0.047)
ASM_LOADS = os.environ.get("CANVAS_ASM_LOADS", "planes")  # loads-first bodies: hoisted gathers as volatile PTX loads (order kept by ptxas): "planes" = plane-major launches only (grad n1: layer3 1.385 -> 1.348 ms, layer2 -0.5%, layers 1/4 flat), "1" all (grad n1 at 7x7 0.088 -> 0.099 ms, grad n7 +5% at 14x14), "0" off
LOADS_FIRST = os.environ.get("CANVAS_LOADS_FIRST", "1") == "1"  # pointwise bodies: gathers hoisted above the arithmetic (grad n1: 0.186 -> 0.165 ms at 14^2, 0.113 -> 0.086 at 7^2, 56^2 unchanged)
FC_SMALL_KS = os.environ.get("CANVAS_FC_SMALL_KS", "1") == "1"  # per-output small FC with few pixels: K split over lanes
WGRAD_SMALL_V = os.environ.get("CANVAS_WGRAD_SMALL_V", "1") == "1"  # register-blocked quad wgrad for M <= 16
WGRAD_SMALL_JT_MAX = 128  # wgrad_small stages (M + JT) x 65 floats: <= 48 KB of static shared memory for M <= 56
INLINE_SMALL_DGRAD = os.environ.get("CANVAS_INLINE_SMALL_DGRAD", "1") == "1"  # few-output FC dgrad inlined into the gradient sum
SOFTMAX_REG_SPAN = int(os.environ.get("CANVAS_SOFTMAX_REG_SPAN", "64"))  # softmax rows up to this long are held in registers
SMALL_FC = 16  # min(out, K) at or below which an FC is a per-pixel SIMT dot (K4 fc_small)
TC_THREADS = 320  # tcgen05 GEMM: 8 producer/epilogue warps + MMA warp + bulk-copy warp
TC_SMEM_BUDGET = 200 * 1024
TC_SMEM_PAIR = 110 * 1024 if os.environ.get("CANVAS_TC_PAIR", "1") == "1" else 0  # two CTAs/SM when a 2-stage ring fits
TC_A_MN = "true" if os.environ.get("CANVAS_TC_AMN", "1") == "1" else "false"  # computed operand layout
TC_NTMAX = int(os.environ.get("CANVAS_TC_NTMAX", "256"))  # widest MMA N tile
TC_PERSIST = os.environ.get("CANVAS_TC_PERSIST", "1") == "1"  # persistent fwd/dgrad GEMMs
TC_PW = int(os.environ.get("CANVAS_TC_PW", "16"))  # producer warps of the persistent GEMM when K > 128 (16 vs 8: +0.4% img/s on config 2, no spills)
SMS = 148
VEC_PRODUCERS = os.environ.get("CANVAS_VEC", "1") == "1"  # tcgen05 producers evaluate 4 consecutive pixels per thread
VEC_POINTWISE = os.environ.get("CANVAS_VEC_PW", "1") == "1"  # pointwise launches: 4 consecutive elements per thread
VEC16 = os.environ.get("CANVAS_VEC16", "1") == "1"  # aligned quads as one 16 B load / store
VEC_RT = int(os.environ.get("CANVAS_VEC_RT", "0"))  # quads at a run-time 4 B offset: two 16 B loads + select (1: selects, 2: one branch per quad with producer rows grouped by shift class; measured 1.5-2.3x slower on the layer1 GEMMs: off)
TC_TMEMA_PW = int(os.environ.get("CANVAS_TMEMA_PW", "8"))  # its producer warps (4 lane quadrants x k shares; 16 measured 0.64 vs 0.40 ms on layer1: one CTA per SM)
TC_TMEMA = os.environ.get("CANVAS_TMEMA", "auto")  # FC forward with the computed operand staged in TMEM (tcgen05.mma A from TMEM): "auto" = when its k loop unrolls fully (K <= TMEMA_UNROLL_MAX), "1" always, "0" never
TMEMA_STAGES = int(os.environ.get("CANVAS_TMEMA_STAGES", "0"))  # TMEM-A operand stages (0: 3, or 2 when that pairs CTAs)
TMEMA_UNROLL_MAX = int(os.environ.get("CANVAS_TMEMA_UNROLL_MAX", "1024"))  # fully unrolled TMEM-A producers up to this K (layer1 FC forward 0.656 -> 0.390 ms; without the unroll TMEM-A measured 0.79 ms; at 2304: layer2 K = 1152 0.40 -> 0.54 ms — NT = 128 + 3 A stages > 256 TMEM columns, one CTA per SM — layer3 0.26 -> 0.25)


def tmema_wanted(K: int) -> bool:
    mode = str(TC_TMEMA)
    return mode in ("1", "True") or (mode == "auto" and K <= TMEMA_UNROLL_MAX)
VEC_PAD = os.environ.get("CANVAS_VEC_PAD", "1") == "1"  # S % 4 != 0: wgrad producers on quads of a padded pixel range
VEC_PAD_MIN_LOADS = int(os.environ.get("CANVAS_VEC_PAD_MIN_LOADS", "2"))
VEC_PAD_FWD = os.environ.get("CANVAS_VEC_PAD_FWD", "0") == "1"  # same for the FC forward / dgrad quads (7x7 fwd fc: 0.524 vs 0.428 ms scalar: off)
VEC_NQ = os.environ.get("CANVAS_VEC_NQ", "0") == "1"  # S % 4 != 0: wgrad producers take quads of 4 images at one pixel (measured 2.7x slower at 7x7: image-strided lanes break coalescing; off)
VEC_SPLIT = os.environ.get("CANVAS_VEC_SPLIT", "1") == "1"  # software-pipelined producers (loads one k-block ahead)
GRAD_SIBLINGS = os.environ.get("CANVAS_GRAD_SIBLINGS", "0") == "1"  # two gradient tensors of one shape in one launch (seed-7 #1 dn7 + dn1: 1.20 vs 0.88 ms, their gathers share no lines: off)
ROW_KEYS = os.environ.get("CANVAS_ROW_KEYS", "1") == "1"  # wgrad producers: tile rows ordered by their gather offset
GRAD_INLINE = os.environ.get("CANVAS_GRAD_INLINE", "1") == "1"  # pointwise gradients pulled inline instead of materialised
FOLD_INLINE = int(os.environ.get("CANVAS_FOLD_INLINE", "3"))  # folds over at most this many values are evaluated inline
PLANES_GUARDED = os.environ.get("CANVAS_PLANES_GUARDED", "0") == "1"  # plane-major launches also for guarded gathers
VEC_SHIFTED = os.environ.get("CANVAS_VEC_SHIFTED", "0") == "1"  # quads also when most gathers sit at sub-16 B shifts
EPI_BC = os.environ.get("CANVAS_EPI_BC", "0") == "1"  # FC dgrad epilogue applies the input broadcast's adjoint (built + parity-tested; measured 1.10 ms vs 0.81 ms for dgrad + replica-sum on layer1: off)
EPI_WPB = int(os.environ.get("CANVAS_EPI_WPB", "1"))  # epilogue warpgroups per TMEM buffer (column shares; 2 measured slower: spills at 960 threads)
EPI_PREFETCH = os.environ.get("CANVAS_EPI_PF", "1") == "1"  # ... with the next replica's operand gathers in flight
TC_ACC_K = int(os.environ.get("CANVAS_TC_ACC_K", "1152"))  # max reduction length per TMEM accumulator
L2_PREFETCH = os.environ.get("CANVAS_L2_PREFETCH", "0") == "1"  # producers prefetch their source rows into L2 (measured no gain: off)
TC_WGRAD_JG_MAX = int(os.environ.get("CANVAS_WGRAD_JG", "1"))  # max row tiles per wgrad CTA (1 vs 2: +0.5% img/s on config 2 with 8192-pixel chunks)
TC_WGRAD_TCHUNK = int(os.environ.get("CANVAS_WGRAD_TCHUNK", "8192"))  # max pixels per wgrad partial (8192 vs 4096: +0.3% img/s on config 2)
TC_WGRAD_PW = int(os.environ.get("CANVAS_WGRAD_PW", "16"))  # wgrad producer warps
TC_PIX_PW = int(os.environ.get("CANVAS_PIX_PW", "0"))  # 0 = auto  # fwd/dgrad (non-persistent) producer warps  # pixels per wgrad split (128 k-blocks of 32)


def tc_tile(cols: int, ntmax: int | None = None) -> tuple[int, int, int]:
    """(NT, number of column tiles, pipeline stages) for an MMA N extent of ``cols``."""
    nct = -(-cols // (ntmax or TC_NTMAX))
    nt = -(-(-(-cols // nct)) // 16) * 16
    stage = 2 * 128 * 128 + 2 * nt * 128
    if 2 * stage + 2048 <= TC_SMEM_PAIR:
        return nt, nct, 2
    stages = max(2, min(4, TC_SMEM_BUDGET // stage))
    return nt, nct, stages


def wgrad_smem_bytes(nt: int, jg: int, stages: int) -> int:
    """Must match canvas::tc::SmemW<NT, JG, STAGES>::BYTES."""
    return stages * (2 * jg * 128 * 128 + 2 * nt * 128) + (2 * stages + 1) * 8 + 16 + 1024


def wgrad_jg(J: int, nt: int) -> int:
    """Row tiles of 128 input channels per wgrad CTA: the output-channel operand
    (nt rows) is gathered once per group, so group as many tiles as TMEM
    (jg*nt <= 512 columns) and a 2-stage ring in 220 KB of smem allow."""
    jg = 1
    if nt < 128:  # measured: at NT = 64 (layer1) grouping is slower (fewer, longer CTAs)
        return 1
    for cand in range(2, TC_WGRAD_JG_MAX + 1):
        if cand * nt <= 512 and wgrad_smem_bytes(nt, cand, 2) <= 220 * 1024 and J > 128 * (cand - 1):
            jg = cand
    return jg


def tc_persist_cfg(nt: int) -> tuple[int, int]:
    """(stages, smem bytes) of tc_gemm_pix_persistent (must match canvas::SmemP)."""
    stage = 2 * 128 * 128 + 2 * nt * 128
    stages = max(2, min(6, (220 * 1024) // stage))
    return stages, stages * stage + (2 * stages + 16) * 8 + 16 + 1024


def tc_smem_bytes(nt: int, stages: int) -> int:
    """Must match canvas::tc::Smem<NT, STAGES>::BYTES."""
    return stages * (2 * 128 * 128 + 2 * nt * 128) + (2 * stages + 1) * 8 + 16 + 1024


@dataclass
class TDesc:
    """Where a tensor lives: global slot + strides (elements).  ``dims`` are
    the node extents; ``strides`` per dim; ``bstride`` per image."""

    slot: int
    bstride: int
    strides: tuple
    dims: tuple


@dataclass
class SizeRule:
    """bytes(N) = ceil(N * a_num / a_den) + b."""

    a_num: int
    a_den: int
    b: int

    def eval(self, n: int) -> int:
        return -(-n * self.a_num // self.a_den) + self.b


@dataclass
class GridRule:
    """g = min(ceil((a*N + b) / d), cap) (cap 0 = none)."""

    a: int
    b: int
    d: int
    cap: int = 0

    def eval(self, n: int) -> int:
        g = -(-(self.a * n + self.b) // self.d)
        return min(g, self.cap) if self.cap else g


@dataclass
class Launch:
    kind: str  # "kernel" | "memset"
    phase: int  # 0 forward, 1 backward
    name: str = ""
    kernel: int = -1
    block: int = 256
    grid: tuple = ()
    slots: tuple = ()
    beta: int = BETA_NONE
    memset_slot: int = -1
    memset_size: SizeRule | None = None
    smem: int = 0  # dynamic shared memory bytes
    what: str = ""  # human-readable role (profiles / DESIGN tables)
    bytes_per_image: int = 0  # algorithmic HBM bytes per image (roofline)
    flops_per_image: int = 0  # useful FLOPs per image (2 per MAC)
    align16: bool = False  # the kernel issues 16 B accesses: the runtime checks slot pointers (blob kind 2)


@dataclass
class Plan:
    graph: ConcreteGraph
    c_in: int
    c_out: int
    stride: int
    h_in: int
    w_in: int
    copies: int
    mode: str  # "concat" (C_out = r C_in) or "sum" (C_in = r C_out)
    source: str = ""
    kernel_names: list = field(default_factory=list)
    launches: list = field(default_factory=list)
    saved: list = field(default_factory=list)  # SizeRule per saved slot (one copy)
    ws: list = field(default_factory=list)  # SizeRule per workspace slot
    x_copy_off: int = 0
    y_copy_off: int = 0
    dx_copy_off: int = 0
    dy_copy_off: int = 0
    fwd_mat: dict = field(default_factory=dict)  # node -> TDesc of its forward value
    notes: list = field(default_factory=list)

    @property
    def n_fc(self) -> int:
        return len(self.graph.fc_nodes)

    def slot_w(self, i: int) -> int:
        return 4 + i

    def slot_dw(self, i: int) -> int:
        return 4 + self.n_fc + i

    def slot_saved(self, k: int) -> int:
        return 4 + 2 * self.n_fc + k

    def slot_ws(self, k: int) -> int:
        return 4 + 2 * self.n_fc + len(self.saved) + k

    # -- C-ABI payload ---------------------------------------------------------------
    def blob(self) -> bytes:
        """Flat little-endian payload parsed by csrc/canvas_runtime.cpp (format v1).

        header: magic[8], then int64s: version, n_kernels, n_launches, n_saved,
        n_ws, n_fc, copies, x_copy_off, y_copy_off, dx_copy_off, dy_copy_off,
        max_batch, src_len, names_len; then (a_num, a_den, b) per saved and per ws slot;
        then per launch: kind, phase, kernel, block, smem, 3x(a,b,d,cap), nslots,
        slots[MAX_KSLOTS], beta, memset_slot, memset (a_num,a_den,b); then the
        CUDA source and the NUL-separated kernel names.
        """
        names = b"\0".join(n.encode() for n in self.kernel_names) + b"\0"
        src = self.source.encode()
        q = struct.Struct("<q")
        out = bytearray(BLOB_MAGIC)
        hdr = [ABI_VERSION, len(self.kernel_names), len(self.launches), len(self.saved), len(self.ws), self.n_fc, self.copies, self.x_copy_off, self.y_copy_off, self.dx_copy_off, self.dy_copy_off, MAX_BATCH, len(src), len(names)]
        for v in hdr:
            out += q.pack(v)
        for r in self.saved + self.ws:
            out += struct.pack("<3q", r.a_num, r.a_den, r.b)
        for L in self.launches:
            grid = list(L.grid) if L.grid else [GridRule(0, 1, 1)] * 3
            slots = list(L.slots) + [-1] * (MAX_KSLOTS - len(L.slots))
            ms = L.memset_size or SizeRule(0, 1, 0)
            out += struct.pack("<5q", (2 if L.align16 else 0) if L.kind == "kernel" else 1, L.phase, L.kernel, L.block, L.smem)
            for g in grid:
                out += struct.pack("<4q", g.a, g.b, g.d, g.cap)
            out += struct.pack("<q", len(L.slots))
            out += struct.pack(f"<{MAX_KSLOTS}q", *slots)
            out += struct.pack("<5q", L.beta, L.memset_slot, ms.a_num, ms.a_den, ms.b)
        out += src + names
        return bytes(out)

    # -- helpers used by module / bench ------------------------------------------------
    def sizes(self, n: int) -> tuple[int, int, int]:
        """(saved bytes for all copies, workspace bytes, fwd workspace bytes) at batch n."""
        al = lambda b: (b + 255) // 256 * 256 + 2 * SLOT_GUARD  # noqa: E731  (canvas_runtime.cpp slot_bytes)
        saved = sum(al(r.eval(n)) for r in self.saved) * self.copies
        ws = sum(al(r.eval(n)) for r in self.ws)
        return saved, ws, 0


# ====================================================================================
# Code emission
# ====================================================================================

_EW_FWD = {
    "relu": "fmaxf({0}, 0.f)",
    "abs": "fabsf({0})",
    "sin": "sinf({0})",
    "exp": "expf({0})",
    "neg": "(-{0})",
}
# forward values are recomputed inline by other kernels (adjoints, inlined
# gradients) and compared for max/min ties (App. A.6/A.8): the round-to-nearest
# intrinsics keep the compiler from contracting a product with a neighbouring
# add/sub into an FMA in one context but not in another
_BC_FWD = {
    "add": "__fadd_rn({0}, {1})",
    "sub": "__fsub_rn({0}, {1})",
    "mul": "__fmul_rn({0}, {1})",
    "min": "fminf({0}, {1})",
    "max": "fmaxf({0}, {1})",
}


class VecUnsupported(Exception):
    """The functor body cannot be emitted in 4-pixel vector form (loops, caller-written
    code, a pixel coordinate used non-affinely where the lanes would diverge)."""


_TERM = re.compile(r"^\(?(-?\w+)\)?(?:\*\(?(-?\d+)\)?)?$")
_MODDIV = re.compile(r"^(\w+) ([%/]) (\d+)$")


def _split_top(expr: str, sep: str = " + ") -> list:
    """Split ``expr`` on ``sep`` outside parentheses."""
    out, depth, cur, i = [], 0, [], 0
    while i < len(expr):
        ch = expr[i]
        if ch == "(":
            depth += 1
        elif ch == ")":
            depth -= 1
        if depth == 0 and expr.startswith(sep, i):
            out.append("".join(cur))
            cur = []
            i += len(sep)
            continue
        cur.append(ch)
        i += 1
    out.append("".join(cur))
    return out


class Fn:
    """Straight-line code for one functor body with memoised coordinates/values.

    Coordinates are C ``int`` expressions; the memo keys on their text, so a
    coordinate reached twice (diamonds, shared prefixes) is computed once
    (common-subexpression elimination at emission time)."""

    def __init__(self, lw: "Lowerer", indent: int = 2):
        self.lw = lw
        self.lines: list[str] = []
        self.scopes: list[dict] = [{}]
        self.indent = indent
        self.k = 0
        self.local_slots: list[int] = []
        self.bases: dict = {}
        self.flat_of: dict = {}  # coordinate tuple -> (flat index var, extents)
        self.raw: set = set()  # coordinate vars that may be out of range (Shift/Unfold sources)
        self.lin_of: dict = {}  # affine coordinate var -> ((var, coef)...), const
        # in-range predicates every load must also satisfy: set while evaluating a
        # computed node at raw (possibly out-of-range) coordinates whose value is
        # selected away when the predicates fail (no clamps, no OOB access)
        self.guard: tuple = ()
        # plane-major functors: (channel extents, spatial extents) of the output whose
        # flat index r = q * S + s is split into a block-uniform plane q and a
        # per-thread spatial s (pointwise_planes)
        self.planes: tuple | None = None
        # warp-/block-uniform index variables (seeded by the caller: "k" rows of a
        # tcgen05 producer, "q"/"n" of a plane-major functor).  Offsets are emitted
        # as (per-lane part) + (uniform part) so the uniform part is shared by all
        # lanes and the per-lane part by all rows: one IMAD.WIDE per gathered element
        self.uniform: set = set()
        # hoist: uniform ivars (functions of the uniform row variable only) are
        # emitted into ``uni_lines`` — the functor's row context, evaluated once
        # per row by the GEMM producers instead of once per element
        self.hoist = False
        self.uni_lines: list[str] = []
        self.uni_vars: list[str] = []
        self.loaded: dict = {}  # (slot, image stride) -> TDesc of every tensor this functor reads
        # vector mode (V > 1): the functor evaluates V consecutive pixels s0 .. s0+V-1
        # (s0 a multiple of V, all in one image).  An int var in ``lanes`` holds its
        # lane-0 value and lane e is var + coef*e (value (coef, align): lane-0 value is
        # a multiple of align); a var in ``copies`` exists per lane as var_0 .. var_{V-1}.
        # Everything else is lane-invariant and shared by the V pixels — the channel /
        # tap / row index math, the image base, the row part of every address.
        self.V = 1
        self.lanes: dict = {}
        self.copies: set = set()
        # element alignment of int vars (their value is a multiple of it; lane-0 value
        # for lane vars): lane-affine unit-stride accesses whose offset is a multiple
        # of 4 become one 16 B access (slot pointers are 16 B aligned: launch kind 2)
        self.al: dict = {}
        self.vec16 = False
        self.ltags: list = []
        self.cur_tag = None
        # lane-context hoisting (the dual of ``hoist``): int / pointer values that depend
        # only on the thread's pixel (n, s) go to ``ctx_lines`` — evaluated once per
        # tile by the TMEM epilogue instead of once per column
        # vector mode over 4 consecutive *images* at one pixel (S % 4 != 0: pixel
        # quads would straddle images): the image bases are the lane-affine vars
        self.lane_n = False
        # vector mode over a padded pixel range (S % 4 != 0): the per-lane validity
        # every load must also satisfy (pixels past S are padding)
        self.lane_pred = ""
        self.ctxh = False
        self.ctx_ok: set = set()
        self.ctx_lines: list[str] = []
        self.ctx_vars: list[tuple] = []  # (ctype, name)
        self.nld = {"aligned": 0, "shifted": 0, "lanes": 0}  # vector-mode load sites by kind
        self.rt_cls: list = []  # row-context offsets of the run-time-shift quads (producer row grouping)
        self.row_keys: list = []  # row-context offsets of the static unit-stride quads (producer row ordering)

    # -- bookkeeping -----------------------------------------------------------
    def emit(self, s: str) -> None:
        """Emit a caller-written statement.  Vector mode: mutable float declarations
        (accumulators, register rows) and statements that read lane values are
        emitted once per lane with the lane's names substituted; lane-invariant
        statements (loop headers, braces) once.  Caller-written ``const``
        bindings are refused (their names would collide across lanes)."""
        if self.V == 1:
            self._emit(s)
            return
        st = s.strip()
        if st.startswith("const "):
            raise VecUnsupported(s)
        if st.startswith("float "):
            body = st[len("float "):].rstrip(";").replace("; float ", ", ")
            for decl in _split_top(body, ", "):
                self.copies.add(re.match(r"\s*(\w+)", decl).group(1))
        elif not self.lane_vars(s):
            self._emit(s)
            return
        if s.count("{") != s.count("}"):
            raise VecUnsupported(s)
        for e in range(self.V):
            self._emit(self.subst(s, e))

    def _emit(self, s: str) -> None:
        self.lines.append("  " * self.indent + s)
        # line kinds for the load / compute split of operand functors: 'i' index
        # math and addresses, 'l' loads, 'c' float arithmetic, 'x' anything else
        st = s.lstrip()
        if self.cur_tag:
            tag = self.cur_tag
        elif st.startswith(("const int ", "float* const ", "const float* const ")):
            tag = "i"
        elif st.startswith("const float ") and "__ldg" not in st:
            tag = "c"
        else:
            tag = "x"
        self.ltags.append(tag)

    # -- vector mode ------------------------------------------------------------
    def lane_vars(self, expr: str) -> set:
        return {t for t in _IDENT.findall(expr) if t in self.lanes or t in self.copies}

    def subst(self, expr: str, e: int) -> str:
        """``expr`` at lane e."""

        def rep(m):
            t = m.group(0)
            if t in self.copies:
                return f"{t}_{e}"
            if t in self.lanes and e:
                return f"({t} + {self.lanes[t][0] * e})"
            return t

        return re.sub(r"\b[A-Za-z_]\w*\b", rep, expr)

    # residue classes (A, c): the value is = c (mod A); A = 0 means exactly c
    @staticmethod
    def _radd(x, y):
        g = math.gcd(x[0], y[0])
        return (g, (x[1] + y[1]) % g if g else x[1] + y[1])

    @staticmethod
    def _rmul(x, k: int):
        return (abs(x[0] * k), (x[1] * k) % abs(x[0] * k) if x[0] * k else x[1] * k)

    def residue(self, x: str):
        x = x.strip()
        if x.lstrip("-").isdigit():
            return (0, int(x))
        if x in self.lanes:
            return self.lanes[x][1:]
        return self.al.get(x, (1, 0))

    def affine_info(self, expr: str):
        """(lane coef, A, c) of an int expression — its (lane-0) value is = c mod A —
        or None when it is not affine in the lanes (per-lane copies needed)."""
        m = _MODDIV.match(expr)
        if m:
            x, op, q = m.group(1), m.group(2), int(m.group(3))
            if x in self.copies:
                return None
            A, c = self.residue(x)
            if x not in self.lanes:
                if op == "%":
                    g = math.gcd(A, q)
                    return (0, g, c % g) if g else (0, 0, c % q)
                return (0, 0, c // q) if A == 0 else (0, 1, 0)
            cf = self.lanes[x][0]
            # x0 % q + cf*(V-1) < q and x0 / q shared by the lanes when the lane-0
            # value is = c mod A with A | q and c + cf*(V-1) < A (lanes stay in one A block)
            if cf > 0 and A and q % A == 0 and c + cf * (self.V - 1) < A:
                return (cf, A, c) if op == "%" else (0, 1, 0)
            return None
        coef, res = 0, (0, 0)
        for t in _split_top(expr):
            t = t.strip()
            mt = _TERM.match(t)
            if not mt:
                mp = re.match(r"^\((.*)\)\*\(?(-?\d+)\)?$", t)
                if not mp:
                    return None
                inner = self.affine_info(mp.group(1))
                if inner is None:
                    return None
                k = int(mp.group(2))
                coef += inner[0] * k
                res = self._radd(res, self._rmul(inner[1:], k))
                continue
            x, k = mt.group(1), int(mt.group(2)) if mt.group(2) else 1
            if x in self.copies:
                return None
            if x in self.lanes:
                coef += self.lanes[x][0] * k
            res = self._radd(res, self._rmul(self.residue(x), k))
        return (coef,) + res

    def lane_affine(self, expr: str):
        """(coef, A, c) when ``expr`` (which reads lane vars) is lane-affine with its
        lane-0 value given by the expression itself; None when the lanes diverge."""
        return self.affine_info(expr)

    def define(self, ctype: str, name: str, expr: str, aff=None) -> None:
        """Emit ``ctype name = expr`` — per lane when expr reads lane vars (unless
        ``aff`` = (coef, align) says it is lane-affine: then once, at lane 0)."""
        if self.ctxh and ctype == "float* const" and all(t in self.ctx_ok for t in _IDENT.findall(expr)):
            self.ctx_lines.append(f"{ctype} {name} = {expr};")
            self.ctx_vars.append(("float*", name))
            self.ctx_ok.add(name)
            return
        if self.V > 1 and self.lane_vars(expr):
            if aff is not None:
                self._emit(f"{ctype} {name} = {expr};")
                if aff[0]:
                    self.lanes[name] = aff
                return
            for e in range(self.V):
                self._emit(f"{ctype} {name}_{e} = {self.subst(expr, e)};")
            self.copies.add(name)
            return
        self._emit(f"{ctype} {name} = {expr};")

    def fresh(self, p: str) -> str:
        self.k += 1
        return f"{p}{self.k}"

    def memo_get(self, key):
        for sc in reversed(self.scopes):
            if key in sc:
                return sc[key]
        return None

    def memo_put(self, key, val) -> None:
        self.scopes[-1][key] = val

    def loop(self, var: str, trip: int) -> None:
        """Counted loop; short trips unrolled fully (independent gathers in flight), long ones by 4."""
        self.emit("#pragma unroll" if trip <= 16 else "#pragma unroll 4")
        self.open(f"for (int {var} = 0; {var} < {trip}; ++{var})")

    def open(self, head: str) -> None:
        self.emit(head + " {")
        self.indent += 1
        self.scopes.append({})

    def close(self) -> None:
        self.scopes.pop()
        self.indent -= 1
        self.emit("}")

    def ivar(self, expr: str) -> str:
        expr = str(expr)
        if expr.lstrip("-").isdigit() or expr.isidentifier():
            return expr
        got = self.memo_get(("i", expr))
        if got:
            return got
        v = self.fresh("i")
        uni = bool(self.uniform) and all(t in self.uniform for t in _IDENT.findall(expr))
        if self.ctxh and all(t in self.ctx_ok for t in _IDENT.findall(expr)):
            self.ctx_lines.append(f"const int {v} = {expr};")
            self.ctx_vars.append(("int", v))
            self.ctx_ok.add(v)
        elif uni and self.hoist:
            self.uni_lines.append(f"const int {v} = {expr};")
            self.uni_vars.append(v)
        elif self.V > 1 and self.lane_vars(expr):
            aff = self.lane_affine(expr)
            self.define("const int", v, expr, aff)
        else:
            self._emit(f"const int {v} = {expr};")
        info = self.affine_info(expr)
        if info is not None and info[1] != 1:
            self.al[v] = info[1:]
        self.memo_put(("i", expr), v)
        if uni:
            self.uniform.add(v)
        return v

    def fvar(self, expr: str, key=None) -> str:
        key = key or ("f", expr)
        got = self.memo_get(key)
        if got:
            return got
        v = self.fresh("v")
        self.define("const float", v, expr)
        self.memo_put(key, v)
        return v

    def ptr(self, slot: int) -> str:
        if slot not in self.local_slots:
            if len(self.local_slots) >= MAX_KSLOTS:
                raise LoweringError("kernel needs too many tensors")
            self.local_slots.append(slot)
        return f"a.p[{self.local_slots.index(slot)}]"

    def base(self, d: TDesc) -> tuple[str, str]:
        """(pointer, per-image element offset) of a tensor (``n`` = image index).

        Tensors whose MAX_BATCH images fit in 2^31 elements use 32-bit offset
        arithmetic (one IMAD per access); larger ones a 64-bit image base."""
        key = (d.slot, d.bstride)
        if key in self.bases:
            return self.bases[key]
        b = self.fresh("b")
        # hoisted: emitted into the preamble (before any scope) by the caller
        if self.lane_n:  # lane e = image n + e: the base is lane-affine with coef = image stride
            if d.bstride * MAX_BATCH >= 2**31:
                raise VecUnsupported("64-bit image base")
            self._emit(f"const int {b} = (int)n * {d.bstride};")
            self.lanes[b] = (d.bstride, 1, 0)
            self.bases[key] = (self.ptr(d.slot), b)
            return self.bases[key]
        if d.bstride * MAX_BATCH < 2**31:
            line = f"const int {b} = (int)n * {d.bstride};"
            self.al[b] = (d.bstride, 0)
            r = (self.ptr(d.slot), b)
            ctype = "int"
        else:
            line = f"float* __restrict__ {b} = {self.ptr(d.slot)} + n * {d.bstride}LL;"
            r = (b, "")
            ctype = "float*"
        if self.ctxh:
            self.ctx_lines.append(line)
            self.ctx_vars.append((ctype, b))
            self.ctx_ok.add(b)
        else:
            self.pre.append(line)
        self.bases[key] = r
        return r

    def _offset_terms(self, d: TDesc, coords):
        """Element offset sum(coord_i * stride_i) as an affine form over base
        coordinates, with every run of coordinates that came from decomposing a
        flat index (over contiguous strides) folded back into that index — e.g.
        (h+1)*W + (w+1) -> s + W + 1, (g*(C/G) + j)*S -> c*S."""
        acc: dict = {}
        const = 0
        for c, st in zip(coords, d.strides):
            if st == 0:
                continue
            t, k = self.lin(c)
            const += k * st
            for v, q in t.items():
                acc[v] = acc.get(v, 0) + q * st
        for dec, (flat, ext) in sorted(self.flat_of.items(), key=lambda kv: -len(kv[0])):
            L = len(dec)
            for j in range(L - 1):  # window dec[j:], longest first
                vars_ = [(v, e) for v, e in zip(dec[j:], ext[j:])]
                live = [(i, v) for i, (v, e) in enumerate(vars_) if v != "0" and e > 1]
                if len(live) < 2 or any(v not in acc for _, v in live):
                    continue
                inner = [math.prod(e for _, e in vars_[i + 1 :]) for i in range(len(vars_))]
                alpha = acc[live[-1][1]] // inner[live[-1][0]] if acc[live[-1][1]] % inner[live[-1][0]] == 0 else None
                if alpha is None or any(acc[v] != alpha * inner[i] for i, v in live):
                    continue
                sub = flat if j == 0 else self.suffix(flat, math.prod(ext[j:]))
                for _, v in live:
                    del acc[v]
                acc[sub] = acc.get(sub, 0) + alpha
                break
        return acc, const

    def offset_parts(self, d: TDesc, coords) -> tuple[str, str]:
        """(per-lane part, uniform part) of the element offset, each an int var or "0"."""
        acc, const = self._offset_terms(d, coords)

        def join(items, c=0):
            terms = [f"{v}" if k == 1 else f"{v}*{k}" for v, k in sorted(items, key=lambda kv: -abs(kv[1])) if k]
            if c:
                terms.append(f"({c})")
            return self.ivar(" + ".join(terms) if terms else "0")

        uni = [(v, k) for v, k in acc.items() if v in self.uniform]
        lane = [(v, k) for v, k in acc.items() if v not in self.uniform]
        if not self.uniform or not uni:
            return join(lane, const), "0"
        return join(lane), join(uni, const)

    def offset(self, d: TDesc, coords) -> str:
        lane, uni = self.offset_parts(d, coords)
        if uni == "0":
            return lane
        return uni if lane == "0" else self.ivar(f"{lane} + {uni}")

    def suffix(self, flat: str, m: int) -> str:
        """``flat % m``; in a plane-major functor r % m = s % m whenever m | S."""
        if flat == "r" and self.planes is not None and math.prod(self.planes[1]) % m == 0:
            return "s" if m == math.prod(self.planes[1]) else self.ivar(f"s % {m}")
        return self.ivar(f"{flat} % {m}")

    def addr(self, d: TDesc, coords) -> str:
        lane, uni = self.offset_parts(d, coords)
        p, nb = self.base(d)
        if nb and "n" in self.uniform:  # image base is uniform too (plane-major functors)
            uni = nb if uni == "0" else self.ivar(f"{nb} + {uni}")
        elif nb:
            lane = nb if lane == "0" else self.ivar(f"{nb} + {lane}")
        if uni == "0":
            return f"{p} + {lane}"
        if lane == "0":
            return f"{p} + {uni}"
        # 64-bit lane pointer (shared by every row of the producer) + per-row 32-bit
        # uniform offset: one IMAD.WIDE per gathered element
        key = ("lp", p, lane)
        lp = self.memo_get(key)
        if not lp:
            lp = self.fresh("lp")
            if lane in self.lanes:  # vector mode, lane-affine: the lane-0 pointer (loads add coef*e)
                self._emit(f"float* const {lp} = {p} + {lane};")
            else:
                self.define("float* const", lp, f"{p} + {lane}")
            self.memo_put(key, lp)
        return f"canvas::ptr_add({lp}, {uni})"

    def vec_addr(self, d: TDesc, coords):
        """Vector mode: (address, coef) — lane e reads address + coef*e — or
        (address, None) when the lanes need their own addresses (substituted)."""
        a = self.addr(d, coords)
        lane, uni = self.offset_parts(d, coords)
        _, nb = self.base(d)
        if nb and "n" in self.uniform:
            uni = nb if uni == "0" else self.ivar(f"{nb} + {uni}")
        elif nb:
            lane = nb if lane == "0" else self.ivar(f"{nb} + {lane}")
        # residue of the lane-0 element offset from the (16 B aligned) slot pointer
        self._vec_res = self._radd(self.residue(lane), self.residue(uni)) if nb or d.bstride % 4 == 0 else (1, 0)
        if lane in self.lanes:
            return a, self.lanes[lane][0]
        if self.lane_vars(a):
            return a, None
        return a, 0

    def raw_ivar(self, expr: str) -> str:
        v = self.ivar(expr)
        self.raw.add(v)
        return v

    def lin(self, x: str) -> tuple[dict, int]:
        """Affine form {var: coef}, const of a coordinate (var, int literal or affine var)."""
        x = str(x)
        if x.lstrip("-").isdigit():
            return {}, int(x)
        if x in self.lin_of:
            terms, c = self.lin_of[x]
            return dict(terms), c
        return {x: 1}, 0

    def affine(self, parts, const: int = 0) -> tuple[str, bool]:
        """Canonical var for sum(coef * part) + const, composing affine coordinates
        (so e.g. (h - k + 1) + k - 1 folds back to h).  Returns (var, raw): raw is
        False when the result is a plain in-range coordinate (no predicate needed)."""
        acc: dict = {}
        c0 = const
        for coef, x in parts:
            t, c = self.lin(x)
            c0 += coef * c
            for v, k in t.items():
                acc[v] = acc.get(v, 0) + coef * k
        acc = {v: k for v, k in acc.items() if k}
        if not acc:
            return str(c0), True
        if c0 == 0 and len(acc) == 1 and next(iter(acc.values())) == 1:
            v = next(iter(acc))
            return v, v in self.raw
        expr = " + ".join(f"{v}" if k == 1 else f"{v}*({k})" for v, k in sorted(acc.items()))
        expr = f"{expr} + ({c0})" if c0 else expr
        v = self.ivar(expr)
        self.lin_of[v] = (tuple(sorted(acc.items())), c0)
        self.raw.add(v)
        return v, True

    def load(self, d: TDesc, coords, preds: tuple = ()) -> str:
        self.loaded.setdefault((d.slot, d.bstride), d)
        # the guard only protects addresses built from raw (possibly out-of-range)
        # coordinates; an all-in-range load is safe and stays unpredicated so the
        # compiler can share it
        if any(str(c) in self.raw for c in coords):
            preds = self.guard + tuple(p for p in preds if p not in self.guard)
        if self.V > 1:
            if self.lane_pred and self.lane_pred not in preds:
                preds = preds + (self.lane_pred,)
            return self._load_vec(d, coords, preds)
        if preds:
            return self.fvar(f"({' && '.join(preds)}) ? __ldg({self.addr(d, coords)}) : 0.f")
        return self.fvar(f"__ldg({self.addr(d, coords)})")

    def _load_vec(self, d: TDesc, coords, preds) -> str:
        old_tag = self.cur_tag
        self.cur_tag = "l"
        try:
            return self._load_vec_tagged(d, coords, preds)
        finally:
            self.cur_tag = old_tag

    def _load_vec_tagged(self, d: TDesc, coords, preds) -> str:
        a, c = self.vec_addr(d, coords)
        if c == 1:
            # the row-context offset of a unit-stride quad: rows with close values
            # read the same lines (producer row ordering, ``{name}key``)
            _, up = self.offset_parts(d, coords)
            if up in self.uni_vars:
                self.row_keys.append(up)
        pe = " && ".join(preds)
        key = ("ldv", a, pe)
        got = self.memo_get(key)
        if got:
            return got
        if c == 0 and not (pe and self.lane_vars(pe)):
            v = self.fvar(f"({pe}) ? __ldg({a}) : 0.f" if pe else f"__ldg({a})")  # lane-invariant
        elif c == 1 and self.V == 4 and VEC16 and (self._vec_res[0] % 4 == 0 or VEC_RT):
            # unit-stride quad: the aligned 16 B chunk(s) holding it.  Offset m =
            # (lane-0 offset) mod 4 from a 16 B boundary is static when the residue
            # analysis knows it (m = 0: one load), else read from the address (row-
            # dependent shifts).  Lanes 0..3-m sit in the first chunk, 4-m..3 in the
            # second; a chunk is read only when one of its lanes is valid, so it lies
            # inside the tensor.  The per-lane select runs on the packed word ``bits``
            # (4 lane-valid bits | m << 4) — tagged 's', so a load / compute split
            # leaves only the chunk loads in the load half.
            static = self._vec_res[0] % 4 == 0
            m = self._vec_res[1] % 4 if static else None
            self.nld["aligned" if static and m == 0 else "shifted"] += 1
            v = self.fresh("v")
            self.vec16 = True
            pl = [self.subst(pe, e) for e in range(4)] if pe and self.lane_vars(pe) else []
            zero = "make_float4(0.f, 0.f, 0.f, 0.f)"
            q = self.fresh("q")
            self._emit(f"const float* const {q} = {a};")
            if static:
                mv = str(m)
            else:
                mv = self.fresh("m")
                self._emit(f"const int {mv} = (int)((reinterpret_cast<unsigned long long>({q}) >> 2) & 3ull);")
                # the row-context part of the offset decides m for every pixel of the
                # row (the lane part is = 0 mod 4): a producer can group rows by it
                _, uni_part = self.offset_parts(d, coords)
                self.rt_cls.append(uni_part if uni_part in self.uni_vars else None)
            if static:
                conds = []
                for ci in ([0] if m == 0 else [0, 1]):
                    lanes_ci = [e for e in range(4) if (m + e) // 4 == ci]
                    conds.append(" || ".join(f"({pl[e]})" for e in lanes_ci) if pl else pe)
            elif pl:
                conds = [" || ".join([f"({pl[0]})"] + [f"(({pl[e]}) && {mv} < {4 - e})" for e in (1, 2, 3)]),
                         f"{mv} > 0 && (" + " || ".join([f"({pl[3]})", f"(({pl[2]}) && {mv} >= 2)", f"(({pl[1]}) && {mv} >= 3)"]) + ")"]
            else:
                conds = [pe, f"{mv} > 0" + (f" && ({pe})" if pe else "")]
            for ci, cond in enumerate(conds):
                off = f" + {4 * ci - m}" if static and 4 * ci - m else ("" if static else f" - {mv}" + (" + 4" if ci else ""))
                src = f"__ldg(reinterpret_cast<const float4*>({q}{off}))"
                self._emit(f"const float4 {v}q{ci} = ({cond}) ? {src} : {zero};" if cond else f"const float4 {v}q{ci} = {src};")
            bits = None
            if pl or not static:
                bits = self.fresh("bits")
                parts = [f"(({pl[e]}) ? {1 << e} : 0)" for e in range(4)] if pl else ["15"]
                if not static:
                    parts.append(f"({mv} << 4)")
                self._emit(f"const int {bits} = {' | '.join(parts)};")
            self.cur_tag = "s"
            w = [f"{v}q0.{x}" for x in "xyzw"] + [f"{v}q1.{x}" for x in "xyzw"]
            if not static and VEC_RT == 2:
                # one branch on m for the 4 lanes (warp-uniform where the producer
                # groups rows by their shift class, tc_gemm_wgrad) instead of 12 selects
                self._emit(f"const float4 {v}w = canvas::win4({v}q0, {v}q1, {bits} >> 4);")
                w = [f"{v}w.{x}" for x in "xyzw"] * 2
            for e in range(4):
                if static:
                    sel = w[m + e]
                elif VEC_RT == 2:
                    sel = w[e]
                else:
                    mb = f"({bits} >> 4)"
                    sel = f"({mb} == 0 ? {w[e]} : {mb} == 1 ? {w[e + 1]} : {mb} == 2 ? {w[e + 2]} : {w[e + 3]})"
                self._emit(f"const float {v}_{e} = ({bits} & {1 << e}) ? {sel} : 0.f;" if pl else f"const float {v}_{e} = {sel};")
            self.cur_tag = "l"
            self.copies.add(v)
        else:
            self.nld["shifted" if c == 1 else "lanes"] += 1
            v = self.fresh("v")
            if c is not None and "(" in a:
                # one address for the lanes (predicated loads would otherwise each
                # recompute it under their own predicate)
                q = self.fresh("q")
                self._emit(f"const float* const {q} = {a};")
                a = q
            for e in range(self.V):
                ae = f"{a} + {c * e}" if c is not None and c * e else (a if c is not None else self.subst(a, e))
                pl = self.subst(pe, e) if pe else ""
                self._emit(f"const float {v}_{e} = ({pl}) ? __ldg({ae}) : 0.f;" if pl else f"const float {v}_{e} = __ldg({ae});")
            self.copies.add(v)
        self.memo_put(key, v)
        return v

    def store(self, d: TDesc, coords, val: str, beta: bool, pred: str = "") -> None:
        if pred:  # predicated scalar store (address computed unconditionally)
            a = self.addr(d, coords)
            self._emit(f"if ({pred}) *({a}) = {val};")
            return
        if self.V > 1:
            a, c = self.vec_addr(d, coords)
            if c == 0:
                raise VecUnsupported("lane-invariant store")
            if c == 1 and self.V == 4 and VEC16 and self._vec_res[0] % 4 == 0 and self._vec_res[1] % 4 == 0:
                self.vec16 = True
                vs = ", ".join(self.subst(val, e) for e in range(4))
                q = self.fresh("q")
                self._emit(f"float4* const {q} = reinterpret_cast<float4*>({a});")
                if beta:
                    self._emit(f"if (a.beta) {{ const float4 o_ = *{q}; const float4 u_ = make_float4({vs}); *{q} = make_float4(o_.x + u_.x, o_.y + u_.y, o_.z + u_.z, o_.w + u_.w); }} else *{q} = make_float4({vs});")
                else:
                    self._emit(f"*{q} = make_float4({vs});")
                return
            for e in range(self.V):
                ae = (f"{a} + {c * e}" if c * e else a) if c is not None else self.subst(a, e)
                ve = self.subst(val, e)
                self._emit(f"if (a.beta) *({ae}) += {ve}; else *({ae}) = {ve};" if beta else f"*({ae}) = {ve};")
            return
        a = self.addr(d, coords)
        if beta:
            self.emit(f"if (a.beta) *({a}) += {val}; else *({a}) = {val};")
        else:
            self.emit(f"*({a}) = {val};")

    def decompose(self, flat: str, ext) -> list[str]:
        """Row-major flat index -> coordinates (constant divisors)."""
        coords = [None] * len(ext)
        rest = flat
        for i in range(len(ext) - 1, -1, -1):
            e = ext[i]
            if i == 0:
                coords[0] = self.ivar(rest) if e > 1 else "0"
            elif e == 1:
                coords[i] = "0"
            else:
                coords[i] = self.ivar(f"{rest} % {e}")
                rest = self.ivar(f"{rest} / {e}")
        if len(ext) > 1:
            self.flat_of.setdefault(tuple(coords), (flat, tuple(ext)))
        return coords

    def flatten(self, coords, ext) -> str:
        got = self.flat_of.get(tuple(coords))
        if got is not None and got[1] == tuple(ext):
            return got[0]  # recomposing a decomposed flat index: it is that index
        expr = None
        for c, e in zip(coords, ext):
            expr = c if expr is None else f"({expr})*{e} + {c}"
        return self.ivar(expr if expr is not None else "0")


class Lowerer:
    """Builds a :class:`Plan` for one concrete graph and replacement target."""

    def __init__(self, g: ConcreteGraph, plan: Plan, use_tc: bool = True):
        self.use_tc = use_tc
        self.g = g
        self.p = plan
        self.nodes = g.nodes
        self.out = g.output
        self.kernels: list[str] = []  # functor + kernel source per kernel
        # forward materialisation: reductions, contractions, input, output (module docstring)
        # small folds (D <= FOLD_INLINE, e.g. a max over the K = 3 taps of an Unfold) are
        # evaluated inline by their consumers like a pointwise node (D loads), unless
        # replicated_pointwise finds them re-evaluated often enough to materialise
        self.fwd_mat = {0} | {v.id for v in self.nodes if v.op in ("softmax", "fc") or (v.op == "fold" and not self.inline_fold(v))} | {self.out}
        self.fwd_mat |= self.replicated_pointwise()
        # gradients materialised in the backward: every non-view node except the
        # output (its gradient is dy) — views pull through gathers
        self.grad_mat = {0} | {v.id for v in self.nodes if v.op not in VIEW_OPS and v.id != self.out and v.op != "input"}
        self.grad_mat -= self.inline_grads()
        self.fwd_desc: dict[int, TDesc] = {}
        self.count_desc: dict[int, TDesc] = {}
        self.grad_desc: dict[int, TDesc] = {}
        self.dgrad_desc: dict[int, TDesc] = {}  # FC node u -> contribution buffer for its input
        self.inline_dgrad: set = set()  # few-output FCs whose input-gradient contribution is evaluated inline
        self.dot_desc: dict[int, TDesc] = {}  # softmax node u -> row dot buffer
        self.computing_grad = None
        # FC dgrads whose epilogue applies the adjoint of their input broadcast
        # (u -> jt): the epilogue writes the broadcast's edge contributions
        # (edge_desc[(bcast, pos)]) and gradients that need no other term (grad_by_epi)
        self.epi_bc: dict = {}
        self.edge_desc: dict = {}
        self.grad_by_epi: set = set()

    @classmethod
    def bare(cls, plan: Plan, use_tc: bool = True) -> "Lowerer":
        """A Lowerer without a kernel graph: the kernel emitters (GEMM templates
        with caller-written functor bodies) for dense layers (dense_conv.py)."""
        lw = cls.__new__(cls)
        lw.use_tc, lw.g, lw.p, lw.nodes, lw.out = use_tc, None, plan, [], None
        lw.kernels = []
        lw.fwd_mat, lw.grad_mat = set(), set()
        lw.fwd_desc, lw.count_desc, lw.grad_desc, lw.dgrad_desc, lw.dot_desc = {}, {}, {}, {}, {}
        lw.inline_dgrad = set()
        lw.computing_grad = None
        lw.epi_bc, lw.edge_desc, lw.grad_by_epi = {}, {}, set()
        return lw

    # -------------------------------------------------------------- materialisation
    def inline_grads(self) -> set:
        """Pointwise / broadcast / small-fold nodes whose gradient is not
        materialised: the adjoint kernels that need dL/dv evaluate it inline (a
        pull through the consumers' adjoints), saving a launch and an HBM round
        trip.  ge[i] = how many times one element of dL/di is evaluated per
        element of the nearest materialised gradient below it: 1 when
        materialised, else sum over i's input edges of (edge fan-in factor:
        Unfold K, broadcast-LHS replicas M, fold window D) x ge[input].  A
        gradient is inlined while ge stays below REPLICATE_MIN (same rule as the
        forward's replicated_pointwise)."""
        if not GRAD_INLINE:
            return set()
        ge = {0: 1}
        inl = set()
        for nd in self.nodes[1:]:
            v = nd.id

            def fac(pos):
                if nd.op == "bcast" and pos == 0:
                    return nd.attr["M"]
                if nd.op == "unfold":
                    return nd.attr["K"]
                if nd.op == "fold":
                    return nd.attr["D"]
                return 1

            e = sum(fac(pos) * ge.get(i, 1) for pos, i in enumerate(nd.ins)) if nd.ins else 1
            cand = (nd.op in ("ew", "bcast") or self.inline_fold(nd)) and v != self.out and not self._grad_is_fc_alias(v)
            if nd.op in VIEW_OPS or (cand and e < REPLICATE_MIN):
                ge[v] = e
                if cand:
                    inl.add(v)
            else:
                ge[v] = 1
        return inl

    @staticmethod
    def inline_fold(nd) -> bool:
        return nd.op == "fold" and nd.attr["D"] <= FOLD_INLINE

    def replicated_pointwise(self) -> set:
        """Pointwise nodes worth one extra HBM round trip: those whose inline
        evaluation would be repeated >= REPLICATE_MIN times per consumer output
        (LHS of a broadcast with ratio M, input of an Unfold, a softmax's three
        passes, a small FC's per-output-channel dot) and that cost >= 2 loads to
        recompute.  Walk consumers first so replication compounds through chains."""
        chosen: set = set()
        evals: dict = {}

        def mat(v):
            return v in self.fwd_mat or v in chosen

        def factor(u, pos):
            nu = self.nodes[u]
            if nu.op == "bcast":
                return nu.attr["M"] if pos == 0 else 1
            if nu.op == "unfold":
                return nu.attr["K"]
            if nu.op == "softmax":
                return 3
            if nu.op == "fc":
                o, k = self.g.fc_shape(u)
                return o if min(o, k) <= SMALL_FC else tc_tile(o)[1]
            return 1

        def loads(v, seen=None):
            seen = set() if seen is None else seen
            if v in seen:
                return 0
            seen.add(v)
            if mat(v):
                return 1
            k = self.nodes[v].attr["D"] if self.nodes[v].op == "fold" else 1
            return k * sum(loads(i, seen) for i in self.nodes[v].ins)

        for v in range(len(self.nodes) - 1, 0, -1):
            nd = self.nodes[v]
            evals[v] = sum(factor(u, pos) * (1 if mat(u) else evals.get(u, 1)) for u, pos in nd.consumers) or 1
            if (nd.op in ("ew", "bcast") or self.inline_fold(nd)) and v != self.out and evals[v] >= REPLICATE_MIN and loads(v) >= 2:
                chosen.add(v)
                evals[v] = 1
        return chosen

    # -------------------------------------------------------------- descriptors
    @staticmethod
    def _contig(ext) -> tuple:
        st, acc = [], 1
        for e in reversed(ext):
            st.append(acc)
            acc *= e
        return tuple(reversed(st))

    def _new_saved(self, ext) -> TDesc:
        n = math.prod(ext)
        self.p.saved.append(SizeRule(4 * n, 1, 0))
        return TDesc(self.p.slot_saved(len(self.p.saved) - 1), n, self._contig(ext), tuple(ext))

    def _new_ws(self, ext) -> tuple[int, TDesc]:
        n = math.prod(ext)
        self.p.ws.append(SizeRule(4 * n, 1, 0))
        k = len(self.p.ws) - 1
        return k, TDesc(-1 - k, n, self._contig(ext), tuple(ext))  # slot fixed up in finish()

    def x_desc(self) -> TDesc:
        p, n0 = self.p, self.nodes[0]
        c, h, w = n0.ext
        s = p.stride
        ctot = p.c_in
        return TDesc(SLOT_X, ctot * p.h_in * p.w_in, (p.h_in * p.w_in, s * p.w_in, s), (c, h, w))

    def dx_desc(self) -> TDesc:
        d = self.x_desc()
        return TDesc(SLOT_DX, d.bstride, d.strides, d.dims)

    def y_desc(self, slot=SLOT_Y) -> TDesc:
        c, h, w = self.nodes[self.out].ext
        ctot = self.p.c_out
        return TDesc(slot, ctot * h * w, (h * w, w, 1), (c, h, w))

    # -------------------------------------------------------------- forward values
    def val(self, f: Fn, v: int, coords: tuple, preds: tuple = ()) -> str:
        """Forward value of node v at ``coords``.  ``preds`` are the in-range
        predicates of the Shift/Unfold stages between the requesting load and v
        (App. A.3: every stage applies its own); they fold into a predicated
        load at a materialised tensor, or a select around a computed node."""
        key = ("val", v, coords, preds, f.guard)
        got = f.memo_get(key)
        if got:
            return got
        nd = self.nodes[v]
        if v in self.fwd_desc and v != getattr(f, "computing", None):
            r = f.load(self.fwd_desc[v], coords, preds)
        elif nd.op in VIEW_OPS:
            r = self.view(f, v, coords, preds)
        elif preds:
            inner = self.guarded(f, preds, lambda: self.compute(f, v, coords))
            r = f.fvar(f"({' && '.join(preds)}) ? {inner} : 0.f")
        else:
            r = self.compute(f, v, coords)
        f.memo_put(key, r)
        return r

    @staticmethod
    def guarded(f: Fn, preds: tuple, fn):
        old = f.guard
        f.guard = old + tuple(p for p in preds if p not in old)
        try:
            return fn()
        finally:
            f.guard = old

    def view(self, f: Fn, v: int, coords: tuple, preds: tuple) -> str:
        nd = self.nodes[v]
        op, at = nd.op, nd.attr
        if op == "group":
            d, b = at["dim"], at["B"]
            merged = f.ivar(f"{coords[d]}*{b} + {coords[d + 1]}" if coords[d] != "0" else coords[d + 1])
            return self.val(f, nd.ins[0], coords[:d] + (merged,) + coords[d + 2 :], preds)
        if op == "shift":
            ax, off = at["ax"], at["off"]
            e = nd.ext[ax]
            src, raw = f.affine([(1, coords[ax])], off)
            pr = preds + (f"((unsigned){src} < {e}u)",) if raw else preds
            return self.val(f, nd.ins[0], coords[:ax] + (src,) + coords[ax + 1 :], pr)
        if op == "unfold":
            k_at, K, ax_out = at["at"], at["K"], at["ax_out"]
            e = nd.ext[ax_out]
            src, raw = f.affine([(1, coords[ax_out]), (1, coords[k_at])], -(K // 2))
            c2 = list(coords)
            c2[ax_out] = src
            del c2[k_at]
            pr = preds + (f"((unsigned){src} < {e}u)",) if raw else preds
            return self.val(f, nd.ins[0], tuple(c2), pr)
        raise LoweringError(op)

    def compute(self, f: Fn, v: int, coords: tuple) -> str:
        nd = self.nodes[v]
        op, at = nd.op, nd.attr
        if op in VIEW_OPS:
            return self.view(f, v, coords, ())
        if op == "ew":
            x = self.val(f, nd.ins[0], coords)
            return f.fvar(_EW_FWD[at["fn"]].format(x))
        if op == "bcast":
            lhs = self.val(f, nd.ins[0], self.lhs_coords(f, nd, coords))
            rhs = self.val(f, nd.ins[1], coords)
            return f.fvar(_BC_FWD[at["op"]].format(lhs, rhs))
        if op == "fold" and self.inline_fold(nd):
            # same order and tie rule as body_fold: acc over j = 0..D-1, first max kept
            xs = self.fold_terms(f, v, coords)
            if at["mode"] == "avg":
                return f.fvar(f"({' + '.join(xs)}) / {float(at['D'])!r}f")
            acc = f.fvar(f"({xs[0]} > -INFINITY) ? {xs[0]} : -INFINITY")
            for x in xs[1:]:
                acc = f.fvar(f"({x} > {acc}) ? {x} : {acc}")
            return acc
        raise LoweringError(f"node {v} ({op}) must be materialised before it is read")

    def fold_terms(self, f: Fn, v: int, coords: tuple) -> list:
        """Input values of fold node v's window at output ``coords`` (j = 0..D-1)."""
        nd = self.nodes[v]
        dim, D = nd.attr["dim"], nd.attr["D"]
        return [self.val(f, nd.ins[0], coords[:dim] + (str(j),) + coords[dim:]) for j in range(D)]

    def lhs_coords(self, f: Fn, nd, coords) -> tuple:
        at = nd.attr
        cs, nl, nr, L = at["cs"], at["nl"], at["nr"], at["L"]
        core = coords[cs : cs + nr]
        if nl == 0:
            lc = ()
        elif at["M"] == 1 and tuple(at["lcore"]) == tuple(at["rcore"]):
            lc = core
        else:
            r = f.flatten(core, at["rcore"])
            l = f.ivar(f"{r} % {L}") if at["M"] > 1 else r
            lc = tuple(f.decompose(l, at["lcore"]))
        return coords[:cs] + lc + coords[cs + nr :]

    # -------------------------------------------------------------- gradients
    def grad(self, f: Fn, v: int, coords: tuple, preds: tuple = ()) -> str:
        key = ("grad", v, coords, preds, f.guard)
        got = f.memo_get(key)
        if got:
            return got
        if v == self.out:
            r = f.load(self.dy_desc, coords, preds)
        elif v in self.grad_desc and v != self.computing_grad:
            r = f.load(self.grad_desc[v], coords, preds)
        elif preds:
            g = self.guarded(f, preds, lambda: self.grad_sum(f, v, coords))
            r = f.fvar(f"({' && '.join(preds)}) ? {g} : 0.f")
        else:
            r = self.grad_sum(f, v, coords)
        f.memo_put(key, r)
        return r

    def grad_sum(self, f: Fn, v: int, coords: tuple) -> str:
        terms = [self.contrib(f, u, pos, v, coords) for u, pos in self.nodes[v].consumers]
        terms = [t for t in terms if t != "0.f"]
        if not terms:
            return "0.f"
        return f.fvar(" + ".join(terms)) if len(terms) > 1 else terms[0]

    def contrib(self, f: Fn, u: int, pos: int, v: int, coords: tuple) -> str:
        """Contribution of edge v -(pos)-> u to dL/dv at ``coords`` (pull form)."""
        nu = self.nodes[u]
        op, at = nu.op, nu.attr
        if op == "group":
            d, b = at["dim"], at["B"]
            c = coords[d]
            hi, lo = f.ivar(f"{c} / {b}"), f.ivar(f"{c} % {b}")
            return self.grad(f, u, coords[:d] + (hi, lo) + coords[d + 1 :])
        if op == "shift":
            ax, off = at["ax"], at["off"]
            e = nu.ext[ax]
            src, raw = f.affine([(1, coords[ax])], -off)
            return self.grad(f, u, coords[:ax] + (src,) + coords[ax + 1 :], (f"((unsigned){src} < {e}u)",) if raw else ())
        if op == "unfold":
            # col2im as a gather: dI[h] = sum_k dU[k, h - k + K//2] (valid terms only)
            k_at, K, ax_in = at["at"], at["K"], at["ax_in"]
            e = nu.ext[at["ax_out"]]
            terms = []
            for k in range(K):
                src, raw = f.affine([(1, coords[ax_in])], -(k - K // 2))
                c2 = list(coords)
                c2[ax_in] = src
                c2.insert(k_at, str(k))
                terms.append(self.grad(f, u, tuple(c2), (f"((unsigned){src} < {e}u)",) if raw else ()))
            return f.fvar(" + ".join(terms))
        if op == "ew":
            g = self.grad(f, u, coords)
            x = self.val(f, v, coords)
            fn = at["fn"]
            if fn == "relu":
                return f.fvar(f"{x} > 0.f ? {g} : 0.f")
            if fn == "abs":
                return f.fvar(f"{x} > 0.f ? {g} : ({x} < 0.f ? -{g} : 0.f)")
            if fn == "sin":
                return f.fvar(f"{g} * cosf({x})")
            if fn == "exp":
                return f.fvar(f"{g} * expf({x})")
            if fn == "neg":
                return f.fvar(f"-{g}")
        if op == "fold":
            dim, D = at["dim"], at["D"]
            uc = coords[:dim] + coords[dim + 1 :]
            g = self.grad(f, u, uc)
            if at["mode"] == "avg":
                return f.fvar(f"{g} / {float(D)!r}f")
            m = self.val(f, u, uc)
            if u in self.count_desc:
                cnt = f.load(self.count_desc[u], uc)
            else:  # inlined fold: count the ties of its window here
                cnt = f.fvar(" + ".join(f"({x} == {m} ? 1.f : 0.f)" for x in self.fold_terms(f, u, uc)))
            x = self.val(f, v, coords)
            return f.fvar(f"{x} == {m} ? {g} / {cnt} : 0.f")
        if op == "softmax":
            y = self.val(f, u, coords)
            g = self.grad(f, u, coords)
            d = self.dot_desc[u]
            rc = self.softmax_row_coords(nu, coords)
            dot = f.load(d, rc)
            return f.fvar(f"{y} * ({g} - {dot})")
        if op == "fc":
            if u in self.inline_dgrad:
                # few-output FC: its input-gradient contribution sum_o W[o, i] g_u[o, s]
                # is an O-term dot evaluated where the gradient sum needs it
                O, K = self.g.fc_shape(u)
                wslot, _ = self.fc_weight_slot(u)
                nv = self.nodes[v]
                i = f.flatten(coords[: nv.nch], nv.ch_ext)
                sp = coords[nv.nch :]
                terms = [f.fvar(f"__ldg({f.ptr(wslot)} + {o * K} + {i}) * {self.grad(f, u, (str(o),) + tuple(sp))}") for o in range(O)]
                return f.fvar(" + ".join(terms))
            return f.load(self.dgrad_desc[u], coords)
        if op == "bcast":
            return self.bcast_contrib(f, nu, pos, v, coords)
        raise LoweringError(f"no adjoint for {op}")

    def bcast_contrib(self, f: Fn, nu, pos: int, v: int, coords: tuple) -> str:
        at = nu.attr
        u = nu.id
        if (u, pos) in self.edge_desc:  # written by the epilogue of the consuming FC's dgrad
            return f.load(self.edge_desc[(u, pos)], coords)
        lhs_n, rhs_n = nu.ins
        bop = at["op"]
        total = []
        if pos == 1:  # v is the RHS: elementwise
            g = self.grad(f, u, coords)
            l = self.val(f, lhs_n, self.lhs_coords(f, nu, coords))
            r = self.val(f, rhs_n, coords)
            total.append(f.fvar(_bc_d_rhs(bop, g, l, r)))
        else:  # v is the LHS: sum over the M replicas r = m*L + l
            cs, nl, nr, L, M = at["cs"], at["nl"], at["nr"], at["L"], at["M"]
            lcore = coords[cs : cs + nl]
            lflat = f.flatten(lcore, at["lcore"]) if nl else "0"
            l = self.val(f, lhs_n, coords) if bop in ("mul", "min", "max") else None

            def term(mexpr: str) -> str:
                rr = f.ivar(f"{mexpr}*{L} + {lflat}" if mexpr != "0" else lflat)
                rc = coords[:cs] + tuple(f.decompose(rr, at["rcore"])) + coords[cs + nl :]
                g = self.grad(f, u, rc)
                r = self.val(f, rhs_n, rc) if bop in ("mul", "min", "max") else None
                return f.fvar(_bc_d_lhs(bop, g, l, r))

            if M == 1:
                total.append(term("0"))
            elif M <= 4:
                total.append(f.fvar(" + ".join(term(str(m)) for m in range(M))))
            else:
                acc = f.fresh("s")
                f.emit(f"float {acc} = 0.f;")
                mv = f.fresh("m")
                f.loop(mv, M)
                t = term(mv)
                f.emit(f"{acc} += {t};")
                f.close()
                total.append(acc)
        return total[0] if len(total) == 1 else f.fvar(" + ".join(total))

    # -------------------------------------------------------------- softmax rows
    @staticmethod
    def softmax_geom(nd) -> tuple:
        s, e = nd.attr["start"], nd.attr["end"]
        pre = nd.ext[:s]
        span = nd.ext[s : e + 1]
        post = nd.ext[e + 1 :]
        return pre, span, post

    def softmax_row_coords(self, nd, coords) -> tuple:
        s, e = nd.attr["start"], nd.attr["end"]
        return coords[:s] + coords[e + 1 :]

    # -------------------------------------------------------------- kernels
    def add_kernel(self, name: str, functor: str, launcher: str) -> int:
        self.kernels.append(functor + launcher)
        self.p.kernel_names.append(name)
        return len(self.p.kernel_names) - 1

    def functor_pointwise(self, name: str, per_image: int, body_fn, planes=None, V: int = 1) -> tuple[str, list]:
        """Functor for ``canvas::pointwise``: one output element (or row) per call;
        with ``planes`` = (channel ext, spatial ext), for ``canvas::pointwise_planes``.
        V = 4: ``run4`` evaluates the 4 consecutive elements r .. r+3 (r a multiple
        of 4) for ``canvas::pointwise4`` / ``pointwise_planes4`` (raises
        VecUnsupported when the body cannot be emitted in that form)."""
        f = Fn(self)
        f.pre = []
        f.computing = None
        f.planes = planes
        if V > 1:
            f.V = V
            f.lanes = {"r": (1, V, 0)} if planes is None else {"r": (1, V, 0), "s": (1, V, 0)}
        body_fn(f)
        self._fn_vec16 = f.vec16
        self._fn_nld = dict(f.nld)
        fn = "run4" if V > 1 else "run"
        if planes is None:
            src = [f"struct {name}_F {{", f"  static constexpr long long PER = {per_image}LL;", f"  static __device__ __forceinline__ void {fn}(const CanvasArgs& a, const long long n, const int r) {{"]
        else:
            Q, S = math.prod(planes[0]), math.prod(planes[1])
            src = [f"struct {name}_F {{", f"  static constexpr int Q = {Q}, S = {S};", f"  static __device__ __forceinline__ void {fn}(const CanvasArgs& a, const long long n, const int q, const int s) {{", f"    const int r = q * {S} + s;"]
        src += ["    " + s for s in f.pre]
        src += self.loads_first(f) if LOADS_FIRST else f.lines
        src += ["  }", "};"]
        return "\n".join(src) + "\n", f.local_slots

    @staticmethod
    def loads_first(f: Fn) -> list:
        """Straight-line bodies (no loops / braces): index math and gathers hoisted
        above the float arithmetic, in order, wherever their operands allow — so
        every gather of the element is issued before the first one is consumed."""
        lines, tags = f.lines, f.ltags
        if any("{" in ln or "}" in ln or ln.lstrip().startswith("#") for ln in lines):
            return lines
        asm = ASM_LOADS == "1" or (ASM_LOADS == "planes" and f.planes is not None)
        early, late, late_names = [], [], set()
        for ln, t in zip(lines, tags):
            m = re.match(r"\s*(?:const )?(?:int|float|float4|float\*|const float\*)\s*(?:const )?(\w+) = (.*);$", ln)
            hoist = t in "il" or (asm and "__ldg(" in ln)  # gathers emitted outside a load tag
            if m and hoist and not (set(_IDENT.findall(m.group(2))) & late_names):
                early.append(ln)
                continue
            late.append(ln)
            if m:
                late_names.add(m.group(1))
        if asm and sum("__ldg(" in ln for ln in early) >= 6:
            # keep the hoisted order: volatile PTX loads are not re-sequenced by ptxas,
            # so every gather of the element is in flight before the first is consumed
            out = []
            for ln in early:
                m = re.match(r"(\s*const float \w+ = )\((.*)\) \? __ldg\((.*)\) : 0\.f;$", ln)
                if m:
                    ln = f"{m.group(1)}canvas::ldg_vp({m.group(3)}, {m.group(2)});"
                elif re.match(r"\s*const float \w+ = __ldg\(", ln):
                    ln = ln.replace("__ldg(", "canvas::ldg_v(", 1)
                out.append(ln)
            early = out
        return early + late

    @staticmethod
    def plane_split(ext, sp_ext, per_image):
        """(channel ext, spatial ext) when a plane-major launch applies, else None."""
        if not PLANES_MIN_S or ext is None:
            return None
        ext, nsp = tuple(ext), len(sp_ext)
        S = math.prod(ext[len(ext) - nsp:]) if nsp else 1
        if nsp == 0 or S < PLANES_MIN_S or math.prod(ext) != per_image:
            return None
        return ext[: len(ext) - nsp], ext[len(ext) - nsp:]

    @staticmethod
    def ks_split(per_image: int, K: int) -> int:
        """Lanes per output element for a long per-element reduction (K terms): the largest
        power of 2 <= 32 keeping the batch-256 thread count within 2 full waves and >= 16
        terms per lane; 1 = no split."""
        if not FC_SMALL_KS or K < 64:
            return 1
        ks = 1
        while ks < 32 and per_image * 256 * ks * 2 <= SMS * 2048 * 2 and K // (ks * 2) >= 16:
            ks *= 2
        return ks

    def launch_ks(self, name, per_image, part_fn, put_fn, nacc, ks, phase, beta, what, nbytes, flops):
        """``canvas::pointwise_ks``: KS consecutive lanes per output element; ``part``
        accumulates the lane's share into acc[0 .. nacc), the template reduces over the KS
        lanes (fixed xor tree), ``put`` stores from the first lane."""
        f = Fn(self)
        f.pre = []
        f.computing = None
        part_fn(f)
        g = Fn(self)
        g.pre = []
        g.computing = None
        g.local_slots = f.local_slots
        put_fn(g)
        src = [f"struct {name}_F {{", f"  static constexpr long long PER = {per_image}LL;", f"  static constexpr int NACC = {nacc};",
               f"  static __device__ __forceinline__ void part(const CanvasArgs& a, const long long n, const int r, const int part, float* acc) {{"]
        src += ["    " + x for x in f.pre] + f.lines + ["  }"]
        src += ["  static __device__ __forceinline__ void put(const CanvasArgs& a, const long long n, const int r, const float* acc) {"]
        src += ["    " + x for x in g.pre] + g.lines + ["  }", "};"]
        functor = "\n".join(src) + "\n"
        launcher = f'extern "C" __global__ void __launch_bounds__({POINTWISE_BLOCK}) {name}(const CanvasArgs a) {{ canvas::pointwise_ks<{name}_F, {ks}>(a); }}\n'
        k = self.add_kernel(name, functor, launcher)
        grid = (GridRule(per_image * ks, 0, POINTWISE_BLOCK, POINTWISE_CAP), GridRule(0, 1, 1), GridRule(0, 1, 1))
        self.p.launches.append(Launch("kernel", phase, name, k, POINTWISE_BLOCK, grid, tuple(f.local_slots), beta, what=what, bytes_per_image=nbytes, flops_per_image=flops))

    def launch_pointwise(self, name, per_image, body_fn, phase, beta=BETA_NONE, what="", nbytes=0, flops=0, inner=1, node=None, align16=False, vec_fill=2048):
        """``inner``: extent of the innermost output dim (per-thread vector width must divide it).
        ``node``: the output node whose elements the threads map to; with H*W >= PLANES_MIN_S
        the launch is plane-major (block-uniform channel plane, threads along pixels)."""
        planes = self.plane_split(node.ext, node.sp_ext, per_image) if node is not None else None
        planes0 = planes
        functor, slots = self.functor_pointwise(name, per_image, body_fn, planes)
        guarded = planes is not None and "? __ldg(" in functor
        if guarded and not PLANES_GUARDED:
            # guarded (Shift / Unfold) gathers: with block-uniform channel math the
            # compiler turns the guards into branches around each load and the
            # gathers serialise (measured 0.63 -> 0.75 ms on seed-7 #1 layer1 grad n7),
            # so these keep the flat grid-stride mapping with predicated loads
            planes = None
            functor, slots = self.functor_pointwise(name, per_image, body_fn, None)
        # 4 consecutive elements per thread (shared index math, one address per
        # lane-affine gather) when the elements per image / plane divide by 4
        vec = None
        # (and enough quads to fill the GPU at the bench batch: per-pixel kernels with
        # a long inner loop — few-output FCs, their adjoints — keep one element per
        # thread at 14x14 and below, measured 45 vs 78 us per launch)
        if VEC_POINTWISE and (per_image if planes is None else math.prod(planes[1])) % 4 == 0 and per_image * 256 // 4 >= SMS * vec_fill:
            try:
                vec = self.functor_pointwise(name, per_image, body_fn, planes, V=4)
                # gathers mostly at sub-16 B shifts (col2im over a 9C gradient): the
                # quad form costs occupancy without saving L1 wavefronts (measured
                # 0.52 vs 0.57 ms on seed-7 #1 layer1 grad n1) — keep one element per thread
                if self._fn_nld["shifted"] > self._fn_nld["aligned"] and not VEC_SHIFTED:
                    vec = None
            except VecUnsupported:
                vec = None
        vec16 = False
        if vec is not None:
            functor, slots = vec
            vec16 = self._fn_vec16
        elif guarded and planes is None:
            # one element per thread with guarded gathers: plane-major after all (the
            # branchy guards cost less than per-thread channel math here: measured
            # 0.49 vs 0.52 ms on seed-7 #1 layer1 grad n1; quads stay flat, above)
            planes = planes0
            functor, slots = self.functor_pointwise(name, per_image, body_fn, planes)
        if planes is None:
            v = POINTWISE_VEC
            block = POINTWISE_BLOCK
            if vec is not None:
                launcher = f'extern "C" __global__ void __launch_bounds__({POINTWISE_BLOCK}) {name}(const CanvasArgs a) {{ canvas::pointwise4<{name}_F>(a); }}\n'
                grid = (GridRule(per_image, 0, POINTWISE_BLOCK * 4, POINTWISE_CAP), GridRule(0, 1, 1), GridRule(0, 1, 1))
            else:
                launcher = f'extern "C" __global__ void __launch_bounds__({POINTWISE_BLOCK}) {name}(const CanvasArgs a) {{ canvas::pointwise<{name}_F, {v}>(a); }}\n'
                grid = (GridRule(per_image, 0, POINTWISE_BLOCK * v, POINTWISE_CAP), GridRule(0, 1, 1), GridRule(0, 1, 1))
        else:
            Q, S = math.prod(planes[0]), math.prod(planes[1])
            Sv = S // 4 if vec is not None else S
            chunks = -(-Sv // POINTWISE_BLOCK)
            block = -(-(-(-Sv // chunks)) // 32) * 32
            tmpl = "pointwise_planes4" if vec is not None else "pointwise_planes"
            launcher = f'extern "C" __global__ void __launch_bounds__({block}) {name}(const CanvasArgs a) {{ canvas::{tmpl}<{name}_F>(a); }}\n'
            grid = (GridRule(0, chunks, 1), GridRule(Q, 0, 1, min(65535, max(1, PLANES_CTAS // chunks))), GridRule(0, 1, 1))
        k = self.add_kernel(name, functor, launcher)
        self.p.launches.append(Launch("kernel", phase, name, k, block, grid, tuple(slots), beta, what=what, bytes_per_image=nbytes, flops_per_image=flops, align16=vec16 or align16))

    # ---- forward
    def fwd_targets(self, v: int) -> list:
        """[(TDesc, beta?)] every store of node v's forward value goes to."""
        if v == self.out:
            t = [(self.y_desc(), self.p.mode == "sum")]
            if self.out in self.fwd_desc:  # also needed by its own adjoint
                t.append((self.fwd_desc[v], False))
            return t
        return [(self.fwd_desc[v], False)]

    def lower_forward(self) -> None:
        g = self.g
        out = self.nodes[self.out]
        # descriptors of materialised forward values (reads)
        self.fwd_desc[0] = self.x_desc()
        for v in sorted(self.fwd_mat - {0}):
            nd = self.nodes[v]
            if v == self.out and not (nd.op == "softmax" or (nd.op == "fold" and nd.attr["mode"] == "max")):
                continue  # output value never read back
            self.fwd_desc[v] = self._new_saved(nd.ext)
        for v in sorted(self.fwd_mat - {0}):
            nd = self.nodes[v]
            if nd.op == "fold" and nd.attr["mode"] == "max":
                self.count_desc[v] = self._new_saved(nd.ext)
        beta_y = BETA_AFTER_FIRST if self.p.mode == "sum" else BETA_NONE
        for v in sorted(self.fwd_mat - {0}):
            nd = self.nodes[v]
            beta = beta_y if v == self.out else BETA_NONE
            name = f"k{len(self.p.kernel_names)}_fwd_{nd.op}{v}"
            tg = self.fwd_targets(v)
            io = 4 * (nd.numel + self._input_numel(nd))
            if nd.op == "fold":
                self.launch_pointwise(name, nd.numel, lambda f, v=v, tg=tg: self.body_fold(f, v, tg), 0, beta, f"fold {nd.attr['mode']} -> n{v}", io, 0, inner=nd.ext[-1] if nd.ext else 1, node=nd)
            elif nd.op == "softmax":
                pre, span, post = self.softmax_geom(nd)
                rows = math.prod(pre) * math.prod(post)
                rext = pre + post
                sl = self.row_split(rows, math.prod(span))
                if sl > 1:
                    self.launch_softmax_split(name, v, tg, sl, beta, io)
                else:
                    self.launch_pointwise(name, rows, lambda f, v=v, tg=tg: self.body_softmax(f, v, tg), 0, beta, f"softmax -> n{v}", io, 0, inner=rext[-1] if rext else 1)
            elif nd.op == "fc":
                self.lower_fc_fwd(name, v, tg, beta)
            else:
                self.launch_pointwise(name, nd.numel, lambda f, v=v, tg=tg: self.body_map(f, v, tg), 0, beta, f"pointwise -> n{v}", io, 0, inner=nd.ext[-1] if nd.ext else 1, node=nd)

    def _input_numel(self, nd) -> int:
        """Compulsory reads: materialised tensors the node's expression touches (once each)."""
        seen, stack, tot = set(), list(nd.ins), 0
        while stack:
            v = stack.pop()
            if v in seen:
                continue
            seen.add(v)
            if v in self.fwd_mat:
                tot += self.nodes[v].numel
            else:
                stack.extend(self.nodes[v].ins)
        return tot

    def coords_of(self, f: Fn, nd) -> tuple:
        if f.planes is not None and tuple(nd.ext) == f.planes[0] + f.planes[1]:
            qc = f.decompose("q", f.planes[0]) if f.planes[0] else []
            sc = f.decompose("s", f.planes[1])
            c = tuple(qc) + tuple(sc)
            if len(c) > 1:
                f.flat_of.setdefault(c, ("r", tuple(nd.ext)))
            return c
        return tuple(f.decompose("r", nd.ext))

    def body_map(self, f: Fn, v: int, targets) -> None:
        nd = self.nodes[v]
        f.computing = v
        c = self.coords_of(f, nd)
        x = self.compute(f, v, c)
        for d, beta in targets:
            f.store(d, c, x, beta)

    def body_fold(self, f: Fn, v: int, targets) -> None:
        nd = self.nodes[v]
        dim, D, mode = nd.attr["dim"], nd.attr["D"], nd.attr["mode"]
        c = self.coords_of(f, nd)
        acc = f.fresh("acc")
        if mode == "avg":
            f.emit(f"float {acc} = 0.f;")
        else:
            cnt = f.fresh("cnt")
            f.emit(f"float {acc} = -INFINITY; float {cnt} = 0.f;")
        j = f.fresh("j")
        f.loop(j, D)
        x = self.val(f, nd.ins[0], c[:dim] + (j,) + c[dim:])
        if mode == "avg":
            f.emit(f"{acc} += {x};")
        else:
            f.emit(f"if ({x} > {acc}) {{ {acc} = {x}; {cnt} = 1.f; }} else if ({x} == {acc}) {{ {cnt} += 1.f; }}")
        f.close()
        res = f.fvar(f"{acc} / {float(D)!r}f") if mode == "avg" else acc
        for d, beta in targets:
            f.store(d, c, res, beta)
        if mode == "max":
            f.store(self.count_desc[v], c, cnt, False)

    def body_softmax(self, f: Fn, v: int, targets) -> None:
        nd = self.nodes[v]
        pre, span, post = self.softmax_geom(nd)
        rc = f.decompose("r", pre + post)
        pc, qc = tuple(rc[: len(pre)]), tuple(rc[len(pre) :])
        S = math.prod(span)
        mx, sm = f.fresh("mx"), f.fresh("sm")
        f.emit(f"float {mx} = -INFINITY, {sm} = 0.f;")

        def loop(stmt_fn):
            j = f.fresh("j")
            f.loop(j, S)
            sc = tuple(f.decompose(j, span))
            c = pc + sc + qc
            x = self.val(f, nd.ins[0], c)
            stmt_fn(c, x)
            f.close()

        if f.V * S > SOFTMAX_REG_SPAN and f.V > 1:
            raise VecUnsupported("softmax rows of 4 lanes do not fit in registers")
        if S <= SOFTMAX_REG_SPAN:
            # short rows: evaluate the input once into registers (fully unrolled), so
            # the row is read from memory once instead of three times
            xs = f.fresh("xs")
            f.emit(f"float {xs}[{S}];")

            def uloop(stmt_fn):
                j = f.fresh("j")
                f.emit("#pragma unroll")
                f.open(f"for (int {j} = 0; {j} < {S}; ++{j})")
                stmt_fn(j)
                f.close()

            def first(j):
                c = pc + tuple(f.decompose(j, span)) + qc
                f.emit(f"{xs}[{j}] = {self.val(f, nd.ins[0], c)};")
                f.emit(f"{mx} = fmaxf({mx}, {xs}[{j}]);")

            uloop(first)
            uloop(lambda j: f.emit(f"{sm} += expf({xs}[{j}] - {mx});"))

            def write_r(j):
                c = pc + tuple(f.decompose(j, span)) + qc
                y = f.fvar(f"expf({xs}[{j}] - {mx}) / {sm}")
                for d, beta in targets:
                    f.store(d, c, y, beta)

            uloop(write_r)
            return
        loop(lambda c, x: f.emit(f"{mx} = fmaxf({mx}, {x});"))
        loop(lambda c, x: f.emit(f"{sm} += expf({x} - {mx});"))

        def write(c, x):
            y = f.fvar(f"expf({x} - {mx}) / {sm}")
            for d, beta in targets:
                f.store(d, c, y, beta)

        loop(write)

    @staticmethod
    def row_split(rows: int, span: int) -> int:
        """Threads per softmax row: enough rows x slices to fill the GPU at batch 256."""
        want = -(-(SMS * 2048) // (256 * rows))
        sl = 1
        while sl < want and sl < 32 and sl * 2 <= span:
            sl *= 2
        return sl

    def _row_functor(self, name: str, nd, methods) -> tuple[str, list]:
        """Functor with ROWS/SPAN and one static method per (signature, body_fn)."""
        pre, span, post = self.softmax_geom(nd)
        slots: list = []
        lines = [f"struct {name}_F {{", f"  static constexpr long long ROWS = {math.prod(pre) * math.prod(post)}LL;", f"  static constexpr int SPAN = {math.prod(span)};"]
        for sig, body in methods:
            f = Fn(self)
            f.pre = []
            f.computing = None
            f.local_slots = slots
            rc = f.decompose("r", pre + post)
            pc, qc = tuple(rc[: len(pre)]), tuple(rc[len(pre) :])
            sc = tuple(f.decompose("j", span)) if "int j" in sig else ()
            ret = body(f, pc + sc + qc, pc + qc)
            lines.append(f"  static __device__ __forceinline__ {sig} {{")
            lines += ["    " + x for x in f.pre] + f.lines
            if ret is not None:
                lines.append(f"    return {ret};")
            lines.append("  }")
        lines.append("};")
        return "\n".join(lines) + "\n", slots

    def launch_softmax_split(self, name, v, targets, sl, beta, io) -> None:
        nd = self.nodes[v]

        def out(f, c, rowc):
            for d, b in targets:
                f.store(d, c, "y", b)

        functor, slots = self._row_functor(name, nd, [
            ("float in(const CanvasArgs& a, const long long n, const int r, const int j)", lambda f, c, rowc: self.val(f, nd.ins[0], c)),
            ("void out(const CanvasArgs& a, const long long n, const int r, const int j, const float y)", out),
        ])
        launcher = f'extern "C" __global__ void __launch_bounds__(256) {name}(const CanvasArgs a) {{ canvas::softmax_rows<{name}_F, {sl}>(a); }}\n'
        k = self.add_kernel(name, functor, launcher)
        rows = math.prod(self.softmax_geom(nd)[0]) * math.prod(self.softmax_geom(nd)[2])
        grid = (GridRule(rows, 0, 256 // sl, POINTWISE_CAP), GridRule(0, 1, 1), GridRule(0, 1, 1))
        self.p.launches.append(Launch("kernel", 0, name, k, 256, grid, tuple(slots), beta, what=f"softmax -> n{v} ({sl} threads/row)", bytes_per_image=io))

    # ---- FC
    def fc_weight_slot(self, u: int) -> tuple[int, int]:
        i = self.nodes[u].attr["fc_index"]
        return self.p.slot_w(i), self.p.slot_dw(i)

    def lower_fc_fwd(self, name, u, targets, beta) -> None:
        nu = self.nodes[u]
        v = nu.ins[0]
        nv = self.nodes[v]
        O, K = self.g.fc_shape(u)
        S = math.prod(nu.sp_ext)
        wslot, _ = self.fc_weight_slot(u)
        io = 4 * (nu.numel + self._input_numel(nu))
        flops = 2 * O * K * S
        if (O <= SMALL_FC or (O <= 32 and O * K <= 1024)) and nu.sp_ext and len(nu.ext) == len(nu.sp_ext) + 1 and math.prod(nu.sp_ext) >= 512:
            # (also tiny square FCs, e.g. a MobileNetV2 1x1 target at C = 24: O*K FMAs
            # per pixel in registers beat a 1-k-block tensor-core tile, 0.16 ms there)
            # few outputs (fc(G), fc(1), ...): one thread per pixel computes all O
            # outputs in one pass over the K inputs (the input is read once, not O
            # times); needs enough pixels to fill the GPU (H*W >= 512 per image:
            # at 7x7 the per-output mapping is faster, measured 0.049 vs 0.084 ms)
            def body(f, u=u):
                sp = tuple(f.decompose("r", nu.sp_ext))
                accs = [f.fresh("acc") for _ in range(O)]
                f.emit("float " + ", ".join(f"{a_} = 0.f" for a_ in accs) + ";")
                i = f.fresh("i")
                if FC_SMALL_W4 and K % 4 == 0 and K >= 8:
                    # 4 inputs per step, one 16 B load per output row of W
                    f.emit("#pragma unroll 2")
                    f.open(f"for (int {i} = 0; {i} < {K}; {i} += 4)")
                    xs = []
                    for e in range(4):
                        ie = f.ivar(f"{i} + {e}") if e else i
                        xs.append(self.val(f, v, tuple(f.decompose(ie, nv.ch_ext)) + sp))
                    for o, a_ in enumerate(accs):
                        w4 = f.fresh("w")
                        f.emit(f"const float4 {w4} = __ldg(reinterpret_cast<const float4*>({f.ptr(wslot)} + {o * K} + {i}));" if f.V == 1 else f"float4 {w4} = __ldg(reinterpret_cast<const float4*>({f.ptr(wslot)} + {o * K} + {i}));")
                        for e, comp in enumerate("xyzw"):
                            f.emit(f"{a_} = fmaf({w4}.{comp}, {xs[e]}, {a_});")
                    f.close()
                else:
                    if FC_SMALL_UNROLL:
                        f.emit(f"#pragma unroll {FC_SMALL_UNROLL}")
                        f.open(f"for (int {i} = 0; {i} < {K}; ++{i})")
                    else:
                        f.loop(i, K)
                    ch = tuple(f.decompose(i, nv.ch_ext))
                    x = self.val(f, v, ch + sp)
                    for o, a_ in enumerate(accs):
                        f.emit(f"{a_} = fmaf(__ldg({f.ptr(wslot)} + {o * K} + {i}), {x}, {a_});")
                    f.close()
                for o, a_ in enumerate(accs):
                    for d, b in targets:
                        f.store(d, (str(o),) + sp, a_, b)

            self.launch_pointwise(name, math.prod(nu.sp_ext), body, 0, beta, f"fc_small {O}x{K} -> n{u}", io, flops, inner=nu.ext[-1] if nu.ext else 1, align16=FC_SMALL_W4 and K % 4 == 0 and K >= 8, vec_fill=FC_SMALL_VEC_FILL)
            return
        ks = self.ks_split(nu.numel, K) if min(O, K) <= SMALL_FC else 1
        if ks > 1:
            # few pixels, long reduction (fc(G) at 14x14 / 7x7: K = 256-512 per output):
            # KS lanes per output element split the K loop, xor-shuffle reduce

            def part(f, u=u):
                c = tuple(f.decompose("r", nu.ext))
                o, sp = c[0], c[1:]
                acc = f.fresh("acc")
                f.emit(f"float {acc} = 0.f;")
                wrow = f.ivar(f"{o}*{K}")
                i = f.fresh("i")
                f.emit("#pragma unroll 4")
                f.open(f"for (int {i} = part; {i} < {K}; {i} += {ks})")
                ch = tuple(f.decompose(i, nv.ch_ext))
                x = self.val(f, v, ch + sp)
                f.emit(f"{acc} = fmaf(__ldg({f.ptr(wslot)} + {wrow} + {i}), {x}, {acc});")
                f.close()
                f.emit(f"acc[0] = {acc};")

            def put(f):
                c = tuple(f.decompose("r", nu.ext))
                for d, b in targets:
                    f.store(d, c, "acc[0]", b)

            self.launch_ks(name, nu.numel, part, put, 1, ks, 0, beta, f"fc_small {O}x{K} -> n{u} (K split {ks})", io, flops)
            return
        if min(O, K) <= SMALL_FC:

            def body(f, u=u):
                c = self.coords_of(f, nu)
                o, sp = c[0], c[1:]
                acc = f.fresh("acc")
                f.emit(f"float {acc} = 0.f;")
                wrow = f.ivar(f"{o}*{K}")
                i = f.fresh("i")
                f.loop(i, K)
                ch = tuple(f.decompose(i, nv.ch_ext))
                x = self.val(f, v, ch + sp)
                f.emit(f"{acc} = fmaf(__ldg({f.ptr(wslot)} + {wrow} + {i}), {x}, {acc});")
                f.close()
                for d, b in targets:
                    f.store(d, c, acc, b)

            self.launch_pointwise(name, nu.numel, body, 0, beta, f"fc_small {O}x{K} -> n{u}", io, flops, inner=nu.ext[-1] if nu.ext else 1, node=nu)
            return
        # A(m,k) = W[m*K + k];  B(n,k,s) = val(v)(decompose k | decompose s)
        fa = Fn(self)
        fa.pre = []
        fa.computing = None
        a_expr = f"__ldg({fa.ptr(wslot)} + m*{K} + k)"

        def bfn(f):
            ch = tuple(f.decompose("k", nv.ch_ext))
            sp = tuple(f.decompose("s", nv.sp_ext))
            return self.val(f, v, ch + sp)

        def sfn(f, val):
            c = ("m",) + tuple(f.decompose("s", nu.sp_ext))
            for d, b in targets:
                f.store(d, c, val, b)

        # a computed operand (not a pure view of a materialised tensor) whose FC
        # has a tensor-core wgrad: the forward producers also write the operand
        # they evaluate, so the wgrad's B is a plain coalesced load instead of
        # re-evaluating the producer chain (computed-operand GEMMs are
        # bound by operand evaluation, not by the tensor pipe)
        save = None
        if SAVE_OPERAND and v not in self.fwd_desc and nv.op not in VIEW_OPS and O > 16 and K >= 32:
            sdesc = self._new_saved(nv.ext)
            sidx = len(self.p.saved) - 1

            def save(f, sdesc=sdesc):
                c = tuple(f.decompose("k", nv.ch_ext)) + tuple(f.decompose("s", nv.sp_ext))
                f.store(sdesc, c, "val", False)

        saved = self.emit_gemm_nk(name, fa, a_expr, bfn, sfn, M=O, K=K, S=S, phase=0, beta=beta, what=f"fc {O}x{K}x{S} -> n{u}", nbytes=io, flops=flops, save=save)
        if save is not None:
            if saved:
                self.fwd_desc[v] = sdesc  # later readers (the wgrad B operand) load it
            else:
                self.p.saved[sidx] = SizeRule(0, 1, 0)  # path without operand write-back: no buffer

    @staticmethod
    def split_operand(name: str, f: Fn, val: str, uvar: str) -> list:
        """Operand functor in row-split form: ``{name}R`` holds the row context
        (every index term that depends on the row variable ``uvar`` only — channel
        decompositions, tap offsets, per-row base offsets), ``{name}row(a, uvar)``
        computes it, ``{name}k(a, R, n, s)`` evaluates one element from it.  The
        tcgen05 producers whose rows are fixed for a whole CTA (wgrad) build the
        row contexts once and pay only the per-pixel part per element;
        ``{name}(a, n, uvar, s)`` composes the two for the other templates."""
        # the row variable itself travels in the context too: caller-written bodies
        # (dense_conv.py) reference it directly
        mem = [uvar + "_"] + list(f.uni_vars)
        out = [f"  struct {name}R {{ int {', '.join(mem)}; }};"]
        out.append(f"  static __device__ __forceinline__ {name}R {name}row(const CanvasArgs& a, const int {uvar}) {{")
        out += ["    " + ln for ln in f.uni_lines]
        out.append(f"    {name}R R;")
        out.append(f"    R.{uvar}_ = {uvar};")
        out += [f"    R.{v} = {v};" for v in mem[1:]]
        out += ["    return R;", "  }"]
        out.append(f"  static __device__ __forceinline__ float {name}k(const CanvasArgs& a, const {name}R& R, const long long n, const int s) {{")
        out.append(f"    const int {uvar} = R.{uvar}_; (void){uvar};")
        out += [f"    const int {v} = R.{v};" for v in mem[1:]]
        out += ["    " + ln for ln in f.pre] + f.lines + [f"    return {val};", "  }"]
        out.append(f"  static __device__ __forceinline__ float {name}(const CanvasArgs& a, const long long n, const int {uvar}, const int s) {{ return {name}k(a, {name}row(a, {uvar}), n, s); }}")
        return out

    def vec_operand(self, name: str, fn, uvar: str, S: int, local_slots: list, lane_n: bool = False, pad: bool = False) -> list:
        """4-pixel form of an operand functor (Fn vector mode): ``{name}R`` /
        ``{name}row(a, uvar)`` (its own row context) and ``{name}k(a, R, n, s, o)``
        writing pixels s .. s+3 (s a multiple of 4) to o[0..3].  The lane-invariant
        index math (channel / tap decomposition, image base, row offsets, the pixel's
        (h, w) split when W % 4 == 0) runs once per 4 pixels and lane-affine loads
        share one address (immediate offsets).  [] when S % 4 != 0 or the body is
        not vectorisable (the template then keeps the scalar producer)."""
        if not VEC_PRODUCERS or (S % 4 and not lane_n and not pad):
            return []
        f = Fn(self)
        f.pre = []
        f.computing = None
        f.local_slots = local_slots
        f.uniform = {uvar}
        f.hoist = True
        f.V = 4
        f.lanes = {} if lane_n else {"s": (1, 4, 0)}
        f.lane_n = lane_n
        if pad and S % 4:
            f.lane_pred = f"(s < {S})"
        try:
            val = fn(f)
        except VecUnsupported:
            return []
        self._op_vec16 = self._op_vec16 or f.vec16
        mem = [uvar + "_"] + list(f.uni_vars)
        out = [f"  struct {name}R {{ int {', '.join(mem)}; }};"]
        out.append(f"  static __device__ __forceinline__ {name}R {name}row(const CanvasArgs& a, const int {uvar}) {{")
        out += ["    " + ln for ln in f.uni_lines]
        out += [f"    {name}R R;", f"    R.{uvar}_ = {uvar};"] + [f"    R.{v} = {v};" for v in mem[1:]] + ["    return R;", "  }"]
        unpack = [f"    const int {uvar} = R.{uvar}_; (void){uvar};"] + [f"    const int {v} = R.{v};" for v in mem[1:]]
        outs = [val + "_" + str(e) if val in f.copies else val for e in range(4)]
        out.append(f"  static __device__ __forceinline__ void {name}k(const CanvasArgs& a, const {name}R& R, const long long n, const int s, float* o) {{")
        out += unpack + ["    " + ln for ln in f.pre] + f.lines
        out += [f"    o[{e}] = {outs[e]};" for e in range(4)]
        out.append("  }")
        out += self.split_load_compute(name, f, outs, unpack, uvar, mem)
        # row class for producer row grouping: the run-time shifts m of the row's quads
        cls = [c for c in dict.fromkeys(f.rt_cls) if c]
        body = " | ".join(f"((R.{c} & 3) << {2 * i})" for i, c in enumerate(cls[:8])) if cls and None not in f.rt_cls else "0"
        out.append(f"  static constexpr bool {name}CLS = {'true' if body != '0' else 'false'};")
        out.append(f"  static __device__ __forceinline__ int {name}cls(const {name}R& R) {{ return {body}; }}")
        # row key: the row-context offset of the last unit-stride gather (on seed-7 #1
        # the unfold read c*HW + dh*W + dw) — producers that sort a tile's rows by it
        # put rows reading the same lines into one warp instruction
        key = f.row_keys[-1] if f.row_keys and ROW_KEYS else None
        out.append(f"  static constexpr bool {name}KEY = {'true' if key else 'false'};")
        out.append(f"  static __device__ __forceinline__ int {name}key(const {name}R& R) {{ return {'R.' + key if key else '0'}; }}")
        return out

    @staticmethod
    def split_load_compute(name: str, f: Fn, outs: list, unpack: list, uvar: str, mem: list) -> list:
        """Load / compute split of a 4-pixel operand functor for software-pipelined
        producers: ``{name}ld(a, R, n, s, raw)`` issues the gathers (index math,
        predicates, 16 B chunks) into ``{name}NRAW`` raw registers, ``{name}cp(a, R,
        raw, o)`` evaluates the pointwise chain from them — so the loads of k-block
        kb+1 are in flight while k-block kb is combined and stored.  ``{name}SPLIT``
        is false when the float chain reads index values (guards on computed nodes)."""
        no = [f"  static constexpr bool {name}SPLIT = false;", f"  static constexpr int {name}NRAW = 1;",
              f"  static __device__ __forceinline__ void {name}ld(const CanvasArgs&, const {name}R&, const long long, const int, float*) {{}}",
              f"  static __device__ __forceinline__ void {name}cp(const CanvasArgs&, const {name}R&, const float*, float*) {{}}"]
        if "x" in f.ltags or not VEC_SPLIT:
            return no
        tagged = list(zip(f.lines, f.ltags))
        ints = {"a", "n", "s", uvar, "R"} | set(mem)
        for ln in f.pre + [x for x, t in tagged if t in "il"]:
            m = re.match(r"\s*(?:const int|float\* const|const float\* const|float\* __restrict__) (\w+) =", ln)
            if m:
                ints.add(m.group(1))
        # load half outputs: scalar loads and 16 B chunks (floats), bit words (ints)
        fl, f4, iw = [], [], []
        for ln, t in tagged:
            if t != "l":
                continue
            m = re.match(r"\s*const (float4|float|int) (\w+) =", ln)
            if m:
                {"float": fl, "float4": f4, "int": iw}[m.group(1)].append(m.group(2))
        comp = [(x, t) for x, t in tagged if t in "sc"]
        used = set()
        for ln, t in comp:
            m = re.match(r"\s*const float4? (\w+) = (.*);$", ln)
            if not m:
                return no
            toks = set(_IDENT.findall(m.group(2))) - {"canvas", "win4"}
            bad = toks & ints - set(iw) if t == "s" else toks & ints
            if bad:
                return no
            used |= toks
        for o in outs:
            used |= set(_IDENT.findall(o))
        fl = [v for v in fl if v in used]
        f4 = [v for v in f4 if v in used]
        iw = [v for v in iw if v in used]
        nr = len(fl) + 4 * len(f4) + len(iw)
        if not nr:
            return no
        out = [f"  static constexpr bool {name}SPLIT = true;", f"  static constexpr int {name}NRAW = {nr};"]
        out.append(f"  static __device__ __forceinline__ void {name}ld(const CanvasArgs& a, const {name}R& R, const long long n, const int s, float* raw) {{")
        out += unpack + ["    " + ln for ln in f.pre]
        out += [x for x, t in tagged if t in "il"]
        j = 0
        put, get = [], []
        for v in fl:
            put.append(f"    raw[{j}] = {v};")
            get.append(f"    const float {v} = raw[{j}];")
            j += 1
        for v in f4:
            put.append(f"    raw[{j}] = {v}.x; raw[{j + 1}] = {v}.y; raw[{j + 2}] = {v}.z; raw[{j + 3}] = {v}.w;")
            get.append(f"    const float4 {v} = make_float4(raw[{j}], raw[{j + 1}], raw[{j + 2}], raw[{j + 3}]);")
            j += 4
        for v in iw:
            put.append(f"    raw[{j}] = __int_as_float({v});")
            get.append(f"    const int {v} = __float_as_int(raw[{j}]);")
            j += 1
        out += put + ["  }"]
        out.append(f"  static __device__ __forceinline__ void {name}cp(const CanvasArgs& a, const {name}R& R, const float* raw, float* o) {{")
        out += get + [x for x, _ in comp]
        out += [f"    o[{e}] = {outs[e]};" for e in range(4)]
        out.append("  }")
        return out

    @staticmethod
    def prefetch_members(f: Fn, fns, S: int) -> list:
        """``NPF`` / ``pf_addr``: one 128 B line per row of every materialised
        tensor the producer functors ``fns`` read, at pixel (n, s) — the
        producers warm L2 with the rows of upcoming k-blocks / of their pixel
        tile, so the gathers hit L2 instead of waiting on DRAM.  A tensor with
        an image stride that is a multiple of S is treated as [rows][S]; every
        address stays inside its image, so a mismatch only wastes a prefetch."""
        rows = []
        seen = set()
        for g in fns:
            for key, d in g.loaded.items():
                if key in seen:
                    continue
                seen.add(key)
                if d.bstride % S == 0 and d.bstride // S >= 1:
                    rows.append((f.ptr(d.slot), d.bstride, d.bstride // S))
        if not L2_PREFETCH or not rows:
            return ["  static constexpr int NPF = 0;", "  static __device__ __forceinline__ const float* pf_addr(const CanvasArgs&, const long long, const int, const int) { return nullptr; }"]
        body = ["  static __device__ __forceinline__ const float* pf_addr(const CanvasArgs& a, const long long n, const int s, int i) {"]
        for ptr, bs, r in rows:
            body.append(f"    if (i < {r}) return {ptr} + n * {bs}LL + (long long)i * {S} + s;")
            body.append(f"    i -= {r};")
        body.append("    return nullptr;")
        body.append("  }")
        return [f"  static constexpr int NPF = {sum(r for _, _, r in rows)};"] + body

    def emit_gemm_nk(self, name, fa: Fn, a_expr: str, bfn, sfn, M, K, S, phase, beta, what, nbytes, flops, save=None, epi=None) -> bool:
        """C[n][m][s] = sum_k A(m,k) * B(n,k,s) through canvas::gemm_nk (one shared slot table).
        ``save(f)``: emit the store of B's value ``val`` at (n, k, s) — the operand
        write-back; honoured (returns True) only on the non-persistent tcgen05 path.
        ``epi`` = (NT, functor lines): a custom TMEM epilogue (EPI_BC) on the
        persistent tcgen05 path with column tiles of NT."""
        fb = Fn(self)
        fb.pre = []
        fb.computing = None
        fb.local_slots = fa.local_slots  # share the pointer table
        fb.uniform = {"k"}  # tcgen05 producers: k-row per warp, lane = pixel
        fb.hoist = True
        bval = bfn(fb)
        fs = Fn(self)
        fs.pre = []
        fs.computing = None
        fs.local_slots = fa.local_slots
        fs.uniform = {"m"}  # TMEM epilogue: column per iteration, lane = pixel
        if sfn is not None:
            sfn(fs, "acc")
        lines = [
            f"struct {name}_F {{",
            f"  static constexpr int M = {M}, K = {K}, S = {S};",
            "  static __device__ __forceinline__ float A(const CanvasArgs& a, const int m, const int k) {",
            f"    return {a_expr};",
            "  }",
        ]
        lines += self.split_operand("B", fb, bval, "k")
        self._op_vec16 = False
        # S % 4 != 0 (7x7): the tc_gemm_pix quad producers run over a per-image pixel
        # range padded to SP (padding columns computed from zero loads, not stored)
        tc = self.use_tc and M >= 8 and K >= 16
        nacc_p = 1
        while nacc_p < 4 and K > TC_ACC_K * nacc_p:
            nacc_p *= 2
        pix_path = tc and not epi and not tmema_wanted(K) and TC_A_MN == "true" and not (TC_PERSIST and K < 4 * tc_tile(M, min(TC_NTMAX, 512 // nacc_p))[0])
        SP = -(-S // 4) * 4 if (pix_path and VEC_PAD_FWD and S % 4) else S
        vec = self.vec_operand("B4", bfn, "k", S, fa.local_slots, pad=SP != S)
        if not vec:
            SP = S
        lines += vec + [f"  static constexpr bool VEC = {'true' if vec else 'false'};", f"  static constexpr int SP = {SP};"]
        if not vec:
            lines += ["  static constexpr bool B4CLS = false, B4KEY = false;"]
        lines += [f"  static constexpr bool SPLIT = {'true' if vec and 'B4SPLIT = true' in chr(10).join(vec) else 'false'};"]
        lines += ["  static __device__ __forceinline__ void store(const CanvasArgs& a, const long long n, const int m, const int s, const float acc) {"]
        lines += ["    " + s for s in fs.pre] + fs.lines + ["  }"]
        lines += epi[1] if epi else ["  static constexpr bool EPI_BC = false;", "  static constexpr int EPI_M = 1, EPI_JT = 16, EPI_NBUF = 2, EPI_WPB = 1;"]
        if epi and not tc:
            raise LoweringError("epilogue fusion needs the tensor-core dgrad")
        nacc0 = 1
        while nacc0 < 4 and K > TC_ACC_K * nacc0:
            nacc0 *= 2
        persistent = tc and TC_PERSIST and K < 4 * tc_tile(M, min(TC_NTMAX, 512 // nacc0))[0]
        do_save = save is not None and tc and not persistent and TC_A_MN == "true"
        if do_save:
            fv = Fn(self)
            fv.pre = []
            fv.computing = None
            fv.local_slots = fa.local_slots
            fv.uniform = {"k"}
            save(fv)
            lines += ["  static constexpr bool SAVE_B = true;", "  static __device__ __forceinline__ void save_b(const CanvasArgs& a, const long long n, const int k, const int s, const float val) {"]
            lines += ["    " + s for s in fv.pre] + fv.lines + ["  }"]
        else:
            lines += ["  static constexpr bool SAVE_B = false;", "  static __device__ __forceinline__ void save_b(const CanvasArgs&, const long long, const int, const int, const float) {}"]
        lines += self.prefetch_members(fa, [fb], S)
        lines += ["};"]
        functor = "\n".join(lines) + "\n"
        if tc:
            # long reductions run over NACC TMEM accumulators (<= TC_ACC_K terms each),
            # which caps the column tile so NACC x NT fits the 512 TMEM columns
            nacc = 1
            while nacc < 4 and K > TC_ACC_K * nacc:
                nacc *= 2
            nt, nct, stages = tc_tile(M, min(TC_NTMAX, 512 // nacc))
            if epi:
                nt, nct = epi[0], M // epi[0]
            smem = tc_smem_bytes(nt, stages)
            kb = -(-K // 32)
            pack_bytes = nct * kb * 2 * nt * 128
            if phase == 0:
                self.p.saved.append(SizeRule(0, 1, pack_bytes))
                pslot = self.p.slot_saved(len(self.p.saved) - 1)
            else:
                k_ws, _ = self._new_ws((1,))
                self.p.ws[k_ws] = SizeRule(0, 1, pack_bytes)
                pslot = -1 - k_ws
            ploc = fa.ptr(pslot)
            functor = functor[: functor.rindex("};")] + f"  static __device__ __forceinline__ float* packed(const CanvasArgs& a) {{ return {ploc}; }}\n}};\n"
            if epi or (TC_PERSIST and K < 4 * nt):  # epilogue-heavy: overlap stores with the next tile
                pstages, psmem = tc_persist_cfg(nt)
                pw = TC_PW if K > 128 else 4  # short reductions: cheap mainloop, store-bound epilogue
                ew = 8 if nt >= 128 else 4
                if epi:  # one warpgroup per (TMEM buffer, column share)
                    me = re.search(r"EPI_NBUF = (\d+), EPI_WPB = (\d+)", "\n".join(epi[1]))
                    ew = 4 * int(me.group(1)) * int(me.group(2))
                threads = (pw + 2 + ew) * 32
                launcher = f'extern "C" __global__ void __launch_bounds__({threads}, 1) {name}(const CanvasArgs a) {{ canvas::tc_gemm_pix_persistent<{name}_F, {nt}, {pstages}, {pw}, {ew}>(a); }}\n'
                k = self.add_kernel(name, functor, launcher)
                pk = self.add_kernel(name + "_pack", "", f'extern "C" __global__ void __launch_bounds__(256) {name}_pack(const CanvasArgs a) {{ canvas::tc_pack_b<{name}_F, {nt}>(a); }}\n')
                total = nct * kb * nt * 32
                self.p.launches.append(Launch("kernel", phase, name + "_pack", pk, 256, (GridRule(0, total, 256, POINTWISE_CAP), GridRule(0, 1, 1), GridRule(0, 1, 1)), tuple(fa.local_slots), BETA_NONE, what=f"pack W tiles for {name}"))
                grid = (GridRule(S * nct, 0, 128, SMS), GridRule(0, 1, 1), GridRule(0, 1, 1))
                self.p.launches.append(Launch("kernel", phase, name, k, threads, grid, tuple(fa.local_slots), beta, smem=psmem, what="tc " + what, bytes_per_image=nbytes, flops_per_image=flops, align16=bool(vec) and self._op_vec16))
                return False
            # computed operand staged in tensor memory (A from TMEM): lane = pixel, no
            # smem stores; needs accumulators + 3 A stages (64 columns each) in TMEM
            if tmema_wanted(K) and not do_save and nacc * nt + 64 * 3 <= 512:
                # 3 A stages; 2 when that lets two CTAs share the SM's 512 TMEM columns
                tstages = TMEMA_STAGES or (3 if nacc * nt + 64 * 3 <= 256 or nacc * nt + 64 * 2 > 256 else 2)
                tcols = nacc * nt + 64 * tstages
                tpair = tcols <= 256
                tsmem = tstages * 2 * nt * 128 + (2 * tstages + 1) * 8 + 16 + 1024
                tpw = TC_TMEMA_PW
                tthreads = (tpw + 2) * 32
                launcher = f'extern "C" __global__ void __launch_bounds__({tthreads}, {2 if tpair and tpw <= 8 else 1}) {name}(const CanvasArgs a) {{ canvas::tc_gemm_pix_tmema<{name}_F, {nt}, {tstages}, {nacc}, {tpw}, {'true' if K <= TMEMA_UNROLL_MAX and tpw in (8, 16) else 'false'}>(a); }}\n'
                k = self.add_kernel(name, functor, launcher)
                pk = self.add_kernel(name + "_pack", "", f'extern "C" __global__ void __launch_bounds__(256) {name}_pack(const CanvasArgs a) {{ canvas::tc_pack_b<{name}_F, {nt}>(a); }}\n')
                total = nct * kb * nt * 32
                self.p.launches.append(Launch("kernel", phase, name + "_pack", pk, 256, (GridRule(0, total, 256, POINTWISE_CAP), GridRule(0, 1, 1), GridRule(0, 1, 1)), tuple(fa.local_slots), BETA_NONE, what=f"pack W tiles for {name}"))
                grid = (GridRule(S, 0, 128), GridRule(0, nct, 1), GridRule(0, 1, 1))
                self.p.launches.append(Launch("kernel", phase, name, k, tthreads, grid, tuple(fa.local_slots), beta, smem=tsmem, what="tc " + what, bytes_per_image=nbytes, flops_per_image=flops))
                return False
            # 2 CTAs x 8 producer warps when a 2-stage ring pairs on an SM, else 1 CTA x 16 warps
            pw = TC_PIX_PW if TC_PIX_PW else (8 if smem <= TC_SMEM_PAIR else 16)
            mraw = re.search(r"B4NRAW = (\d+)", functor)
            if not TC_PIX_PW and mraw and "SPLIT = true" in functor and (32 // 8) * int(mraw.group(1)) * 2 > 64:
                pw = 16  # pipelined producers: two k-blocks of raw gathers per thread must fit in registers
            threads = (pw + 2) * 32
            if pw > 8:
                stages = max(2, min(4, (220 * 1024) // (2 * 128 * 128 + 2 * nt * 128)))
                smem = tc_smem_bytes(nt, stages)
            pair = smem <= TC_SMEM_PAIR and pw <= 8 and 2 * nt * nacc <= 512
            launcher = f'extern "C" __global__ void __launch_bounds__({threads}, {2 if pair else 1}) {name}(const CanvasArgs a) {{ canvas::tc_gemm_pix<{name}_F, {nt}, {stages}, true, {TC_A_MN}, {pw}, {nacc}>(a); }}\n'
            k = self.add_kernel(name, functor, launcher)
            pk = self.add_kernel(name + "_pack", "", f'extern "C" __global__ void __launch_bounds__(256) {name}_pack(const CanvasArgs a) {{ canvas::tc_pack_b<{name}_F, {nt}>(a); }}\n')
            total = nct * kb * nt * 32
            self.p.launches.append(Launch("kernel", phase, name + "_pack", pk, 256, (GridRule(0, total, 256, POINTWISE_CAP), GridRule(0, 1, 1), GridRule(0, 1, 1)), tuple(fa.local_slots), BETA_NONE, what=f"pack W tiles for {name}"))
            grid = (GridRule(SP, 0, 128), GridRule(0, nct, 1), GridRule(0, 1, 1))
            self.p.launches.append(Launch("kernel", phase, name, k, threads, grid, tuple(fa.local_slots), beta, smem=smem, what="tc " + what, bytes_per_image=nbytes, flops_per_image=flops, align16=bool(vec) and self._op_vec16))
            return do_save
        launcher = f'extern "C" __global__ void __launch_bounds__(256) {name}(const CanvasArgs a) {{ canvas::gemm_nk<{name}_F>(a); }}\n'
        k = self.add_kernel(name, functor, launcher)
        grid = (GridRule(S, 0, GEMM_TILE), GridRule(0, M, GEMM_TILE), GridRule(0, 1, 1))
        self.p.launches.append(Launch("kernel", phase, name, k, 256, grid, tuple(fa.local_slots), beta, what=what, bytes_per_image=nbytes, flops_per_image=flops))
        return False

    def emit_gemm_wgrad(self, name, afn, bfn, M, J, S, dw_slot, what, nbytes, flops, trans: bool = False) -> None:
        """dW[m][j] = sum_{t=(n,s)} A(n,m,s) * B(n,j,s): deterministic split over t + ordered reduce.
        ``trans``: the reduce writes dW transposed ([J][M]) — callers swap the operand
        roles so the costlier computed operand sits on the less padded MMA side."""
        # tensor-core wgrad down to J = 8 rows (rows past J are never gathered) and
        # N >= 32 columns: the SIMT fallback was 72% of a MobileNetV2 1x1 layer at
        # C = 24 (1.56 -> 0.16 ms); wgrad_small stays for M <= 16 (faster at N = 16:
        # 0.40 vs 0.50 ms at 16x16 over 112^2)
        small = M <= 16
        use_tc = self.use_tc and J >= 8 and not small
        fa, fb = Fn(self), Fn(self)
        fa.pre, fb.pre = [], []
        fa.computing = fb.computing = None
        fb.local_slots = fa.local_slots
        fa.uniform, fb.uniform = {"m"}, {"k"}  # tcgen05 wgrad producers: row per warp, lane = pixel
        fa.hoist = fb.hoist = True
        aval = afn(fa)
        bval = bfn(fb)
        # vector producers over a padded pixel range when S % 4 != 0 (7x7: 49 -> 52):
        # the reduction's entries are (image, padded pixel), padding masked to zero.
        # At 7x7 the quads' loads are unaligned (4 B lane stride), so they pay off only
        # where the scalar producers are gather-bound: >= VEC_PAD_MIN_LOADS loads per
        # element of the (input-channel side) operand — seed-7 #1 (2 loads) 0.68 ->
        # 0.44 ms, im2col / involution (1 load) 0.32 -> 0.39 / 0.064 -> 0.070 ms
        nld_b = sum(ln.count("__ldg") for ln in fb.pre + fb.lines)
        SP = -(-S // 4) * 4 if (use_tc and VEC_PAD and S % 4 and not VEC_NQ and nld_b >= VEC_PAD_MIN_LOADS) else S
        # register-blocked small wgrad over pixel quads (wgrad_small_v): JW rows of the
        # J side x all M rows per warp, WJ row groups x 8/WJ pixel streams per CTA
        small_v = small and WGRAD_SMALL_V and S % 4 == 0
        if small_v:
            jw = min(8 if M <= 8 else 2, 1 << max(0, (J - 1).bit_length()))
            wj = min(8, 1 << max(0, (-(-J // jw) - 1).bit_length()))
            jblk = -(-J // (jw * wj))
            z = -(-(4 * SMS) // jblk)  # ~4 CTAs per SM at batch 256
            tchunk = max(128, -(-(-(-(256 * S) // z)) // 128) * 128)
        elif small:  # ~8 CTAs per SM at batch 256: chunk = 256*S*jtiles / (8*148), multiple of 64
            jt0 = min(1 << max(0, (256 // M).bit_length() - 1), 1 << max(0, (J - 1).bit_length()), WGRAD_SMALL_JT_MAX)
            tchunk = max(64, -(-(256 * S * -(-J // jt0)) // (8 * SMS * 64)) * 64)
        else:
            if use_tc:  # >= ~6 CTAs per SM at batch 256 without going below 512 pixels per partial
                tiles = -(-J // (128 * wgrad_jg(J, tc_tile(M)[0]))) * tc_tile(M)[1]
                z = -(-(6 * SMS) // tiles)
                tchunk = min(TC_WGRAD_TCHUNK, max(512, -(-(-(-(256 * SP) // z)) // 128) * 128))
            else:
                tchunk = max(2048, -(-4096 * S // 60000) * GEMM_TILE)
        k_ws, pdesc = self._new_ws((1,))
        self.p.ws[k_ws] = SizeRule(4 * SP * M * J, tchunk, 4 * M * J)
        pslot_local = fa.ptr(-1 - k_ws)  # partials (fixed up to the real ws slot in finish())
        lines = [
            f"struct {name}_F {{",
            f"  static constexpr int M = {M}, J = {J}, S = {S}, SP = {SP}, TCHUNK = {tchunk};",
        ]
        lines += self.split_operand("A", fa, aval, "m")
        lines += self.split_operand("B", fb, bval, "k")
        self._op_vec16 = False
        nq = S % 4 != 0 and VEC_NQ  # quads over 4 images at one pixel (7x7: 49 pixels)
        va4 = self.vec_operand("A4", afn, "m", S, fa.local_slots, lane_n=nq, pad=SP != S)
        vb4 = self.vec_operand("B4", bfn, "k", S, fa.local_slots, lane_n=nq, pad=SP != S) if va4 else []
        if nld_b < VEC_PAD_MIN_LOADS or SP != S:  # row ordering pays only on gather-bound rows (seed-7 #1: 0.787 -> 0.742 ms; im2col / involution: 1-5% slower; 7x7 padded quads: 0.44 -> 0.48 ms)
            vb4 = [ln.replace("B4KEY = true", "B4KEY = false") for ln in vb4]
        lines += (va4 + vb4) if vb4 else []
        lines += [f"  static constexpr bool VEC = {'true' if vb4 else 'false'}, NQ = {'true' if vb4 and nq else 'false'};"]
        if not vb4:
            lines += ["  static constexpr bool B4CLS = false, B4KEY = false;"]
        both = vb4 and "A4SPLIT = true" in chr(10).join(va4) and "B4SPLIT = true" in chr(10).join(vb4)
        lines += [f"  static constexpr bool SPLIT = {'true' if both else 'false'};"]
        lines += [f"  static __device__ __forceinline__ float* partials(const CanvasArgs& a) {{ return {pslot_local}; }}"]
        lines += self.prefetch_members(fa, [fb, fa], S)
        lines += ["};"]
        functor = "\n".join(lines) + "\n"
        if use_tc:
            nt, nct, stages = tc_tile(M)
            jg = wgrad_jg(J, nt)
            if jg > 1:
                stages = 2
                smem = wgrad_smem_bytes(nt, jg, stages)
            else:
                smem = tc_smem_bytes(nt, stages)
            pw = TC_WGRAD_PW
            threads = (pw + 2) * 32
            pair = smem <= TC_SMEM_PAIR and pw <= 8
            launcher = f'extern "C" __global__ void __launch_bounds__({threads}, {2 if pair else 1}) {name}(const CanvasArgs a) {{ canvas::tc_gemm_wgrad<{name}_F, {nt}, {stages}, {pw}, {jg}>(a); }}\n'
            k = self.add_kernel(name, functor, launcher)
            grid = (GridRule(0, J, 128 * jg), GridRule(0, nct, 1), GridRule(SP, 0, tchunk))
            self.p.launches.append(Launch("kernel", 1, name, k, threads, grid, tuple(fa.local_slots), BETA_NONE, smem=smem, what="tc " + what, bytes_per_image=nbytes, flops_per_image=flops, align16=bool(vb4) and self._op_vec16))
        elif small_v and vb4 and not nq:
            functor = functor[: functor.rindex("};")] + f"  static constexpr int JW = {jw}, WJ = {wj};\n}};\n"
            launcher = f'extern "C" __global__ void __launch_bounds__(256, 2) {name}(const CanvasArgs a) {{ canvas::wgrad_small_v<{name}_F>(a); }}\n'
            k = self.add_kernel(name, functor, launcher)
            grid = (GridRule(0, J, jw * wj), GridRule(0, 1, 1), GridRule(S, 0, tchunk))
            self.p.launches.append(Launch("kernel", 1, name, k, 256, grid, tuple(fa.local_slots), BETA_NONE, what="small " + what, bytes_per_image=nbytes, flops_per_image=flops, align16=self._op_vec16))
        elif small:
            jt = min(1 << max(0, (256 // M).bit_length() - 1), WGRAD_SMALL_JT_MAX)
            jt = min(jt, 1 << (J - 1).bit_length()) if J > 1 else 1
            functor = functor[: functor.rindex("};")] + f"  static constexpr int JT = {jt};\n}};\n"
            launcher = f'extern "C" __global__ void __launch_bounds__(256) {name}(const CanvasArgs a) {{ canvas::wgrad_small<{name}_F>(a); }}\n'
            k = self.add_kernel(name, functor, launcher)
            grid = (GridRule(0, J, jt), GridRule(0, 1, 1), GridRule(S, 0, tchunk))
            self.p.launches.append(Launch("kernel", 1, name, k, 256, grid, tuple(fa.local_slots), BETA_NONE, what="small " + what, bytes_per_image=nbytes, flops_per_image=flops))
        else:
            launcher = f'extern "C" __global__ void __launch_bounds__(256) {name}(const CanvasArgs a) {{ canvas::gemm_wgrad<{name}_F>(a); }}\n'
            k = self.add_kernel(name, functor, launcher)
            grid = (GridRule(0, J, GEMM_TILE), GridRule(0, M, GEMM_TILE), GridRule(S, 0, tchunk))
            self.p.launches.append(Launch("kernel", 1, name, k, 256, grid, tuple(fa.local_slots), BETA_NONE, what=what, bytes_per_image=nbytes, flops_per_image=flops))
        # ordered reduction of the partials into dW
        rname = name + "_reduce"
        rsrc = (
            f"struct {rname}_F {{ static constexpr int MJ = {M * J}, S = {SP}, TCHUNK = {tchunk}, TJ = {J if trans else 0}; }};\n"
            f'extern "C" __global__ void __launch_bounds__(256) {rname}(const CanvasArgs a) {{ canvas::reduce_partials<{rname}_F>(a); }}\n'
        )
        k2 = self.add_kernel(rname, "", rsrc)
        grid2 = (GridRule(0, M * J * (1 if M * J >= 4096 else 32), 256), GridRule(0, 1, 1), GridRule(0, 1, 1))
        self.p.launches.append(Launch("kernel", 1, rname, k2, 256, grid2, (-1 - k_ws, dw_slot), BETA_NONE, what=f"wgrad reduce {M}x{J}"))

    # ---- backward
    def lower_backward(self) -> None:
        p = self.p
        self.dy_desc = self.y_desc(SLOT_DY)
        stride_gt1 = p.stride > 1
        dx_beta = BETA_ALWAYS if stride_gt1 else (BETA_AFTER_FIRST if (p.copies > 1 and p.mode == "concat") else BETA_NONE)
        if stride_gt1:
            p.launches.append(Launch("memset", 1, "dx_zero", memset_slot=SLOT_DX, memset_size=SizeRule(4 * p.c_in * p.h_in * p.w_in, 1, 0), what="dx zero-fill (stride > 1)"))
        # FC dgrads that absorb the adjoint of their input broadcast (epilogue fusion)
        for u in (nd.id for nd in self.nodes if nd.op == "fc"):
            jt = self.epi_bc_tile(u)
            if jt:
                self.epi_bc[u] = jt
        # where each materialised gradient lives
        for v in sorted(self.grad_mat):
            nd = self.nodes[v]
            if v == 0:
                self.grad_desc[0] = self.dx_desc()
                continue
            only_fc = len(nd.consumers) == 1 and self.nodes[nd.consumers[0][0]].op == "fc"
            if only_fc:
                continue  # the FC dgrad writes this gradient directly (no extra pass)
            _, d = self._new_ws(nd.ext)
            self.grad_desc[v] = d
        for u in sorted(self.nodes[i].id for i in range(len(self.nodes)) if self.nodes[i].op == "fc"):
            v = self.nodes[u].ins[0]
            nv = self.nodes[v]
            if u in self.epi_bc:
                # dL/dv itself is never stored: the epilogue writes the rhs edge
                # contribution (shape of v) and the lhs replica sum
                lhs, rhs = nv.ins
                _, self.edge_desc[(v, 1)] = self._new_ws(nv.ext)
                nl = self.nodes[lhs]
                if lhs in self.grad_mat and len(nl.consumers) == 1:
                    self.edge_desc[(v, 0)] = self.grad_desc[lhs]
                    self.grad_by_epi.add(lhs)
                else:
                    _, self.edge_desc[(v, 0)] = self._new_ws(nl.ext)
                self.grad_by_epi.add(v)
                continue
            if v in self.grad_mat and len(nv.consumers) == 1:
                if v == 0:
                    self.dgrad_desc[u] = self.dx_desc()
                else:
                    _, d = self._new_ws(nv.ext)
                    self.dgrad_desc[u] = d
                    self.grad_desc[v] = d
            elif INLINE_SMALL_DGRAD and self.g.fc_shape(u)[0] <= SMALL_FC and len(self.nodes[u].ext) == len(self.nodes[u].sp_ext) + 1:
                self.inline_dgrad.add(u)  # consumers of v evaluate this FC's contribution inline
            else:
                _, d = self._new_ws(nv.ext)
                self.dgrad_desc[u] = d
        for u in (nd.id for nd in self.nodes if nd.op == "softmax"):
            pre, span, post = self.softmax_geom(self.nodes[u])
            _, self.dot_desc[u] = self._new_ws(pre + post)

        # gradient tensors not yet written at a point of the schedule (slots)
        self._pending = {d.slot for d in self.grad_desc.values()} | {d.slot for d in self.dgrad_desc.values()}
        self._pending |= {d.slot for d in self.dot_desc.values()} | {d.slot for d in self.edge_desc.values()}
        self._pending.discard(self.dx_desc().slot)
        fused_early: set = set()
        for u in range(len(self.nodes) - 1, -1, -1):
            nu = self.nodes[u]
            # 1) materialise dL/du if it is a gradient sum point (not dy, not aliased to an FC dgrad)
            if u in self.grad_mat and not self._grad_is_fc_alias(u) and u not in self.grad_by_epi and u not in fused_early:
                beta = dx_beta if u == 0 else BETA_NONE
                d = self.grad_desc[u]
                sib = self.grad_sibling(u) if u != 0 else None
                if sib is None:
                    name = f"k{len(p.kernel_names)}_bwd_grad{u}"
                    self.launch_pointwise(name, nu.numel, lambda f, u=u, d=d: self.body_grad(f, u, d), 1, beta, f"grad n{u}", 4 * 3 * nu.numel, 0, inner=nu.ext[-1] if nu.ext else 1, node=nu)
                else:
                    w, dw_ = sib, self.grad_desc[sib]
                    name = f"k{len(p.kernel_names)}_bwd_grad{u}_{w}"

                    def body2(f, u=u, d=d, w=w, dw_=dw_):
                        self.body_grad(f, u, d)
                        self.body_grad(f, w, dw_)

                    self.launch_pointwise(name, nu.numel, body2, 1, beta, f"grad n{u} + n{w}", 4 * 6 * nu.numel, 0, inner=nu.ext[-1] if nu.ext else 1, node=nu)
                    fused_early.add(w)
                    self._pending.discard(dw_.slot)
                self._pending.discard(d.slot)
            # 2) adjoint kernels of the producer edge that need dL/du as a whole
            if nu.op == "fc":
                self.lower_fc_bwd(u, dx_beta)
                for dd in (self.dgrad_desc.get(u),) + tuple(self.edge_desc.get((nu.ins[0], i)) for i in (0, 1)):
                    if dd is not None:
                        self._pending.discard(dd.slot)
            elif nu.op == "softmax":
                self.lower_softmax_dot(u)
                self._pending.discard(self.dot_desc[u].slot)

    def grad_sibling(self, u: int):
        """A later gradient tensor dL/dw (w < u) computable in the same launch as
        dL/du: same elements per image and spatial extent, and every gradient it
        reads already written before this point (checked by emitting its body into
        a scratch functor).  One pass then reads their shared sources once — on
        seed-7 #1 dL/dn7 and dL/dn1 both gather the 9C-wide dL/dn8 (the FC dgrad's
        output) at the same and at neighbouring pixels."""
        if not GRAD_SIBLINGS:
            return None
        nu = self.nodes[u]
        for w in range(u - 1, 0, -1):
            nw = self.nodes[w]
            if w not in self.grad_mat or self._grad_is_fc_alias(w) or w in self.grad_by_epi:
                continue
            if nw.numel != nu.numel or tuple(nw.sp_ext) != tuple(nu.sp_ext) or tuple(nw.ext[len(nw.ext) - len(nw.sp_ext):]) != tuple(nu.ext[len(nu.ext) - len(nu.sp_ext):]):
                continue
            f = Fn(self)
            f.pre = []
            f.computing = None
            f.planes = None
            try:
                self.body_grad(f, w, self.grad_desc[w])
            except (VecUnsupported, LoweringError):
                continue
            finally:
                self.computing_grad = None
            reads = {d.slot for d in f.loaded.values()}
            if reads & (self._pending - {self.grad_desc[w].slot}):
                continue
            return w
        return None

    def _grad_is_fc_alias(self, v: int) -> bool:
        nd = self.nodes[v]
        return len(nd.consumers) == 1 and self.nodes[nd.consumers[0][0]].op == "fc"

    def body_grad(self, f: Fn, v: int, d: TDesc) -> None:
        nd = self.nodes[v]
        c = self.coords_of(f, nd)
        self.computing_grad = v
        g = self.grad_sum(f, v, c)
        self.computing_grad = None
        f.store(d, c, g, v == 0)

    def lower_softmax_dot(self, u: int) -> None:
        nu = self.nodes[u]
        pre, span, post = self.softmax_geom(nu)
        rows = math.prod(pre) * math.prod(post)
        S = math.prod(span)
        d = self.dot_desc[u]

        def body(f):
            rc = f.decompose("r", pre + post)
            pc, qc = tuple(rc[: len(pre)]), tuple(rc[len(pre) :])
            acc = f.fresh("acc")
            f.emit(f"float {acc} = 0.f;")
            j = f.fresh("j")
            f.loop(j, S)
            c = pc + tuple(f.decompose(j, span)) + qc
            g = self.grad(f, u, c)
            y = self.val(f, u, c)
            f.emit(f"{acc} = fmaf({g}, {y}, {acc});")
            f.close()
            f.store(d, pc + qc, acc, False)

        name = f"k{len(self.p.kernel_names)}_bwd_softmaxdot{u}"
        rext = pre + post
        sl = self.row_split(rows, S)
        if sl > 1:

            def term(f, c, rowc):
                return f.fvar(f"{self.grad(f, u, c)} * {self.val(f, u, c)}")

            def put(f, c, rowc):
                f.store(d, rowc, "v", False)

            functor, slots = self._row_functor(name, nu, [
                ("float term(const CanvasArgs& a, const long long n, const int r, const int j)", term),
                ("void put(const CanvasArgs& a, const long long n, const int r, const float v)", put),
            ])
            launcher = f'extern "C" __global__ void __launch_bounds__(256) {name}(const CanvasArgs a) {{ canvas::rowdot_rows<{name}_F, {sl}>(a); }}\n'
            k = self.add_kernel(name, functor, launcher)
            grid = (GridRule(rows, 0, 256 // sl, POINTWISE_CAP), GridRule(0, 1, 1), GridRule(0, 1, 1))
            self.p.launches.append(Launch("kernel", 1, name, k, 256, grid, tuple(slots), BETA_NONE, what=f"softmax row-dot n{u} ({sl} threads/row)", bytes_per_image=4 * (2 * nu.numel + rows)))
            return
        self.launch_pointwise(name, rows, body, 1, BETA_NONE, f"softmax row-dot n{u}", 4 * (2 * nu.numel + rows), 0, inner=rext[-1] if rext else 1)

    def lower_fc_bwd(self, u: int, dx_beta: int) -> None:
        nu = self.nodes[u]
        v = nu.ins[0]
        nv = self.nodes[v]
        O, K = self.g.fc_shape(u)
        S = math.prod(nu.sp_ext)
        wslot, dwslot = self.fc_weight_slot(u)
        if u in self.inline_dgrad:
            self.lower_fc_wgrad(u)
            return
        if u in self.epi_bc:
            self.lower_fc_dgrad_bc(u)
            self.lower_fc_wgrad(u)
            return
        dd = self.dgrad_desc[u]
        beta = dx_beta if dd.slot == SLOT_DX else BETA_NONE
        flops = 2 * O * K * S
        # dgrad: D[n,i,s] = sum_o W[o,i] * dL/du[n,o,s]
        name = f"k{len(self.p.kernel_names)}_bwd_dgrad{u}"
        if min(O, K) <= SMALL_FC:

            def body(f):
                c = self.coords_of(f, nv)
                i = f.flatten(c[: nv.nch], nv.ch_ext)
                sp = c[nv.nch :]
                acc = f.fresh("acc")
                f.emit(f"float {acc} = 0.f;")
                o = f.fresh("o")
                f.loop(o, O)
                g = self.grad(f, u, (o,) + sp)
                f.emit(f"{acc} = fmaf(__ldg({f.ptr(wslot)} + {o}*{K} + {i}), {g}, {acc});")
                f.close()
                f.store(dd, c, acc, beta != BETA_NONE)

            self.launch_pointwise(name, nv.numel, body, 1, beta, f"dgrad_small {O}x{K} n{u}->n{v}", 4 * (nu.numel + nv.numel), flops, inner=nv.ext[-1] if nv.ext else 1, node=nv)
        else:
            fa = Fn(self)
            fa.pre = []
            fa.computing = None
            a_expr = f"__ldg({fa.ptr(wslot)} + k*{K} + m)"

            def bfn(f):
                sp = tuple(f.decompose("s", nu.sp_ext))
                return self.grad(f, u, ("k",) + sp)

            def sfn(f, val):
                c = tuple(f.decompose("m", nv.ch_ext)) + tuple(f.decompose("s", nv.sp_ext))
                f.store(dd, c, val, beta != BETA_NONE)

            self.emit_gemm_nk(name, fa, a_expr, bfn, sfn, M=K, K=O, S=S, phase=1, beta=beta, what=f"dgrad {K}x{O}x{S} n{u}->n{v}", nbytes=4 * (nu.numel + nv.numel), flops=flops)
        self.lower_fc_wgrad(u)

    def epi_bc_tile(self, u: int):
        """JT (lhs indices per column tile) when FC u's dgrad can apply the adjoint of
        its input broadcast v = bcast(op)(lhs, rhs) in its TMEM epilogue, else None.
        Needs: v read only by u (dL/dv is exactly the dgrad), a tensor-core dgrad,
        the broadcast core spanning all of v's channel dims (no prefix), and a column
        tile of M replicas x JT lhs indices that fits one MMA (N = M*JT <= 256)."""
        if not EPI_BC or not self.use_tc:
            return None
        nu = self.nodes[u]
        v = nu.ins[0]
        nv = self.nodes[v]
        if v == 0 or nv.op != "bcast" or len(nv.consumers) != 1 or 0 in nv.ins:
            return None
        O, K = self.g.fc_shape(u)
        if min(O, K) <= SMALL_FC or O < 16 or K < 8:
            return None
        at = nv.attr
        if at["cs"] != 0 or at["nr"] != nv.nch or at["M"] < 2:
            return None
        L, M = at["L"], at["M"]
        for jt in (16, 8):
            if L % jt == 0 and (M * jt) % 16 == 0 and M * jt <= 256:
                return jt
        return None

    def lower_fc_dgrad_bc(self, u: int) -> None:
        """dgrad of FC u (tcgen05, persistent) with the input broadcast's adjoint in
        the epilogue.  Columns of dL/dv are packed replica-major per tile — tile ct
        holds k = m*L + ct*JT + jj (m < M, jj < JT) — so each epilogue thread (one
        pixel) owns all M replicas of its JT lhs indices: it writes the rhs edge
        contribution dv * d op/d rhs per column and sums dv * d op/d lhs over the
        replicas in registers (App. A.8 tie split, replica order m = 0..M-1).
        Removes the materialised 9C gradient and the replica-sum pass (SURVEY §7,
        PAPER.md:177: an Unfold never copies)."""
        nu = self.nodes[u]
        v = nu.ins[0]
        nv = self.nodes[v]
        lhs_n, rhs_n = nv.ins
        at = nv.attr
        L, M, op = at["L"], at["M"], at["op"]
        jt = self.epi_bc[u]
        nt = M * jt
        O, K = self.g.fc_shape(u)
        S = math.prod(nu.sp_ext)
        wslot, _ = self.fc_weight_slot(u)
        flops = 2 * O * K * S
        name = f"k{len(self.p.kernel_names)}_bwd_dgrad{u}"
        fa = Fn(self)
        fa.pre = []
        fa.computing = None
        # packed column col of tile ct = col / NT -> k = m*L + ct*JT + jj
        a_expr = f"__ldg({fa.ptr(wslot)} + k*{K} + ((m % {nt}) / {jt}) * {L} + (m / {nt}) * {jt} + (m % {jt}))"

        def bfn(f):
            sp = tuple(f.decompose("s", nu.sp_ext))
            return self.grad(f, u, ("k",) + sp)

        need_r = op in ("min", "max", "mul")
        need_l = op in ("min", "max", "mul")
        ld, rd = self.edge_desc[(v, 0)], self.edge_desc[(v, 1)]

        def mk(fname, rtype, params, body, uni):
            """{fname}_ctx(a, n, s) -> {fname}X: everything of the functor that depends
            only on the thread's pixel (image bases, pixel decomposition, lane
            pointers), built once per tile; {fname}(a, X, params) the per-column rest."""
            f = Fn(self)
            f.pre = []
            f.computing = None
            f.local_slots = fa.local_slots
            f.uniform = set(uni)
            f.ctxh = True
            f.ctx_ok = {"a", "p", "n", "s"}
            ret = body(f)
            mem = f.ctx_vars or [("int", "unused_")]
            out = [f"  struct {fname}X {{ " + " ".join(f"{t} {v};" for t, v in mem) + " };"]
            out.append(f"  static __device__ __forceinline__ {fname}X {fname}_ctx(const CanvasArgs& a, const long long n, const int s) {{")
            out += ["    " + x for x in f.ctx_lines] + [f"    {fname}X X;"] + [f"    X.{v} = {v};" if v != "unused_" else "    X.unused_ = 0;" for _, v in mem] + ["    return X;", "  }"]
            out.append(f"  static __device__ __forceinline__ {rtype} {fname}(const CanvasArgs& a, const {fname}X& X{params}) {{")
            out += [f"    {'float* const' if t == 'float*' else 'const int'} {v} = X.{v};" for t, v in mem if v != "unused_"]
            out += ["    " + x for x in f.pre] + f.lines
            if ret is not None:
                out.append(f"    return {ret};")
            return out + ["  }"]

        def lhs_val(f):
            lc = tuple(f.decompose("j", at["lcore"]))
            sp = tuple(f.decompose("s", nv.sp_ext))
            return self.val(f, lhs_n, lc + sp) if need_l else "0.f"

        def rhs_val(f):
            kk = f.ivar(f"m*{L} + j")
            rc = tuple(f.decompose(kk, at["rcore"]))
            sp = tuple(f.decompose("s", nv.sp_ext))
            return self.val(f, rhs_n, rc + sp) if need_r else "0.f"

        def term(f):
            kk = f.ivar(f"m*{L} + j")
            rc = tuple(f.decompose(kk, at["rcore"]))
            sp = tuple(f.decompose("s", nv.sp_ext))
            dr = f.fvar(_bc_d_rhs(op, "g", "l", "r"))
            f.store(rd, rc + sp, dr, False, pred="ok")
            return f.fvar(_bc_d_lhs(op, "g", "l", "r"))

        def store_l(f):
            lc = tuple(f.decompose("j", at["lcore"]))
            sp = tuple(f.decompose("s", nv.sp_ext))
            f.store(ld, lc + sp, "dl", False, pred="ok")

        nbuf = max(2, min(8, 512 // nt))  # TMEM accumulators in flight (3 at N = 144)
        epi = [f"  static constexpr bool EPI_BC = true, EPI_PF = {'true' if EPI_PREFETCH else 'false'};",
               f"  static constexpr int EPI_M = {M}, EPI_JT = {jt}, EPI_NBUF = {nbuf}, EPI_WPB = {EPI_WPB if jt // EPI_WPB >= 8 else 1};"]
        epi += mk("epi_lhs", "float", ", const int j", lhs_val, {"j"})
        epi += mk("epi_rhs", "float", ", const int m, const int j", rhs_val, {"m", "j"})
        epi += mk("epi_term", "float", ", const int m, const int j, const float g, const float l, const float r, const bool ok", term, {"m", "j"})
        epi += mk("epi_store_l", "void", ", const int j, const float dl, const bool ok", store_l, {"j"})
        self.emit_gemm_nk(name, fa, a_expr, bfn, None, M=K, K=O, S=S, phase=1, beta=BETA_NONE,
                          what=f"dgrad+bcast adjoint {K}x{O}x{S} n{u}->n{lhs_n},n{v}",
                          nbytes=4 * (nu.numel + nv.numel + self.nodes[lhs_n].numel), flops=flops, epi=(nt, epi))

    def lower_fc_wgrad(self, u: int) -> None:
        """dW[o,i] = sum_{n,s} dL/du[n,o,s] * v[n,i,s]."""
        nu = self.nodes[u]
        v = nu.ins[0]
        nv = self.nodes[v]
        O, K = self.g.fc_shape(u)
        S = math.prod(nu.sp_ext)
        _, dwslot = self.fc_weight_slot(u)
        flops = 2 * O * K * S
        name = f"k{len(self.p.kernel_names)}_bwd_wgrad{u}"

        def afn(f):
            sp = tuple(f.decompose("s", nu.sp_ext))
            return self.grad(f, u, ("m",) + sp)

        def bfn2(f):
            ch = tuple(f.decompose("k", nv.ch_ext))
            sp = tuple(f.decompose("s", nv.sp_ext))
            return self.val(f, v, ch + sp)

        self.emit_gemm_wgrad(name, afn, bfn2, O, K, S, dwslot, f"wgrad {O}x{K} over {S}/img n{u}", 4 * (nu.numel + self._input_numel(nu)), flops)

    # -------------------------------------------------------------- assemble
    def finish(self) -> None:
        p = self.p
        nsv = len(p.saved)
        fix = lambda s: p.slot_ws(-1 - s) if s < 0 else s  # noqa: E731
        for L in p.launches:
            L.slots = tuple(fix(s) for s in L.slots)
        header = ("#define CANVAS_RAW_HI 1\n" if os.environ.get("CANVAS_RAW_HI") == "1" else "") + ("#define CANVAS_WGRAD_STACK 0\n" if os.environ.get("CANVAS_WGRAD_STACK") == "0" else "") + '#include "canvas_kernels.cuh"\n'
        p.source = header + "\n".join(self.kernels)
        del nsv


def lower(g: ConcreteGraph, *, c_in: int, c_out: int, stride: int = 1, h_in: int | None = None, w_in: int | None = None, use_tc: bool = True) -> Plan:
    """Build the fwd+bwd plan of one replacement target (SPEC.md:417-425 Fig.-2, App. A.10).

    ``g`` is evaluated at C = min(c_in, c_out) and the *output* resolution;
    ``h_in``/``w_in`` are the full-resolution input extents (stride policy:
    x[..., ::s, ::s] first, fused into the first loads).
    """
    c = g.nodes[0].ext[0]
    if c != min(c_in, c_out) or max(c_in, c_out) % c:
        raise LoweringError(f"C={c} does not replicate to {c_in}->{c_out}")
    h, w = g.nodes[0].ext[1:]
    h_in = h_in if h_in is not None else h * stride
    w_in = w_in if w_in is not None else w * stride
    if -(-h_in // stride) != h or -(-w_in // stride) != w:
        raise LoweringError(f"stride {stride} maps {h_in}x{w_in} to {-(-h_in // stride)}x{-(-w_in // stride)}, kernel is {h}x{w}")
    r = max(c_in, c_out) // c
    mode = "concat" if c_out >= c_in else "sum"
    p = Plan(g, c_in, c_out, stride, h_in, w_in, r, mode)
    hw_in, hw = h_in * w_in, h * w
    if mode == "concat":
        p.y_copy_off = c * hw
        p.dy_copy_off = c * hw
    else:
        p.x_copy_off = c * hw_in
        p.dx_copy_off = c * hw_in
    lw = Lowerer(g, p, use_tc)
    lw.lower_forward()
    lw.lower_backward()
    lw.finish()
    p.fwd_mat = lw.fwd_desc
    return p


# ------------------------------------------------------------------ derivatives
def _bc_d_rhs(op: str, g: str, l: str, r: str) -> str:
    if op == "add":
        return g
    if op == "sub":
        return f"-{g}"
    if op == "mul":
        return f"{g} * {l}"
    if op == "min":
        return f"({r} < {l} ? {g} : ({r} == {l} ? 0.5f * {g} : 0.f))"
    if op == "max":
        return f"({r} > {l} ? {g} : ({r} == {l} ? 0.5f * {g} : 0.f))"
    raise LoweringError(op)


def _bc_d_lhs(op: str, g: str, l: str, r: str) -> str:
    if op in ("add", "sub"):
        return g
    if op == "mul":
        return f"{g} * {r}"
    if op == "min":
        return f"({l} < {r} ? {g} : ({l} == {r} ? 0.5f * {g} : 0.f))"
    if op == "max":
        return f"({l} > {r} ? {g} : ({l} == {r} ? 0.5f * {g} : 0.f))"
    raise LoweringError(op)
