"""Host side of the executor: IR text -> plan -> libcanvas_b200.so (ctypes).

``plan_for`` is the reference-facing entry (SPEC.md:637-645 ``build_module``
takes the kernel IR + a target assignment): it parses ``canvas-ir v1`` with
the reference-compatible front end (ref ir.py:97-169), evaluates the target
assignment (ref ir.py:48-53, C = min(Cin, Cout)), solves free variables
(constraint_solver.proportional_values) and lowers the concrete graph.

``DevicePlan`` owns one ``canvas_plan*`` from the C ABI and runs forward /
backward on torch tensors (torch is only the allocator/stream provider here).
There is no CPU or eager fallback: if the library or a B200 is missing,
construction raises.
"""

from __future__ import annotations

import collections
import ctypes
import functools
import hashlib
import threading
from pathlib import Path

from .canvas import ir as cir
from .canvas.constraint_solver import proportional_values
from .canvas.shape_algebra import Assignment
from .graph import build_graph
from .lowering import Plan, lower

LIB_PATH = Path(__file__).resolve().parent / "libcanvas_b200.so"


class CanvasError(RuntimeError):
    """A C-ABI call failed (message from canvas_last_error)."""


def solve_target(ir_text: str, *, c_in: int, c_out: int, h: int, w: int, k: int = 3, g: int = 4, stride: int = 1, xs: dict | None = None):
    """(template, Assignment) of one replacement target, at the output resolution."""
    t = cir.parse(ir_text).template
    ho, wo = -(-h // stride), -(-w // stride)
    consts = {"C": min(c_in, c_out), "G": g, "H": ho, "W": wo, "KH": k, "KW": k}
    dyn = dict(xs) if xs is not None else proportional_values(t, consts)
    return t, Assignment(consts, dyn)


@functools.lru_cache(maxsize=256)
def _plan_cached(ir_text, c_in, c_out, h, w, k, g, stride, xs_items) -> Plan:
    t, a = solve_target(ir_text, c_in=c_in, c_out=c_out, h=h, w=w, k=k, g=g, stride=stride, xs=dict(xs_items) if xs_items is not None else None)
    return lower(build_graph(t, a), c_in=c_in, c_out=c_out, stride=stride, h_in=h, w_in=w)


def plan_for(ir_text: str, *, c_in: int, c_out: int, h: int, w: int, k: int = 3, g: int = 4, stride: int = 1, xs: dict | None = None) -> Plan:
    """Lower one kernel for one conv target (input resolution h x w)."""
    xi = tuple(sorted(xs.items())) if xs is not None else None
    return _plan_cached(ir_text, c_in, c_out, h, w, k, g, stride, xi)


# ----------------------------------------------------------------------- C ABI
_lib = None
_lib_lock = threading.Lock()


def load_library() -> ctypes.CDLL:
    """Load libcanvas_b200.so (raises if it was not built — no fallback)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise CanvasError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(str(LIB_PATH))
        c = ctypes
        lib.canvas_abi_version.restype = c.c_int
        lib.canvas_last_error.restype = c.c_char_p
        lib.canvas_plan_create.argtypes = [c.c_void_p, c.c_size_t, c.c_int, c.POINTER(c.c_void_p)]
        lib.canvas_plan_destroy.argtypes = [c.c_void_p]
        lib.canvas_plan_query.argtypes = [c.c_void_p, c.c_int64, c.POINTER(c.c_size_t), c.POINTER(c.c_size_t), c.POINTER(c.c_size_t)]
        lib.canvas_plan_launches.argtypes = [c.c_void_p, c.c_int]
        lib.canvas_forward.argtypes = [c.c_void_p, c.c_int64, c.c_void_p, c.c_void_p, c.c_int, c.c_void_p, c.c_void_p, c.c_void_p, c.c_void_p]
        lib.canvas_plan_profile.argtypes = [c.c_void_p, c.c_int, c.c_void_p, c.c_int]
        lib.canvas_plan_profile_count.argtypes = [c.c_void_p, c.c_int]
        lib.canvas_plan_profile_count.restype = c.c_int64
        lib.canvas_backward.argtypes = [c.c_void_p, c.c_int64, c.c_void_p, c.c_void_p, c.c_int, c.c_void_p, c.c_void_p, c.c_void_p, c.c_void_p, c.c_void_p, c.c_void_p]
        _lib = lib
        return lib


def _check(rc: int) -> None:
    if rc != 0:
        msg = load_library().canvas_last_error().decode(errors="replace")
        raise CanvasError(f"canvas C-ABI error {rc}: {msg}")


class DevicePlan:
    """A compiled plan on one CUDA device (``canvas_plan*``)."""

    def __init__(self, plan: Plan, device: int):
        self.plan = plan
        self.device = device
        self.lib = load_library()
        blob = plan.blob()
        h = ctypes.c_void_p()
        _check(self.lib.canvas_plan_create(blob, len(blob), device, ctypes.byref(h)))
        self.handle = h
        self.n_fc_total = plan.n_fc * plan.copies
        self._ptr_cache: dict = {}

    def __del__(self):  # pragma: no cover - interpreter teardown order
        try:
            if getattr(self, "handle", None):
                self.lib.canvas_plan_destroy(self.handle)
        except Exception:
            pass

    def sizes(self, batch: int) -> tuple[int, int]:
        """(saved bytes, backward workspace bytes)."""
        f, s, b = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
        _check(self.lib.canvas_plan_query(self.handle, batch, ctypes.byref(f), ctypes.byref(s), ctypes.byref(b)))
        return s.value, b.value

    def launches(self, phase: int) -> int:
        return self.lib.canvas_plan_launches(self.handle, phase)

    def record_index(self, pattern: str) -> int:
        """Index of the first launch record whose kernel name contains ``pattern``."""
        for i, L in enumerate(self.plan.launches):
            if L.kind == "kernel" and pattern in L.name:
                return i
        raise KeyError(pattern)

    def profile(self, record: int, events) -> None:
        """Record ``events`` (list of (start, end) torch.cuda.Event) around launches of ``record``."""
        arr = (ctypes.c_void_p * max(1, 2 * len(events)))()
        for i, (a, b) in enumerate(events):
            arr[2 * i] = a.cuda_event
            arr[2 * i + 1] = b.cuda_event
        _check(self.lib.canvas_plan_profile(self.handle, record, arr, len(events)))

    def profile_count(self, record: int) -> int:
        return self.lib.canvas_plan_profile_count(self.handle, record)

    @staticmethod
    def _ptr_array(tensors) -> ctypes.Array:
        arr = (ctypes.c_void_p * max(1, len(tensors)))()
        for i, t in enumerate(tensors):
            arr[i] = t.data_ptr()
        return arr

    def forward(self, x, weights, y, saved, stream: int) -> None:
        w = self._ptr_array(weights)
        _check(self.lib.canvas_forward(self.handle, x.shape[0], x.data_ptr(), w, len(weights), y.data_ptr(), saved.data_ptr() if saved is not None else None, None, stream))

    def backward(self, x, weights, saved, dy, dx, dws, workspace, stream: int) -> None:
        w = self._ptr_array(weights)
        dw = self._ptr_array(dws)
        _check(
            self.lib.canvas_backward(
                self.handle, x.shape[0], x.data_ptr(), w, len(weights), saved.data_ptr() if saved is not None else None, dy.data_ptr(), dx.data_ptr(), dw, workspace.data_ptr() if workspace is not None else None, stream
            )
        )


_DEV_PLAN_CACHE = 512  # compiled plans kept alive by the cache (LRU); callers may hold more
_dev_plans: "collections.OrderedDict[tuple, DevicePlan]" = collections.OrderedDict()
_dev_lock = threading.Lock()


def device_plan(plan: Plan, device: int) -> DevicePlan:
    """The compiled plan of ``plan`` on ``device``, shared by every caller with the
    same plan content (keyed by the blob digest, not the Python object).  The
    cache is a bounded LRU: an evicted plan is destroyed (and its module unloaded
    by the runtime) once no caller holds it, so long searches stay bounded."""
    blob = plan.blob()
    key = (hashlib.sha1(blob).hexdigest(), device)
    with _dev_lock:
        dp = _dev_plans.get(key)
        if dp is not None:
            _dev_plans.move_to_end(key)
            return dp
    dp = DevicePlan(plan, device)  # NVRTC compile outside the lock: plans build in parallel
    with _dev_lock:
        got = _dev_plans.setdefault(key, dp)
        _dev_plans.move_to_end(key)
        while len(_dev_plans) > _DEV_PLAN_CACHE:
            _dev_plans.popitem(last=False)
        return got
