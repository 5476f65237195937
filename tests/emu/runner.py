"""TEST INFRASTRUCTURE: run a lowering Plan on the CPU through host_emu.h.

Mirrors csrc/canvas_runtime.cpp (slot pointers, per-copy offsets, beta
policy, memset records) in Python so the generated functors + schedule can be
checked against the oracle without a GPU.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import subprocess
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
CACHE = Path(tempfile.gettempdir()) / "canvas_emu_cache"


class CanvasArgs(ctypes.Structure):
    _fields_ = [("p", ctypes.c_void_p * 24), ("n", ctypes.c_longlong), ("beta", ctypes.c_int), ("copy", ctypes.c_int)]


def compile_plan(plan) -> ctypes.CDLL:
    src = plan.source.replace('#include "canvas_kernels.cuh"', f'#include "{HERE / "host_emu.h"}"')
    h = hashlib.sha256(src.encode()).hexdigest()[:20]
    CACHE.mkdir(exist_ok=True)
    so = CACHE / f"{h}.so"
    if not so.exists():
        cpp = CACHE / f"{h}.cpp"
        cpp.write_text(src)
        tmp = CACHE / f"{h}.{os.getpid()}.so"
        subprocess.run(["g++", "-O1", "-shared", "-fPIC", "-w", "-ffp-contract=off", str(cpp), "-o", str(tmp)], check=True)
        tmp.replace(so)
    return ctypes.CDLL(str(so))


class EmuPlan:
    def __init__(self, plan):
        self.plan = plan
        self.lib = compile_plan(plan)
        self.fns = [getattr(self.lib, n) for n in plan.kernel_names]
        for f in self.fns:
            f.argtypes = [CanvasArgs]

    PAD = 1 << 14  # NaN guard zone around every scratch tensor: a read outside a tensor poisons the result

    def _alloc(self, rules, n):
        out = []
        for r in rules:
            m = max(1, r.eval(n) // 4)
            buf = np.full(m + 2 * self.PAD, np.nan, np.float32)
            out.append(buf[self.PAD : self.PAD + m])
        return out

    def run(self, phase, x, ws_list, y=None, dy=None, dx=None, dws=None, saved=None):
        """Arrays are float32 numpy, C-contiguous.  ``saved``: list per copy of per-slot arrays."""
        p = self.plan
        n = x.shape[0]
        work = self._alloc(p.ws, n)
        nf = p.n_fc

        def ptr(a, off=0):
            return a.ctypes.data + 4 * off

        for copy in range(p.copies):
            def slot(s):
                if s == 0:
                    return ptr(x, copy * p.x_copy_off)
                if s == 1:
                    return ptr(y, copy * p.y_copy_off)
                if s == 2:
                    return ptr(dy, copy * p.dy_copy_off)
                if s == 3:
                    return ptr(dx, copy * p.dx_copy_off)
                s -= 4
                if s < nf:
                    return ptr(ws_list[copy * nf + s])
                s -= nf
                if s < nf:
                    return ptr(dws[copy * nf + s])
                s -= nf
                if s < len(p.saved):
                    return ptr(saved[copy][s])
                s -= len(p.saved)
                return ptr(work[s])

            for L in p.launches:
                if L.phase != phase:
                    continue
                if L.kind == "memset":
                    if copy == 0:
                        ctypes.memset(slot(L.memset_slot), 0, L.memset_size.eval(n))
                    continue
                a = CanvasArgs()
                for i, s in enumerate(L.slots):
                    a.p[i] = slot(s)
                a.n = n
                a.beta = int(L.beta == 2 or (L.beta == 1 and copy > 0))
                a.copy = copy
                self.fns[L.kernel](a)

    def forward(self, x, weights):
        p = self.plan
        n = x.shape[0]
        ho, wo = p.graph.nodes[p.graph.output].ext[1:]
        y = np.zeros((n, p.c_out, ho, wo), np.float32)
        saved = [self._alloc(p.saved, n) for _ in range(p.copies)]
        self.run(0, x, weights, y=y, saved=saved)
        return y, saved

    def backward(self, x, weights, saved, dy):
        dx = np.full(x.shape, np.nan, np.float32) if self.plan.stride == 1 else np.zeros_like(x)
        dws = [np.full(w.shape, np.nan, np.float32) for w in weights]
        self.run(1, x, weights, dy=dy, dx=dx, dws=dws, saved=saved)
        return dx, dws
