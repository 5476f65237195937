"""Build the native pieces in-tree (they travel to the GPU box with the repo).

1. ``csrc/kernels/canvas_kernels.cuh`` (hand-written templates) is embedded
   as a string into ``libcanvas_b200.so`` so NVRTC can instantiate it per plan.
2. ``libcanvas_b200.so`` (C ABI, include/canvas_b200.h) is built with g++; it
   dlopens the CUDA driver and NVRTC at first use.
   ``libcanvas_post.so`` (include/canvas_post.h, the fused BN post-pass) is
   compiled by nvcc for sm_100a from ``csrc/post_kernels.cu``.
3. Build check: the pinned kernels (zoo.py) are lowered and their generated
   functors compiled together with the templates by ``nvcc`` for sm_100a
   (``-gencode arch=compute_100a,code=sm_100a -lineinfo``) into
   ``build/pinned_sm100a.cubin`` — the same code NVRTC produces on the box,
   checked here without a GPU (register/spill report with ``verbose``).
"""

from __future__ import annotations

import os
import re
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libcanvas_b200.so"
POST_LIB = PKG / "libcanvas_post.so"
BUILD = ROOT / "build"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _run(cmd: list[str]) -> str:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(f"command failed ({r.returncode}): {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r.stdout + r.stderr


def embed_templates() -> Path:
    src = (CSRC / "kernels" / "canvas_kernels.cuh").read_text()
    if ')CNVS"' in src:
        raise RuntimeError("template source contains the raw-string delimiter")
    out = CSRC / "canvas_kernels_embed.inc"
    text = 'R"CNVS(' + src + ')CNVS"\n'
    if not out.exists() or out.read_text() != text:
        out.write_text(text)
    return out


def build_lib() -> Path:
    embed_templates()
    srcs = [CSRC / "canvas_runtime.cpp"]
    newest = max(p.stat().st_mtime for p in srcs + [CSRC / "canvas_kernels_embed.inc", ROOT / "include" / "canvas_b200.h"])
    if LIB.exists() and LIB.stat().st_mtime >= newest:
        return LIB
    tmp = LIB.with_suffix(".so.tmp")
    _run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-Wall", "-I", str(ROOT / "include"), *map(str, srcs), "-o", str(tmp), "-ldl", "-lpthread"])
    tmp.replace(LIB)
    return LIB


def build_post() -> Path:
    """libcanvas_post.so: BN post-pass kernels (include/canvas_post.h), nvcc for sm_100a."""
    src = CSRC / "post_kernels.cu"
    hdr = ROOT / "include" / "canvas_post.h"
    if POST_LIB.exists() and POST_LIB.stat().st_mtime >= max(src.stat().st_mtime, hdr.stat().st_mtime):
        return POST_LIB
    tmp = POST_LIB.with_suffix(".so.tmp")
    _run([NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-I", str(ROOT / "include"), str(src), "-o", str(tmp)])
    tmp.replace(POST_LIB)
    return POST_LIB


def pinned_source() -> str:
    """Generated functors of every pinned kernel at config-1 shapes, one file."""
    from . import zoo
    from .executor import plan_for

    from .dense_conv import lower_conv2d

    plans = [(name, plan_for(text, c_in=64, c_out=64, h=56, w=56, k=3, g=4)) for name, text in zoo.ALL.items()]
    # dense backbone convs (ResNet stem 7x7/2 and a strided 1x1 downsample with dgrad)
    plans.append(("stem", lower_conv2d(3, 64, 7, 2, 3, 224, 224, False)))
    plans.append(("down", lower_conv2d(64, 128, 1, 2, 0, 56, 56, True)))
    parts = []
    for name, p in plans:
        src = p.source.replace('#include "canvas_kernels.cuh"\n', "")
        # kernel names are per-plan; prefix them so one translation unit holds all
        pat = re.compile(r"\b((?:" + "|".join(map(re.escape, p.kernel_names)) + r")(?:_F)?)\b")
        src = pat.sub(lambda m: f"{name}_{m.group(1)}", src)
        parts.append(f"// ---- {name}\n" + src)
    return '#include "canvas_kernels.cuh"\n' + "\n".join(parts)


def build_check(verbose: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    cu = BUILD / "pinned_sm100a.cu"
    cu.write_text(pinned_source())
    out = BUILD / "pinned_sm100a.cubin"
    cmd = [NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-cubin", "-I", str(CSRC / "kernels"), "-diag-suppress", "177", str(cu), "-o", str(out)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    log = _run(cmd)
    if verbose:
        print(log, file=sys.stderr)
    return out


def build(verbose: bool = False) -> None:
    build_lib()
    build_post()
    build_check(verbose)


if __name__ == "__main__":
    build(verbose="-v" in sys.argv)
    print(LIB)
