"""BN post-pass of a replaced conv, on ``libcanvas_post.so`` (include/canvas_post.h).

SPEC.md:658 gives ``build_module`` an optional BatchNorm after the kernel, and
in a network every replaced ``nn.Conv2d`` is followed by the backbone's own
BatchNorm2d.  ``FusedBatchNorm2d`` is a drop-in
``nn.BatchNorm2d`` (same parameters, buffers and state_dict) whose training
forward/backward run as two hand-written HBM passes each, with the block's
ReLU and residual add fused in.  ``fuse_backbone`` rewires torchvision
ResNets so that ``conv -> bn -> (+identity) -> relu`` becomes
``conv -> FusedBatchNorm2d(relu, residual)``.

There is no fallback: a CUDA tensor without the library raises.  Eval mode
and CPU tensors use ``torch.nn.functional.batch_norm`` (they are not on the
training hot path).
"""

from __future__ import annotations

import ctypes
import threading
import types
from pathlib import Path

import torch
import torch.nn.functional as F
from torch import nn

LIB_PATH = Path(__file__).resolve().parent / "libcanvas_post.so"
ABI_VERSION = 2
_lib = None
_lock = threading.Lock()


class PostError(RuntimeError):
    pass


def load_library() -> ctypes.CDLL:
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise PostError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(str(LIB_PATH))
        c = ctypes
        lib.canvas_post_abi_version.restype = c.c_int
        lib.canvas_post_last_error.restype = c.c_char_p
        lib.canvas_bn_workspace.restype = c.c_size_t
        lib.canvas_bn_workspace.argtypes = [c.c_int64] * 3
        p = c.c_void_p
        lib.canvas_bn_forward.argtypes = [c.c_int64] * 3 + [p] * 9 + [c.c_float, c.c_float, c.c_int, p, p, p]
        lib.canvas_bn_backward.argtypes = [c.c_int64] * 3 + [p] * 11 + [c.c_int, p, p]
        lib.canvas_maxpool2d_forward.argtypes = [c.c_int64] * 4 + [c.c_int] * 3 + [p] * 4
        lib.canvas_maxpool2d_backward.argtypes = [c.c_int64] * 4 + [c.c_int] * 3 + [p] * 4
        if lib.canvas_post_abi_version() != ABI_VERSION:
            raise PostError("libcanvas_post.so ABI version mismatch")
        _lib = lib
        return lib


def _check(rc: int) -> None:
    if rc != 0:
        raise PostError(f"canvas_post C-ABI error {rc}: {load_library().canvas_post_last_error().decode(errors='replace')}")


def _ptr(t):
    return None if t is None else t.data_ptr()


class _BnFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, residual, weight, bias, running_mean, running_var, momentum, eps, relu):
        lib = load_library()
        x = x.contiguous()
        n, c = x.shape[0], x.shape[1]
        hw = x.numel() // max(1, n * c)
        if residual is not None:
            residual = residual.contiguous()
            if residual.shape != x.shape:
                raise ValueError(f"residual shape {tuple(residual.shape)} != {tuple(x.shape)}")
        y = torch.empty_like(x)
        mean = torch.empty(c, device=x.device, dtype=torch.float32)
        invstd = torch.empty_like(mean)
        # ReLU mask bytes (y > 0): the backward reads 1 byte instead of y's 4 per element
        mask = torch.empty(x.shape, device=x.device, dtype=torch.uint8) if relu else None
        ws = torch.empty(lib.canvas_bn_workspace(n, c, hw), device=x.device, dtype=torch.uint8)
        st = torch.cuda.current_stream(x.device).cuda_stream
        _check(lib.canvas_bn_forward(n, c, hw, _ptr(x), _ptr(residual), _ptr(y), _ptr(weight), _ptr(bias), _ptr(running_mean), _ptr(running_var), _ptr(mean), _ptr(invstd), float(momentum), float(eps), int(relu), _ptr(mask), _ptr(ws), st))
        ctx.relu = bool(relu)
        ctx.has_res = residual is not None
        ctx.save_for_backward(x, mask, weight, mean, invstd)
        return y

    @staticmethod
    def backward(ctx, dy):
        lib = load_library()
        x, mask, weight, mean, invstd = ctx.saved_tensors
        dy = dy.contiguous()
        n, c = x.shape[0], x.shape[1]
        hw = x.numel() // max(1, n * c)
        dx = torch.empty_like(x)
        dres = torch.empty_like(x) if ctx.has_res and ctx.relu else None
        dw = torch.empty_like(weight)
        db = torch.empty_like(weight)
        ws = torch.empty(lib.canvas_bn_workspace(n, c, hw), device=x.device, dtype=torch.uint8)
        st = torch.cuda.current_stream(x.device).cuda_stream
        _check(lib.canvas_bn_backward(n, c, hw, _ptr(x), None, _ptr(mask), _ptr(dy), _ptr(weight), _ptr(mean), _ptr(invstd), _ptr(dx), _ptr(dres), _ptr(dw), _ptr(db), int(ctx.relu), _ptr(ws), st))
        if ctx.has_res and not ctx.relu:
            dres = dy
        return dx, dres, dw, db, None, None, None, None, None


class FusedBatchNorm2d(nn.BatchNorm2d):
    """``nn.BatchNorm2d`` (affine, fp32, NCHW) whose training pass is the fused
    native post-pass: ``y = relu?(bn(x) + residual?)``."""

    def __init__(self, num_features, eps=1e-5, momentum=0.1, relu: bool = False, **kw):
        super().__init__(num_features, eps=eps, momentum=momentum, **kw)
        self.relu = relu

    @classmethod
    def from_bn(cls, bn: nn.BatchNorm2d, relu: bool = False) -> "FusedBatchNorm2d":
        if not bn.affine or bn.momentum is None:
            raise ValueError("FusedBatchNorm2d needs an affine BatchNorm2d with a momentum")
        new = cls(bn.num_features, eps=bn.eps, momentum=bn.momentum, relu=relu, track_running_stats=bn.track_running_stats)
        new.load_state_dict(bn.state_dict())
        return new.to(bn.weight.device)

    def forward(self, x: torch.Tensor, residual: torch.Tensor | None = None) -> torch.Tensor:
        if not (self.training and x.is_cuda):
            y = super().forward(x)
            if residual is not None:
                y = y + residual
            return F.relu(y) if self.relu else y
        if x.dtype != torch.float32 or x.dim() != 4:
            raise TypeError("FusedBatchNorm2d: fp32 NCHW input expected")
        track = self.track_running_stats and self.running_mean is not None
        if track:
            self.num_batches_tracked.add_(1)
        return _BnFn.apply(x, residual, self.weight, self.bias, self.running_mean if track else None, self.running_var if track else None, self.momentum, self.eps, self.relu)

    def extra_repr(self) -> str:
        return super().extra_repr() + f", relu={self.relu}"


class _PoolFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, k, s, p):
        lib = load_library()
        x = x.contiguous()
        n, c, h, w = x.shape
        oh, ow = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
        y = torch.empty((n, c, oh, ow), device=x.device, dtype=x.dtype)
        idx = torch.empty((n, c, oh, ow), device=x.device, dtype=torch.uint8)
        st = torch.cuda.current_stream(x.device).cuda_stream
        _check(lib.canvas_maxpool2d_forward(n, c, h, w, k, s, p, x.data_ptr(), y.data_ptr(), idx.data_ptr(), st))
        ctx.geo = (n, c, h, w, k, s, p)
        ctx.save_for_backward(idx)
        ctx.mark_non_differentiable(idx)
        return y

    @staticmethod
    def backward(ctx, dy):
        lib = load_library()
        (idx,) = ctx.saved_tensors
        n, c, h, w, k, s, p = ctx.geo
        dy = dy.contiguous()
        dx = torch.empty((n, c, h, w), device=dy.device, dtype=dy.dtype)
        st = torch.cuda.current_stream(dy.device).cuda_stream
        _check(lib.canvas_maxpool2d_backward(n, c, h, w, k, s, p, dy.data_ptr(), idx.data_ptr(), dx.data_ptr(), st))
        return dx, None, None, None


class FusedMaxPool2d(nn.MaxPool2d):
    """``nn.MaxPool2d`` (square, no dilation, floor mode, fp32) on
    libcanvas_post: byte argmax, deterministic gather backward."""

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        if not x.is_cuda:
            return super().forward(x)
        if x.dtype != torch.float32 or x.dim() != 4:
            raise TypeError("FusedMaxPool2d: fp32 NCHW input expected")
        return _PoolFn.apply(x, self.kernel_size, self.stride, self.padding)

    @classmethod
    def from_pool(cls, m: nn.MaxPool2d) -> "FusedMaxPool2d":
        k, s, p = (m.kernel_size, m.stride, m.padding)
        if not all(isinstance(v, int) for v in (k, s, p)) or m.dilation not in (1, (1, 1)) or m.ceil_mode or m.return_indices:
            raise ValueError("FusedMaxPool2d: square window, int stride/padding, no dilation / ceil mode / indices")
        return cls(k, s, p)


def _basic_forward(self, x):
    identity = x if self.downsample is None else self.downsample(x)
    out = self.bn1(self.conv1(x))
    return self.bn2(self.conv2(out), identity)


def _bottleneck_forward(self, x):
    identity = x if self.downsample is None else self.downsample(x)
    out = self.bn1(self.conv1(x))
    out = self.bn2(self.conv2(out))
    return self.bn3(self.conv3(out), identity)


def fuse_backbone(model: nn.Module) -> int:
    """Rewire a torchvision ResNet so each BN runs as a fused post-pass.

    Stem ``bn1 -> relu`` and the block tails ``bn -> (+identity) -> relu`` fuse;
    downsample BNs stay plain (no activation); the stem max-pool runs on the
    native pool kernels.  Returns the number of fused BNs.
    """
    from torchvision.models.resnet import BasicBlock, Bottleneck, ResNet

    count = 0

    def swap(parent, name, relu):
        nonlocal count
        bn = getattr(parent, name)
        if isinstance(bn, nn.BatchNorm2d) and not isinstance(bn, FusedBatchNorm2d):
            setattr(parent, name, FusedBatchNorm2d.from_bn(bn, relu=relu))
            count += 1

    for m in list(model.modules()):
        if isinstance(m, ResNet) or getattr(m, "_canvas_stem", False):
            swap(m, "bn1", True)
            m.relu = nn.Identity()
            if isinstance(getattr(m, "maxpool", None), nn.MaxPool2d) and not isinstance(m.maxpool, FusedMaxPool2d):
                m.maxpool = FusedMaxPool2d.from_pool(m.maxpool)
        elif isinstance(m, BasicBlock):
            swap(m, "bn1", True)
            swap(m, "bn2", True)
            m.forward = types.MethodType(_basic_forward, m)
        elif isinstance(m, Bottleneck):
            swap(m, "bn1", True)
            swap(m, "bn2", True)
            swap(m, "bn3", True)
            m.forward = types.MethodType(_bottleneck_forward, m)
        if getattr(m, "downsample", None) is not None and isinstance(m.downsample, nn.Sequential):
            for i, sub in enumerate(m.downsample):
                if isinstance(sub, nn.BatchNorm2d) and not isinstance(sub, FusedBatchNorm2d):
                    m.downsample[i] = FusedBatchNorm2d.from_bn(sub, relu=False)
                    count += 1
    return count
