"""Standard (dense) convolutions of the backbone on the same tcgen05 GEMM
templates as the Canvas FCs.

The ResNet stem (3 -> 64, 7x7, stride 2, pad 3) is not a replacement target
(3 does not divide 64) and stays a plain convolution; on cuDNN in fp32 it took
~10% of the Canvas-ResNet-18 step.  Here it is an implicit GEMM: the operand
B(n, k, s) = x[n, c, oh*S + kh - P, ow*S + kw - P] (k = (c, kh, kw), zero
outside the image) is produced on the fly by the producer warps of
``canvas::tc_gemm_pix`` / ``tc_gemm_pix_persistent`` and the weight gradient
by ``canvas::tc_gemm_wgrad`` — 3xTF32, fp32-accurate, deterministic.  The
input gradient (when the input requires it, e.g. the strided 1x1 downsample
convs) is a third GEMM over K' = (C_out, kh, kw) whose operand gathers dy at
((ih + P - kh) / S, (iw + P - kw) / S) where divisible (col2im as a gather).

``lower_conv2d`` builds a plan blob for ``libcanvas_b200.so`` (one FC slot =
the [C_out, C_in*K*K] weight, i.e. ``nn.Conv2d.weight`` flattened); ``TcConv2d``
is a drop-in ``nn.Conv2d`` using it.
"""

from __future__ import annotations

import functools

import torch
from torch import nn

from .lowering import BETA_NONE, SLOT_DY, SLOT_X, SLOT_Y, Fn, Lowerer, Plan


class _DenseGraph:
    """Stand-in for ConcreteGraph: one FC (the conv weight)."""

    def __init__(self, c_out: int, k: int):
        self.fc_nodes = [0]
        self._shape = (c_out, k)

    def fc_shape(self, v: int):
        return self._shape


@functools.lru_cache(maxsize=32)
def lower_conv2d(c_in: int, c_out: int, k: int, stride: int, pad: int, h_in: int, w_in: int, dgrad: bool = False) -> Plan:
    ho = (h_in + 2 * pad - k) // stride + 1
    wo = (w_in + 2 * pad - k) // stride + 1
    K, S, kk = c_in * k * k, ho * wo, k * k
    p = Plan(_DenseGraph(c_out, K), c_in, c_out, stride, h_in, w_in, 1, "concat")
    lw = Lowerer.bare(p)

    def im2col(f: Fn) -> str:
        xp = f.ptr(SLOT_X)
        f.emit(f"const int c_ = k / {kk}; const int r_ = k - c_ * {kk}; const int kh_ = r_ / {k}; const int kw_ = r_ - kh_ * {k};")
        f.emit(f"const int oh_ = s / {wo}; const int ow_ = s - oh_ * {wo};")
        f.emit(f"const int ih_ = oh_ * {stride} + kh_ - {pad}; const int iw_ = ow_ * {stride} + kw_ - {pad};")
        f.emit(f"const float x_ = ((unsigned)ih_ < {h_in}u && (unsigned)iw_ < {w_in}u) ? __ldg({xp} + (long long)n * {c_in * h_in * w_in} + (c_ * {h_in} + ih_) * {w_in} + iw_) : 0.f;")
        return "x_"

    def store(f: Fn, val: str) -> None:
        f.emit(f"*({f.ptr(SLOT_Y)} + (long long)n * {c_out * S} + m * {S} + s) = {val};")

    fa = Fn(lw)
    fa.pre = []
    fa.computing = None
    a_expr = f"__ldg({fa.ptr(p.slot_w(0))} + m * {K} + k)"
    flops = 2 * c_out * K * S
    lw.emit_gemm_nk("k0_fwd_conv", fa, a_expr, im2col, store, M=c_out, K=K, S=S, phase=0, beta=BETA_NONE, what=f"conv {c_out}x{K}x{S} k{k}s{stride}", nbytes=4 * (c_in * h_in * w_in + c_out * S), flops=flops)

    def dy(f: Fn) -> str:
        return f.fvar(f"__ldg({f.ptr(SLOT_DY)} + (long long)n * {c_out * S} + m * {S} + s)")

    if dgrad and k == 1 and pad == 0 and stride > 1:
        # strided 1x1 (ResNet downsample): only the (stride-aligned) sampled inputs
        # get gradient — dx[n, c, oh*S, ow*S] = sum_m W[m, c] dy[n, m, oh, ow].  The GEMM
        # runs over the H_o*W_o sampled pixels only and its epilogue also writes the
        # zeros of the S*S - 1 skipped positions (no memset, no zero MMA work).
        from .lowering import SLOT_DX

        def dy_plain(f: Fn) -> str:
            return f.fvar(f"__ldg({f.ptr(SLOT_DY)} + (long long)n * {c_out * S} + k * {S} + s)")

        def store_dx_strided(f: Fn, val: str) -> None:
            f.emit(f"const int oh_ = s / {wo}; const int ow_ = s - oh_ * {wo};")
            f.emit(f"float* const d_ = {f.ptr(SLOT_DX)} + (long long)n * {c_in * h_in * w_in} + m * {h_in * w_in} + oh_ * {stride * w_in} + ow_ * {stride};")
            for dh in range(stride):
                for dw in range(stride):
                    conds = []
                    if (ho - 1) * stride + dh >= h_in:
                        conds.append(f"oh_ * {stride} + {dh} < {h_in}")
                    if (wo - 1) * stride + dw >= w_in:
                        conds.append(f"ow_ * {stride} + {dw} < {w_in}")
                    st = f"d_[{dh * w_in + dw}] = {val if dh == 0 and dw == 0 else '0.f'};"
                    f.emit(f"if ({' && '.join(conds)}) {st}" if conds else st)

        fd = Fn(lw)
        fd.pre = []
        fd.computing = None
        a_d = f"__ldg({fd.ptr(p.slot_w(0))} + k * {K} + m)"
        lw.emit_gemm_nk(f"k{len(p.kernel_names)}_bwd_dgrad_conv", fd, a_d, dy_plain, store_dx_strided, M=c_in, K=c_out, S=S, phase=1, beta=BETA_NONE, what=f"dgrad conv 1x1/{stride} {c_in}x{c_out}x{S}", nbytes=4 * (c_out * S + c_in * h_in * w_in), flops=2 * c_in * c_out * S)
    elif dgrad:
        # dx[n, c, ih, iw] = sum_{m, kh, kw} W[m, c, kh, kw] dy[n, m, (ih+P-kh)/S, (iw+P-kw)/S]
        Kd, Sd = c_out * kk, h_in * w_in

        def col2im(f: Fn) -> str:
            dp = f.ptr(SLOT_DY)
            f.emit(f"const int m_ = k / {kk}; const int r_ = k - m_ * {kk}; const int kh_ = r_ / {k}; const int kw_ = r_ - kh_ * {k};")
            f.emit(f"const int ih_ = s / {w_in}; const int iw_ = s - ih_ * {w_in};")
            f.emit(f"const int th_ = ih_ + {pad} - kh_; const int tw_ = iw_ + {pad} - kw_;")
            f.emit(f"const int oh_ = th_ / {stride}; const int ow_ = tw_ / {stride};")
            f.emit(f"const bool in_ = th_ >= 0 && tw_ >= 0 && th_ - oh_ * {stride} == 0 && tw_ - ow_ * {stride} == 0 && oh_ < {ho} && ow_ < {wo};")
            f.emit(f"const float g_ = in_ ? __ldg({dp} + (long long)n * {c_out * S} + (m_ * {ho} + oh_) * {wo} + ow_) : 0.f;")
            return "g_"

        def store_dx(f: Fn, val: str) -> None:
            from .lowering import SLOT_DX

            f.emit(f"*({f.ptr(SLOT_DX)} + (long long)n * {c_in * Sd} + m * {Sd} + s) = {val};")

        fd = Fn(lw)
        fd.pre = []
        fd.computing = None
        a_d = f"__ldg({fd.ptr(p.slot_w(0))} + (k / {kk}) * {K} + m * {kk} + (k % {kk}))"
        lw.emit_gemm_nk(f"k{len(p.kernel_names)}_bwd_dgrad_conv", fd, a_d, col2im, store_dx, M=c_in, K=Kd, S=Sd, phase=1, beta=BETA_NONE, what=f"dgrad conv {c_in}x{Kd}x{Sd}", nbytes=4 * (c_out * S + c_in * Sd), flops=2 * c_in * Kd * Sd)
    # wgrad orientation: MMA rows (padded to 128) take one operand, the N side
    # (padded to 16) the other.  Put the rows on whichever side pads less overall;
    # at the stem (K = 147, C_out = 64) that moves the im2col gathers from 256
    # produced rows to 160 (dy takes the 128 padded rows: plain loads).
    rows = lambda j, m: -(-j // 128) * 128 + -(-m // 16) * 16  # noqa: E731
    wname = f"k{len(p.kernel_names)}_bwd_wgrad_conv"
    wwhat = f"wgrad conv {c_out}x{K} over {S}/img"
    if rows(c_out, K) < rows(K, c_out):

        def im2col_m(f: Fn) -> str:  # the im2col operand indexed by the A-row variable m
            f.emit("const int k = m;")
            return im2col(f)

        def dy_k(f: Fn) -> str:
            return f.fvar(f"__ldg({f.ptr(SLOT_DY)} + (long long)n * {c_out * S} + k * {S} + s)")

        lw.emit_gemm_wgrad(wname, im2col_m, dy_k, K, c_out, S, p.slot_dw(0), wwhat + " (transposed)", 4 * (c_in * h_in * w_in + c_out * S), flops, trans=True)
    else:
        lw.emit_gemm_wgrad(wname, dy, im2col, c_out, K, S, p.slot_dw(0), wwhat, 4 * (c_in * h_in * w_in + c_out * S), flops)
    lw.finish()
    return p


class _ConvFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, mod, x, w):
        from .executor import device_plan

        x = x.contiguous()
        n, _, h, wd = x.shape
        need_dx = ctx.needs_input_grad[1]
        dp = device_plan(lower_conv2d(mod.in_channels, mod.out_channels, mod.kernel_size[0], mod.stride[0], mod.padding[0], h, wd, need_dx), x.device.index or 0)
        ho = (h + 2 * mod.padding[0] - mod.kernel_size[0]) // mod.stride[0] + 1
        wo = (wd + 2 * mod.padding[1] - mod.kernel_size[1]) // mod.stride[1] + 1
        y = torch.empty((n, mod.out_channels, ho, wo), device=x.device, dtype=torch.float32)
        saved_b, ws_b = dp.sizes(n)
        saved = torch.empty(max(saved_b, 1), device=x.device, dtype=torch.uint8)
        wf = w.contiguous().view(mod.out_channels, -1)
        dp.forward(x, [wf], y, saved, torch.cuda.current_stream(x.device).cuda_stream)
        ctx.dp, ctx.ws_b = dp, ws_b
        ctx.save_for_backward(x, saved, wf)
        ctx.wshape = w.shape
        ctx.x_grad = ctx.needs_input_grad[1]
        return y

    @staticmethod
    def backward(ctx, dy):
        x, saved, wf = ctx.saved_tensors
        dy = dy.contiguous()
        dw = torch.empty_like(wf)
        dx = torch.empty_like(x) if ctx.x_grad else dy  # dy: never written when no dgrad launch
        ws = torch.empty(max(ctx.ws_b, 1), device=x.device, dtype=torch.uint8)
        ctx.dp.backward(x, [wf], saved, dy, dx, [dw], ws, torch.cuda.current_stream(x.device).cuda_stream)
        return None, (dx if ctx.x_grad else None), dw.view(ctx.wshape)


class TcConv2d(nn.Conv2d):
    """``nn.Conv2d`` (groups 1, no bias, square kernel, fp32) whose training
    forward and weight gradient run on the tcgen05 GEMM templates.  CPU tensors
    use torch (not on the training hot path); CUDA tensors never fall back."""

    @classmethod
    def from_conv(cls, c: nn.Conv2d) -> "TcConv2d":
        if c.groups != 1 or c.bias is not None or c.dilation != (1, 1) or c.kernel_size[0] != c.kernel_size[1] or c.stride[0] != c.stride[1] or c.padding[0] != c.padding[1]:
            raise ValueError("TcConv2d: square, undilated, ungrouped, bias-free convolutions only")
        new = cls(c.in_channels, c.out_channels, c.kernel_size, c.stride, c.padding, bias=False)
        new.load_state_dict(c.state_dict())
        return new.to(c.weight.device)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        if not x.is_cuda:
            return super().forward(x)
        if x.dtype != torch.float32 or x.dim() != 4:
            raise TypeError("TcConv2d: fp32 NCHW input expected")
        return _ConvFn.apply(self, x, self.weight)


def _eligible(c) -> bool:
    return isinstance(c, nn.Conv2d) and not isinstance(c, TcConv2d) and c.bias is None and c.groups == 1 and c.dilation == (1, 1) and c.kernel_size[0] == c.kernel_size[1] and c.stride[0] == c.stride[1] and c.padding[0] == c.padding[1]


def accelerate_stem(model: nn.Module) -> bool:
    """Swap a ResNet-style stem ``model.conv1`` (input = data batch) for TcConv2d."""
    c = getattr(model, "conv1", None)
    if _eligible(c) and c.in_channels == 3:
        model.conv1 = TcConv2d.from_conv(c)
        return True
    return False


def accelerate_dense(model: nn.Module) -> int:
    """Swap the stem and every ResNet downsample conv (the remaining standard
    convs of a ResNet after Canvas replacement) for TcConv2d."""
    count = int(accelerate_stem(model))
    for m in model.modules():
        ds = getattr(m, "downsample", None)
        if isinstance(ds, nn.Sequential) and len(ds) and _eligible(ds[0]):
            ds[0] = TcConv2d.from_conv(ds[0])
            count += 1
    return count
