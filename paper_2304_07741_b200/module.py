"""Kernel-graph -> differentiable nn.Module replacement.

``CanvasConv2d`` is the trainer-plugin module of the SPEC (``build_module``,
SPEC.md:637-645) realised on the B200 executor: it holds the r x #FC weights
of one replacement target (Fig.-2 replication), applies the
stride policy (x[..., ::s, ::s] fused into the first loads)
and runs forward/backward through ``libcanvas_b200.so``.  ``replace`` swaps
every eligible ``nn.Conv2d`` of a network — the paper's
``canvas.sample(nn, budget)`` flow for one chosen kernel.

BN post-pass is off (App. A.10): the backbone's own BN follows
each replaced conv.
"""

from __future__ import annotations

import math

import torch
from torch import nn

from .executor import device_plan, plan_for


def conv_is_target(m: nn.Module) -> bool:
    """groups == 1 square odd kernel, 'same' padding, C_in | C_out or C_out | C_in."""
    if not isinstance(m, nn.Conv2d) or m.groups != 1 or m.dilation != (1, 1):
        return False
    kh, kw = m.kernel_size
    if kh != kw or m.stride[0] != m.stride[1] or m.padding != (kh // 2, kw // 2):
        return False
    ci, co = m.in_channels, m.out_channels
    return max(ci, co) % min(ci, co) == 0


class _CanvasFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, mod, x, *weights):
        dp = mod.device_plan(x)
        x = x.contiguous()
        n = x.shape[0]
        saved_b, ws_b = dp.sizes(n)
        ho, wo = mod.out_hw(x.shape[2], x.shape[3])
        y = torch.empty((n, mod.out_channels, ho, wo), device=x.device, dtype=torch.float32)
        saved = torch.empty(saved_b, device=x.device, dtype=torch.uint8)
        dp.forward(x, weights, y, saved, torch.cuda.current_stream(x.device).cuda_stream)
        ctx.dp = dp
        ctx.ws_b = ws_b
        ctx.save_for_backward(x, saved, *weights)
        return y

    @staticmethod
    def backward(ctx, dy):
        x, saved, *weights = ctx.saved_tensors
        dy = dy.contiguous()
        dx = torch.empty_like(x)
        dws = [torch.empty_like(w) for w in weights]
        ws = torch.empty(max(ctx.ws_b, 1), device=x.device, dtype=torch.uint8)
        ctx.dp.backward(x, weights, saved, dy, dx, dws, ws, torch.cuda.current_stream(x.device).cuda_stream)
        return (None, dx, *dws)


class CanvasConv2d(nn.Module):
    """One sampled Canvas kernel standing in for ``nn.Conv2d(c_in, c_out, k, stride, k//2)``."""

    def __init__(self, ir_text: str, in_channels: int, out_channels: int, kernel_size: int = 3, stride: int = 1, g: int = 4, xs: dict | None = None, bias: bool = False):
        super().__init__()
        self.ir_text = ir_text
        self.in_channels, self.out_channels = in_channels, out_channels
        self.kernel_size, self.stride, self.g, self.xs = kernel_size, stride, g, xs
        c = min(in_channels, out_channels)
        self.copies = max(in_channels, out_channels) // c
        # weight shapes do not depend on H, W (channel dims carry no spatial atom)
        probe = plan_for(ir_text, c_in=in_channels, c_out=out_channels, h=8 * stride, w=8 * stride, k=kernel_size, g=g, stride=stride, xs=xs)
        self.fc_shapes = [probe.graph.fc_shape(v) for v in probe.graph.fc_nodes]
        self.weights = nn.ParameterList()
        for _ in range(self.copies):
            for o, k in self.fc_shapes:
                w = torch.empty(o, k)
                b = 1.0 / math.sqrt(k)
                nn.init.uniform_(w, -b, b)  # U(+-1/sqrt(fan_in)), IR edge order (App. A.10)
                self.weights.append(nn.Parameter(w))
        self.bias = nn.Parameter(torch.zeros(out_channels)) if bias else None
        self._plans: dict = {}

    def __getstate__(self):
        """Compiled device plans (ctypes handles) are a cache: dropped on
        copy / pickle and rebuilt lazily (deduplicated by executor.device_plan)."""
        state = self.__dict__.copy()
        state["_plans"] = {}
        return state

    def out_hw(self, h: int, w: int) -> tuple[int, int]:
        return -(-h // self.stride), -(-w // self.stride)

    def plan(self, h: int, w: int):
        return plan_for(self.ir_text, c_in=self.in_channels, c_out=self.out_channels, h=h, w=w, k=self.kernel_size, g=self.g, stride=self.stride, xs=self.xs)

    def device_plan(self, x: torch.Tensor):
        if x.device.type != "cuda":
            raise RuntimeError("CanvasConv2d runs on the B200 executor only (no CPU fallback); move the module to cuda")
        if x.dtype != torch.float32:
            raise TypeError(f"CanvasConv2d computes in fp32, got {x.dtype}")
        if x.shape[1] != self.in_channels:
            raise ValueError(f"expected {self.in_channels} input channels, got {x.shape[1]}")
        key = (x.shape[2], x.shape[3], x.device.index)
        dp = self._plans.get(key)
        if dp is None:
            dp = device_plan(self.plan(x.shape[2], x.shape[3]), x.device.index or 0)
            self._plans[key] = dp
        return dp

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        y = _CanvasFn.apply(self, x, *self.weights)
        if self.bias is not None:
            y = y + self.bias.view(1, -1, 1, 1)
        return y

    def extra_repr(self) -> str:
        return f"{self.in_channels}, {self.out_channels}, k={self.kernel_size}, stride={self.stride}, copies={self.copies}, fc={self.fc_shapes}"


def replace(model: nn.Module, ir_text: str, *, g: int = 4, xs: dict | None = None, xs_by_name: dict | None = None, kernel_sizes=(3,), factory=None) -> list[str]:
    """Swap every eligible ``nn.Conv2d`` (kernel size in ``kernel_sizes``) for a Canvas module.

    ``xs_by_name`` gives per-target free-variable values (a level-2
    ``Solution``, see ``solve_for_model``); ``factory(conv) -> nn.Module``
    overrides the replacement (the CPU reference path uses it with oracle
    modules).  Returns the replaced names.
    """
    done = []
    for name, parent in list(model.named_modules()):
        for cname, child in list(parent.named_children()):
            if conv_is_target(child) and child.kernel_size[0] in kernel_sizes:
                full = f"{name}.{cname}" if name else cname
                txs = (xs_by_name or {}).get(full, xs)
                if factory is not None:
                    new = factory(child)
                else:
                    # G must divide C = min(C_in, C_out) (group(G), App. A.1); targets whose C
                    # it does not divide use the largest common divisor of the two
                    tg = math.gcd(min(child.in_channels, child.out_channels), g)
                    new = CanvasConv2d(ir_text, child.in_channels, child.out_channels, child.kernel_size[0], child.stride[0], g=tg, xs=txs, bias=child.bias is not None)
                setattr(parent, cname, new)
                done.append(f"{name}.{cname}" if name else cname)
    return done


def backbone_spec(model: nn.Module, input_shape=(1, 3, 224, 224), kernel_sizes=(3,)):
    """SPEC.md:376-381 BackboneSpec of a torch model: replacement targets with
    their output resolution (traced with forward hooks on a CPU copy of one
    image) and the analytical cost of everything that stays (other convs,
    linears: MACs and weights; BN: 2 params per channel)."""
    import copy

    from .canvas.constraint_solver import BackboneSpec, Target

    m = copy.deepcopy(model).cpu().eval()
    shapes: dict = {}
    hooks = []
    for name, mod in m.named_modules():
        if isinstance(mod, (nn.Conv2d, nn.Linear)):
            hooks.append(mod.register_forward_hook(lambda mod_, i, o, name=name: shapes.__setitem__(name, tuple(o.shape))))
    with torch.no_grad():
        m(torch.zeros(input_shape))
    for h in hooks:
        h.remove()
    targets, nf, npar = [], 0, 0
    for name, mod in m.named_modules():
        if isinstance(mod, nn.Conv2d):
            kh, kw = mod.kernel_size
            ho, wo = shapes[name][2:]
            params = mod.in_channels * mod.out_channels * kh * kw // mod.groups
            flops = params * ho * wo
            if conv_is_target(mod) and kh in kernel_sizes:
                targets.append(Target(name, mod.in_channels, mod.out_channels, ho, wo, kh, kw, flops, params))
            else:
                nf += flops
                npar += params + (mod.out_channels if mod.bias is not None else 0)
        elif isinstance(mod, nn.Linear):
            nf += mod.in_features * mod.out_features
            npar += mod.in_features * mod.out_features + (mod.out_features if mod.bias is not None else 0)
        elif isinstance(mod, nn.BatchNorm2d):
            npar += 2 * mod.num_features
    return BackboneSpec(tuple(targets), nf, npar)


def solve_for_model(model: nn.Module, ir_text: str, *, flops_frac: float | None = None, params_frac: float | None = None, g: int | None = None, input_shape=(1, 3, 224, 224)):
    """The paper's ``canvas.sample(nn, budget)`` solve step (§6.3):
    level-2 solve of one kernel over a network under a budget given as a
    fraction of the original totals.  Returns (Solution | None, spec, xs_by_name)."""
    from .canvas import ir as cir
    from .canvas.constraint_solver import Budget, solve_network
    from .canvas.cost_model import original_cost

    spec = backbone_spec(model, input_shape)
    of, op = original_cost(spec)
    budget = Budget(int(of * flops_frac) if flops_frac is not None else None, int(op * params_frac) if params_frac is not None else None)
    tmpl = cir.parse(ir_text).template
    sol = solve_network(tmpl, spec, budget, g=g)
    xs_by_name = {t.name: sol.target_xs(i) for i, t in enumerate(spec.targets)} if sol else {}
    return sol, spec, xs_by_name
