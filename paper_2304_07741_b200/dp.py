"""Batch-sharded data parallelism for Canvas networks.

One process per GPU, per-GPU batch fixed (weak scaling).  Every Canvas kernel
is per-image independent and the FC wgrad stays local, so the gradient
all-reduce is the only collective of a training step.

:class:`GradBuckets` gives every parameter's ``.grad`` a view into one flat
buffer (the parameters' dtype: fp32 on the GPU), split into buckets of
~``bucket_mb`` in *reverse* registration order (the order the backward
produces them).  A post-accumulate-grad hook
counts the parameters of each bucket as their gradients land; when a bucket
is complete its all-reduce (sum) is issued on a side stream that first waits
for the compute stream — so the all-reduce of the late layers overlaps the
backward of the early ones — and :meth:`finish` joins the side stream and
scales by 1/world before the optimizer step.  Everything is stream-ordered
with no host sync, so the whole step (forward, backward, bucketed NCCL
all-reduces, SGD) can be captured once as a CUDA graph (bench.py).  On CPU
(gloo) the same hooks issue the all-reduce synchronously; the multi-process
gloo test (tests/test_data_parallel_gloo.py) checks the sharded gradients
against full-batch gradients.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


class GradBuckets:
    def __init__(self, params, world: int, bucket_mb: float = 25.0, group=None, collective: bool | None = None):
        """``collective``: issue the all-reduces (default: world > 1; True at world 1
        runs the NCCL path on one GPU — bench.py's CANVAS_DP_SELFTEST)."""
        self.params = [p for p in params if p.requires_grad]
        self.world = world
        self.collective = world > 1 if collective is None else collective
        self.group = group
        total = sum(p.numel() for p in self.params)
        dev = self.params[0].device
        dtypes = {p.dtype for p in self.params}
        if len(dtypes) != 1:
            raise TypeError(f"GradBuckets: one parameter dtype expected, got {dtypes}")
        self.flat = torch.zeros(total, dtype=dtypes.pop(), device=dev)
        self.cuda = dev.type == "cuda"
        self.side = torch.cuda.Stream(dev) if self.cuda else None
        # reverse order: the last layers' gradients are ready first
        cap = max(1, int(bucket_mb * 2**20 // self.flat.element_size()))
        self.buckets: list[tuple[int, int, list]] = []  # (start, end, params) over the flat buffer
        off = total
        cur: list = []
        cur_end = total
        for p in reversed(self.params):
            n = p.numel()
            off -= n
            p.grad = self.flat[off : off + n].view_as(p)
            cur.append(p)
            if cur_end - off >= cap:
                self.buckets.append((off, cur_end, cur))
                cur, cur_end = [], off
        if cur:
            self.buckets.append((off, cur_end, cur))
        self.bucket_of = {id(p): b for b, (_, _, ps) in enumerate(self.buckets) for p in ps}
        self.pending = [0] * len(self.buckets)
        self.issued = [False] * len(self.buckets)
        self._hooks = [p.register_post_accumulate_grad_hook(self._on_grad) for p in self.params]

    # ----------------------------------------------------------------- step API
    def zero(self) -> None:
        """Start of a step: zero the flat buffer (the grads stay views of it)."""
        self.flat.zero_()
        self.pending = [len(ps) for _, _, ps in self.buckets]
        self.issued = [False] * len(self.buckets)

    def _on_grad(self, p) -> None:
        b = self.bucket_of[id(p)]
        self.pending[b] -= 1
        if self.pending[b] == 0:
            self._issue(b)

    def _issue(self, b: int) -> None:
        if self.issued[b]:
            return
        self.issued[b] = True
        s, e, _ = self.buckets[b]
        if not self.collective:
            return
        if self.cuda:
            self.side.wait_stream(torch.cuda.current_stream(self.flat.device))
            with torch.cuda.stream(self.side):
                dist.all_reduce(self.flat[s:e], group=self.group)
        else:
            dist.all_reduce(self.flat[s:e], group=self.group)

    def finish(self) -> None:
        """After backward: issue any bucket whose hooks did not all fire (unused
        parameters), join the side stream, average."""
        for b in range(len(self.buckets)):
            self._issue(b)
        if self.cuda and self.collective:  # join only a side stream that was forked (graph capture)
            torch.cuda.current_stream(self.flat.device).wait_stream(self.side)
        if self.world > 1:
            self.flat.div_(self.world)

    def remove(self) -> None:
        for h in self._hooks:
            h.remove()
