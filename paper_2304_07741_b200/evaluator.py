"""Candidate-parallel kernel evaluation (config 4).

The reference specifies a harness whose dispatcher hands independent tasks to a
pool of workers with at-least-once delivery (PAPER.md
:432-435 "complete independence of all tasks").  Here a task is one sampled
kernel's IR text.  A worker owns one GPU.  For each task it:

1. solves the target shapes (config 1: N=8, C=64, H=W=56, G=4, K=3) and lowers the kernel;
2. compiles the plan;
3. times forward and backward on its device;
4. with ``parity_batch`` > 0, runs the *same* plan once more at that batch on
   seeded CPU-drawn inputs (x ~ N(0,1) seed 0, dy ~ N(0,1) seed 1, FC weights
   U(+-1/sqrt(fan_in)) seed 2 in IR edge order per replica — SURVEY §8d) and
   hands the outputs to the caller's ``checker(ir_text, shapes, y, dx, dws)``,
   which returns ``{"ok": bool, ...}``.  The checker is injected by the caller
   (the parity tests pass one that compares against the fp64 CPU oracle); the
   evaluator itself never imports the oracle.  A failed check is reported as
   status ``parity_fail``.

Work is partitioned as **replicas only**: there is no collective, and results return
over host IPC.  A task whose worker fails or dies is re-queued once (SPEC.md:567
``WorkerLost`` -> requeue), then reported ``failed``.  Non-finite outputs are
reported ``nonfinite``.

``evaluate_fn`` is injectable, so the dispatch logic is tested on CPU with
fake workers (tests/test_evaluator.py).

A worker whose device context is broken after a failed task (a sticky CUDA
error such as an illegal address: every later launch in that process would
fail too) exits; the dispatcher treats it as lost, re-queues what it held and
starts a fresh worker process for that device (at most ``respawns`` times per
device).  ``evaluate_fn.healthy(device)`` is the check (evaluate_kernel: a
device synchronize).

Compile-ahead (``prefetch`` > 0): plan creation is host work (lowering + NVRTC,
~0.6 s per kernel) while timing is device work, so a worker compiles the next
``prefetch`` kernels on host threads (the C ABI call releases the GIL) while it
times the current one — device timings stay serial and unperturbed.  Used when
``evaluate_fn`` carries a ``prepare`` attribute (``evaluate_kernel`` does).
"""

from __future__ import annotations

import collections
import multiprocessing as mp
import queue
import time
from dataclasses import asdict, dataclass, field


@dataclass
class EvalTask:
    task_id: int
    ir_text: str
    attempts: int = 0


@dataclass
class EvalResult:
    task_id: int
    status: str  # "ok" | "nonfinite" | "failed"
    worker: int = -1
    plan_ms: float = 0.0  # host lowering + NVRTC compile + module load
    fwd_ms: float = 0.0
    bwd_ms: float = 0.0
    fc_macs_per_image: int = 0
    error: str = ""
    extra: dict = field(default_factory=dict)

    def as_dict(self) -> dict:
        return asdict(self)


CONFIG1 = {"c_in": 64, "c_out": 64, "h": 56, "w": 56, "k": 3, "g": 4, "batch": 8, "stride": 1}


def parity_inputs(plan, shapes: dict, batch: int):
    """Seeded CPU inputs of the parity sample (x, flat FC weights, dy) — the
    recipe of SURVEY §8d, drawn on the host so a checker re-drawing them with
    the same seeds sees identical bits."""
    import math

    import torch

    sh = dict(CONFIG1, **shapes)
    x = torch.randn(batch, sh["c_in"], sh["h"], sh["w"], generator=torch.Generator().manual_seed(0), dtype=torch.float32)
    g = torch.Generator().manual_seed(2)
    ws = []
    for _ in range(plan.copies):
        for v in plan.graph.fc_nodes:
            o, k = plan.graph.fc_shape(v)
            b = 1.0 / math.sqrt(k)
            ws.append((torch.rand((o, k), generator=g, dtype=torch.float64) * 2 - 1).mul_(b).to(torch.float32))
    ho, wo = -(-sh["h"] // sh["stride"]), -(-sh["w"] // sh["stride"])
    dy = torch.randn(batch, sh["c_out"], ho, wo, generator=torch.Generator().manual_seed(1), dtype=torch.float32)
    return x, ws, dy


def prepare_kernel(ir_text: str, device: int, *, shapes: dict | None = None, iters: int = 5, **_) -> dict:
    """Host half of an evaluation: lower + compile + load (thread-safe)."""
    from .executor import device_plan, plan_for

    del iters
    sh = dict(CONFIG1, **(shapes or {}))
    t0 = time.perf_counter()
    plan = plan_for(ir_text, c_in=sh["c_in"], c_out=sh["c_out"], h=sh["h"], w=sh["w"], k=sh["k"], g=sh["g"], stride=sh["stride"])
    dp = device_plan(plan, device)
    return {"plan": plan, "dp": dp, "plan_ms": (time.perf_counter() - t0) * 1e3}


def _run_once(dp, plan, x, ws, dy, device):
    """One forward + backward of ``dp`` on device copies of host tensors -> host (y, dx, dws)."""
    import torch

    dev = torch.device("cuda", device)
    xd, dyd = x.to(dev), dy.to(dev)
    wd = [w.to(dev) for w in ws]
    n = x.shape[0]
    sb, wb = dp.sizes(n)
    saved = torch.empty(max(sb, 1), dtype=torch.uint8, device=dev)
    work = torch.empty(max(wb, 1), dtype=torch.uint8, device=dev)
    y = torch.empty(dyd.shape, device=dev)
    dx = torch.zeros_like(xd)
    dws = [torch.empty_like(w) for w in wd]
    st = torch.cuda.current_stream(dev).cuda_stream
    dp.forward(xd, wd, y, saved, st)
    dp.backward(xd, wd, saved, dyd, dx, dws, work, st)
    torch.cuda.synchronize(dev)
    return y.cpu(), dx.cpu(), [d.cpu() for d in dws]


def evaluate_kernel(ir_text: str, device: int, *, shapes: dict | None = None, iters: int = 5, prepared: dict | None = None, parity_batch: int = 0, checker=None, graph: bool = True) -> dict:
    """Plan + fwd/bwd latency of one kernel on ``cuda:device`` (CUDA events; with
    ``graph`` replayed from one CUDA graph per direction, eager timings in
    ``extra``); with ``parity_batch`` and ``checker``: the parity sample (module
    doc, step 4)."""
    import torch

    sh = dict(CONFIG1, **(shapes or {}))
    prepared = prepared or prepare_kernel(ir_text, device, shapes=shapes)
    plan, dp, plan_ms = prepared["plan"], prepared["dp"], prepared["plan_ms"]
    dev = torch.device("cuda", device)
    torch.cuda.set_device(dev)
    n = sh["batch"]
    gen = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn(n, sh["c_in"], sh["h"], sh["w"], device=dev, generator=gen)
    ws = [torch.rand(o, k_, device=dev, generator=gen).sub_(0.5).mul_(2 / k_**0.5) for _ in range(plan.copies) for o, k_ in (plan.graph.fc_shape(v) for v in plan.graph.fc_nodes)]
    ho, wo = -(-sh["h"] // sh["stride"]), -(-sh["w"] // sh["stride"])
    y = torch.empty(n, sh["c_out"], ho, wo, device=dev)
    sb, wb = dp.sizes(n)
    saved = torch.empty(max(sb, 1), dtype=torch.uint8, device=dev)
    work = torch.empty(max(wb, 1), dtype=torch.uint8, device=dev)
    dy = torch.randn(y.shape, device=dev, generator=gen)
    dx = torch.empty_like(x)
    dws = [torch.empty_like(w) for w in ws]
    st = torch.cuda.current_stream(dev).cuda_stream
    for _ in range(2):
        dp.forward(x, ws, y, saved, st)
        dp.backward(x, ws, saved, dy, dx, dws, work, st)

    def timed(fwd, bwd):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
        for _ in range(iters):
            fwd()
        ev[1].record()
        for _ in range(iters):
            bwd()
        ev[2].record()
        torch.cuda.synchronize(dev)
        return ev[0].elapsed_time(ev[1]) / iters, ev[1].elapsed_time(ev[2]) / iters

    fwd_e, bwd_e = timed(lambda: dp.forward(x, ws, y, saved, st), lambda: dp.backward(x, ws, saved, dy, dx, dws, work, st))
    extra = {"launches_fwd": dp.launches(0), "launches_bwd": dp.launches(1), "fwd_ms_eager": fwd_e, "bwd_ms_eager": bwd_e}
    fwd_ms, bwd_ms = fwd_e, bwd_e
    if graph:
        # one CUDA graph per (plan, batch) for each direction: a config-1 kernel is
        # 4-16 short launches, so the eager numbers are host-launch bound; the
        # graph replay is the device latency the search ranks candidates by
        try:
            gf, gb = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            cs = torch.cuda.Stream(dev)
            cs.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(cs):
                with torch.cuda.graph(gf, stream=cs):
                    dp.forward(x, ws, y, saved, cs.cuda_stream)
                with torch.cuda.graph(gb, stream=cs):
                    dp.backward(x, ws, saved, dy, dx, dws, work, cs.cuda_stream)
            torch.cuda.current_stream(dev).wait_stream(cs)
            gf.replay()
            gb.replay()
            fwd_ms, bwd_ms = timed(gf.replay, gb.replay)
            extra["graph"] = True
        except Exception as e:  # capture unsupported here: eager timings stand
            extra["graph"] = False
            extra["graph_error"] = str(e)[:200]
    finite = bool(torch.isfinite(y).all()) and bool(torch.isfinite(dx).all())
    status = "ok" if finite else "nonfinite"
    if parity_batch > 0 and checker is not None:
        px, pws, pdy = parity_inputs(plan, sh, parity_batch)
        py, pdx, pdws = _run_once(dp, plan, px, pws, pdy, device)
        verdict = checker(ir_text, sh, py.numpy(), pdx.numpy(), [d.numpy() for d in pdws])
        extra["parity"] = verdict
        if status == "ok" and not verdict.get("ok", False):
            status = "parity_fail"
    return {
        "status": status,
        "plan_ms": plan_ms,
        "fwd_ms": fwd_ms,
        "bwd_ms": bwd_ms,
        "fc_macs_per_image": plan.graph.fc_macs_per_image(),
        "extra": extra,
    }


def _cuda_healthy(device: int) -> bool:
    """False when the process's CUDA context on ``device`` is broken (sticky error)."""
    try:
        import torch

        torch.cuda.synchronize(device)
        torch.empty(1, device=torch.device("cuda", device)).add_(1)
        torch.cuda.synchronize(device)
        return True
    except Exception:
        return False


evaluate_kernel.prepare = prepare_kernel
evaluate_kernel.healthy = _cuda_healthy


def _hold(held, tid: int) -> None:
    """Record a task this worker holds in shared memory (a synchronous write, so it
    survives the worker dying with queued messages still unflushed).  Only the
    dispatcher releases a slot, once the task's result has actually arrived."""
    while True:
        for i in range(len(held)):
            if held[i] < 0:
                held[i] = tid
                return
        time.sleep(0.01)  # all slots await results still in flight


def _release(held, tid: int) -> None:
    for i in range(len(held)):
        if held[i] == tid:
            held[i] = -1
            return


def _exit_if_broken(evaluate_fn, device: int, results) -> None:
    """After a failed task: a worker whose device context is broken exits (its
    held tasks are re-queued and a fresh worker replaces it, module doc)."""
    healthy = getattr(evaluate_fn, "healthy", None)
    if healthy is not None and not healthy(device):
        results.close()
        results.join_thread()  # flush the error report before dying
        import os

        os._exit(70)


def _worker(wid: int, device: int, tasks, results, evaluate_fn, kwargs, prefetch: int = 0, held=None) -> None:
    held = held if held is not None else [-1]
    prep = getattr(evaluate_fn, "prepare", None) if prefetch > 0 else None
    if prep is not None:
        return _worker_pipelined(wid, device, tasks, results, evaluate_fn, prep, kwargs, prefetch, held)
    while True:
        t = tasks.get()
        if t is None:
            return
        _hold(held, t.task_id)
        results.put(("start", wid, t.task_id))
        try:
            r = evaluate_fn(t.ir_text, device, **kwargs)
            results.put(("done", wid, EvalResult(t.task_id, worker=wid, **r)))
        except Exception as err:  # reported, re-queued by the dispatcher
            results.put(("error", wid, EvalResult(t.task_id, "failed", worker=wid, error=f"{type(err).__name__}: {err}"[:500])))
            _exit_if_broken(evaluate_fn, device, results)


def _worker_pipelined(wid, device, tasks, results, evaluate_fn, prep, kwargs, prefetch, held) -> None:
    from concurrent.futures import ThreadPoolExecutor

    pool = ThreadPoolExecutor(prefetch)
    ahead: collections.deque = collections.deque()
    exhausted = False
    while True:
        while not exhausted and len(ahead) <= prefetch:
            try:  # block only when nothing is held, so held tasks never wait on the queue
                t = tasks.get() if not ahead else tasks.get_nowait()
            except queue.Empty:
                break
            if t is None:
                exhausted = True
                break
            _hold(held, t.task_id)
            results.put(("start", wid, t.task_id))
            ahead.append((t, pool.submit(prep, t.ir_text, device, **kwargs)))
        if not ahead:
            if exhausted:
                pool.shutdown()
                return
            continue
        t, fut = ahead.popleft()
        try:
            r = evaluate_fn(t.ir_text, device, prepared=fut.result(), **kwargs)
            results.put(("done", wid, EvalResult(t.task_id, worker=wid, **r)))
        except Exception as err:
            results.put(("error", wid, EvalResult(t.task_id, "failed", worker=wid, error=f"{type(err).__name__}: {err}"[:500])))
            _exit_if_broken(evaluate_fn, device, results)


class CandidateEvaluator:
    """Dispatch kernels to one worker process per device; collect results in task order."""

    def __init__(self, devices, evaluate_fn=evaluate_kernel, max_attempts: int = 2, prefetch: int = 0, respawns: int = 3, **kwargs):
        self.devices = list(devices)
        self.prefetch = prefetch
        self.evaluate_fn = evaluate_fn
        self.max_attempts = max_attempts
        self.respawns = respawns
        self.kwargs = kwargs

    def run(self, ir_texts, timeout_s: float = 3600.0) -> list[EvalResult]:
        ctx = mp.get_context("spawn")
        # results: a SimpleQueue, whose put writes the pipe synchronously in the worker's
        # own thread — a worker that exits (os._exit on a broken context, a crash) right
        # after a put cannot leave a half-flushed message or a held feeder-thread write
        # lock behind, which with mp.Queue stalls every other worker's reports
        tasks, results = ctx.Queue(), ctx.SimpleQueue()

        def results_get(timeout: float):
            if not results._reader.poll(timeout):
                raise queue.Empty
            return results.get()

        pending = {i: EvalTask(i, t) for i, t in enumerate(ir_texts)}
        for t in pending.values():
            tasks.put(t)
        procs = {}
        held = {}
        device_of = {}

        def spawn(wid: int, dev: int) -> None:
            held[wid] = ctx.Array("q", [-1] * (self.prefetch + 64), lock=False)
            device_of[wid] = dev
            p = ctx.Process(target=_worker, args=(wid, dev, tasks, results, self.evaluate_fn, self.kwargs, self.prefetch, held[wid]), daemon=True)
            p.start()
            procs[wid] = p

        for wid, dev in enumerate(self.devices):
            spawn(wid, dev)
        respawned = {dev: 0 for dev in self.devices}
        inflight: dict = {}  # worker -> task ids it holds
        lost: set = set()
        done: dict[int, EvalResult] = {}
        deadline = time.monotonic() + timeout_s
        try:
            while len(done) < len(pending) and time.monotonic() < deadline:
                try:
                    kind, wid, payload = results_get(0.5)
                except queue.Empty:
                    # worker lost (process died mid-task): re-queue its task
                    for wid, p in procs.items():
                        if p.is_alive() or wid in lost:
                            continue
                        lost.add(wid)  # its held tasks: from shared memory (messages may be lost with it)
                        for tid in sorted(inflight.pop(wid, set()) | {v for v in held[wid][:] if v >= 0}):
                            if tid not in done:
                                self._retry(pending[tid], tasks, done, "worker lost")
                        dev = device_of[wid]
                        if respawned[dev] < self.respawns and len(done) < len(pending):
                            respawned[dev] += 1  # a fresh process (fresh CUDA context) for that device
                            spawn(max(procs) + 1, dev)
                        break  # procs changed size
                    if not any(p.is_alive() for p in procs.values()):
                        break
                    continue
                if kind == "start":
                    inflight.setdefault(wid, set()).add(payload)
                    continue
                inflight.get(wid, set()).discard(payload.task_id)
                _release(held[wid], payload.task_id)
                if kind == "done":
                    done[payload.task_id] = payload
                else:
                    self._retry(pending[payload.task_id], tasks, done, payload.error, payload)
        finally:
            for _ in procs:
                tasks.put(None)
            for p in procs.values():
                p.join(timeout=5)
                if p.is_alive():
                    p.terminate()
        for i in pending:
            done.setdefault(i, EvalResult(i, "failed", error="not completed"))
        return [done[i] for i in sorted(done)]

    def _retry(self, task: EvalTask, tasks, done, why: str, result: EvalResult | None = None) -> None:
        task.attempts += 1
        if task.attempts < self.max_attempts:
            tasks.put(task)
        else:
            done[task.task_id] = result or EvalResult(task.task_id, "failed", error=why)
