"""Search harness: accuracy-curve pruning, leaderboard and a progress-aware
dispatcher (SPEC.md:535-596 [MODULE] harness; §7).

* ``PruneRule`` / ``prune_decision`` — a candidate is pruned at epoch e when
  its accuracy is below lambda(e / total) * best[e], lambda(x) = theta +
  (1 - theta) x, theta = 0.5 by default (the normalised-epoch
  reading of SPEC.md:586); no pruning until a first candidate has completed
  (cold start).
* ``Leaderboard`` — idempotent by task_id (at-least-once delivery),
  ordered by (final accuracy within budget, then measured latency); the best
  curve is replaced atomically when a completed candidate ends higher.
* ``Dispatcher`` — independent tasks on one worker process each (replicas,
  no collective); workers stream per-epoch progress over a queue, the
  dispatcher answers with a prune message when ``prune_decision`` fires, and a
  task whose worker dies is re-queued on a fresh worker (SPEC.md:567 WorkerLost).  Message
  passing only: the dispatcher is the single writer of the leaderboard
  (SPEC.md:589).  The reference's line-delimited socket transport is not built
  (networking is outside this build's scope); the message fields are the
  protocol's (type, task_id, kernel_ir, epochs, epoch, accuracy, latency_ms,
  reason).

``train_fn(task, report) -> dict`` is the worker body: it calls
``report(epoch, accuracy)`` after each epoch (epochs 0, 1, ...); when the
dispatcher prunes the task, ``report`` raises and the task ends there; it
returns ``{"accuracy": final, "latency_ms": ...}``.
``synthetic_accuracy_worker`` trains a replaced model on a synthetic task on a
GPU; tests inject scripted curves.
"""

from __future__ import annotations

import collections
import multiprocessing as mp
import queue
import time
from dataclasses import dataclass, field


@dataclass
class PruneRule:
    theta: float = 0.5
    best_curve: list | None = None

    def lam(self, x: float) -> float:
        """lambda(x) = theta + (1 - theta) x on [0, 1] (§7)."""
        if not 0.0 <= self.theta <= 1.0:
            raise ValueError("theta must be in [0, 1]")
        x = min(max(x, 0.0), 1.0)
        return self.theta + (1.0 - self.theta) * x


def prune_threshold(rule: PruneRule, epoch: int, total_epochs: int) -> float | None:
    if rule.best_curve is None or epoch >= len(rule.best_curve):
        return None
    return rule.lam(epoch / total_epochs) * rule.best_curve[epoch]


def final_epoch_index(epochs: int) -> int:
    """``total_epochs`` argument for curves reported at epochs 0 .. E-1: the index
    of the final epoch, so that lambda reaches 1 there ("final epoch:
    threshold = best[last] exactly") while epoch 0 stays at theta."""
    return max(epochs - 1, 1)


def prune_decision(rule: PruneRule, candidate: list, epoch: int, total_epochs: int) -> str:
    """'prune' iff candidate[epoch] < lambda(epoch / total) * best[epoch], else 'continue'."""
    thr = prune_threshold(rule, epoch, total_epochs)
    if thr is None or epoch >= len(candidate):
        return "continue"
    return "prune" if candidate[epoch] < thr else "continue"


@dataclass
class HarnessTask:
    task_id: int
    kernel_ir: str
    epochs: int = 1
    kind: str = "accuracy"  # accuracy | latency
    flops: int = 0
    params: int = 0
    attempts: int = 0


@dataclass
class Entry:
    task_id: int
    status: str  # completed | pruned | failed
    curve: list = field(default_factory=list)
    accuracy: float = 0.0
    latency_ms: float = float("inf")
    within_budget: bool = True
    reason: str = ""
    worker: int = -1


class Leaderboard:
    """Single-writer leaderboard; results are idempotent by task_id."""

    def __init__(self, rule: PruneRule | None = None):
        self.rule = rule or PruneRule()
        self.entries: dict[int, Entry] = {}

    def record(self, e: Entry) -> bool:
        if e.task_id in self.entries:
            return False  # at-least-once delivery: the first result wins
        self.entries[e.task_id] = e
        if e.status == "completed" and e.curve:
            best = self.rule.best_curve
            if best is None or e.curve[-1] > best[-1]:
                self.rule.best_curve = list(e.curve)
        return True

    def ranking(self) -> list[Entry]:
        done = [e for e in self.entries.values() if e.status == "completed"]
        return sorted(done, key=lambda e: (not e.within_budget, -e.accuracy, e.latency_ms, e.task_id))

    def best(self) -> Entry | None:
        r = self.ranking()
        return r[0] if r else None


def _worker(wid: int, inbox, results, train_fn, kwargs) -> None:
    """Worker loop: tasks and prune/continue answers arrive on ``inbox`` (the
    dispatcher assigns each task to one worker, so it always knows what a lost
    worker held).  The first message is ``ready`` (the process is up)."""
    results.put({"type": "ready", "worker": wid, "task_id": -1})
    while True:
        t = inbox.get()
        if t is None:
            return

        def report(epoch: int, accuracy: float, t=t) -> None:
            results.put({"type": "progress", "worker": wid, "task_id": t.task_id, "epoch": epoch, "accuracy": accuracy})
            msg = inbox.get()  # the dispatcher answers every progress report
            if msg.get("type") == "prune":
                raise _Pruned(msg.get("reason", ""))

        try:
            r = train_fn(t, report, **kwargs)
            results.put({"type": "result", "worker": wid, "task_id": t.task_id, **r})
        except _Pruned:
            results.put({"type": "result", "worker": wid, "task_id": t.task_id, "reason": "pruned"})
        except Exception as err:  # reported, re-queued by the dispatcher
            results.put({"type": "bye", "worker": wid, "task_id": t.task_id, "reason": f"{type(err).__name__}: {err}"[:300]})


class _Pruned(Exception):
    pass


class Dispatcher:
    """Runs HarnessTasks on ``workers`` processes with accuracy-curve pruning."""

    def __init__(self, workers: int, train_fn, rule: PruneRule | None = None, max_attempts: int = 2, budget=None, warm_start: bool = False, **kwargs):
        self.n = workers
        # warm_start: start every worker and wait for its ``ready`` before the first
        # task, so process start-up is not charged to the dispatch (steady state,
        # SPEC.md:679 simulated-worker throughput); ``timing`` records both phases
        self.warm_start = warm_start
        self.timing: dict = {}
        self.train_fn = train_fn
        self.board = Leaderboard(rule)
        self.max_attempts = max_attempts
        self.budget = budget  # (max_flops, max_params) or None
        self.kwargs = kwargs
        self.messages: list = []  # every prune message sent (observability)

    def run(self, tasks: list[HarnessTask], timeout_s: float = 3600.0) -> Leaderboard:
        ctx = mp.get_context("spawn")
        # results: a SimpleQueue, whose put writes the pipe synchronously in the
        # worker's own thread — a worker that dies (os._exit, a fault) after a put
        # cannot leave a half-flushed message or a held feeder-thread write lock
        # behind, which with mp.Queue can stall every other worker's reports
        rq = ctx.SimpleQueue()

        def rq_get(timeout: float):
            if not rq._reader.poll(timeout):
                raise queue.Empty
            return rq.get()

        pending = {t.task_id: t for t in tasks}
        todo = collections.deque(tasks)
        procs: dict[int, tuple] = {}  # worker id -> (process, inbox)
        inflight: dict[int, int] = {}  # worker id -> task id
        curves: dict[int, list] = {}
        next_wid = 0

        def spawn() -> int:
            nonlocal next_wid
            w, next_wid = next_wid, next_wid + 1
            inbox = ctx.Queue()
            p = ctx.Process(target=_worker, args=(w, inbox, rq, self.train_fn, self.kwargs), daemon=True)
            p.start()
            procs[w] = (p, inbox)
            return w

        def assign(w: int) -> None:
            while todo:
                t = todo.popleft()
                if t.task_id in self.board.entries:
                    continue
                inflight[w] = t.task_id
                curves[t.task_id] = []
                procs[w][1].put(t)
                return

        t_spawn = time.monotonic()
        first = [spawn() for _ in range(min(self.n, len(tasks)))]
        deadline = time.monotonic() + timeout_s
        early: list = []
        if self.warm_start:
            ready: set = set()
            while len(ready) < len(first) and time.monotonic() < deadline:
                try:
                    m = rq_get(0.2)
                except queue.Empty:
                    if any(not procs[w][0].is_alive() for w in first):
                        break
                    continue
                if m["type"] == "ready":
                    ready.add(m["worker"])
                else:
                    early.append(m)
        t_run = time.monotonic()
        self.timing = {"startup_s": t_run - t_spawn}
        for w in first:
            assign(w)
        try:
            while len(self.board.entries) < len(pending) and time.monotonic() < deadline:
                for w in [w for w in inflight if not procs[w][0].is_alive()]:  # WorkerLost
                    procs.pop(w)
                    self._retry(pending[inflight.pop(w)], todo, "worker lost")
                    assign(spawn())
                if not inflight and not todo:
                    break
                try:
                    m = early.pop() if early else rq_get(0.2)
                except queue.Empty:
                    continue
                if m["type"] == "ready":
                    continue
                w, tid = m["worker"], m["task_id"]
                if w not in procs or inflight.get(w) != tid:
                    continue  # stale message from a worker already declared lost
                if m["type"] == "progress":
                    c = curves[tid]
                    c.append(m["accuracy"])
                    t = pending[tid]
                    last = final_epoch_index(t.epochs)  # epochs are reported 0 .. E-1
                    if prune_decision(self.board.rule, c, m["epoch"], last) == "prune":
                        thr = prune_threshold(self.board.rule, m["epoch"], last)
                        msg = {"type": "prune", "task_id": tid, "reason": f"accuracy {m['accuracy']:.4f} < {thr:.4f} at epoch {m['epoch']}"}
                        self.messages.append(msg)
                        self.board.record(Entry(tid, "pruned", list(c), c[-1], reason=msg["reason"], worker=w))
                        procs[w][1].put(msg)
                    else:
                        procs[w][1].put({"type": "continue", "task_id": tid})
                    continue
                inflight.pop(w)
                if m["type"] == "result" and m.get("reason") != "pruned":  # pruned: recorded when the message was sent
                    t = pending[tid]
                    within = self.budget is None or ((self.budget[0] is None or t.flops <= self.budget[0]) and (self.budget[1] is None or t.params <= self.budget[1]))
                    self.board.record(Entry(tid, "completed", curves[tid], float(m.get("accuracy", 0.0)), float(m.get("latency_ms", float("inf"))), within, worker=w))
                elif m["type"] == "bye":
                    self._retry(pending[tid], todo, m.get("reason", "error"))
                assign(w)
        finally:
            self.timing["run_s"] = time.monotonic() - t_run
            for p, inbox in procs.values():
                inbox.put(None)
            for p, _ in procs.values():
                p.join(timeout=5)
                if p.is_alive():
                    p.terminate()
        for tid in pending:
            if tid not in self.board.entries:
                self.board.record(Entry(tid, "failed", reason="not completed"))
        return self.board

    def _retry(self, t: HarnessTask, todo, why: str) -> None:
        t.attempts += 1
        if t.attempts < self.max_attempts:
            todo.append(t)
        else:
            self.board.record(Entry(t.task_id, "failed", reason=why))


def synthetic_accuracy_worker(task: HarnessTask, report, device: int = 0, batch: int = 64, steps_per_epoch: int = 20, channels: int = 16) -> dict:
    """Train a 2-layer CNN whose middle conv is the candidate kernel (CanvasConv2d
    on the B200) on a fixed synthetic 10-class task; report per-epoch accuracy on a
    held-out synthetic batch; measure the kernel's fwd+bwd latency."""
    import torch
    import torch.nn.functional as F
    from torch import nn

    from .module import CanvasConv2d

    dev = torch.device("cuda", device)
    torch.manual_seed(0)
    proto = torch.randn(10, 3, 16, 16, generator=torch.Generator().manual_seed(1)).to(dev)

    def data(n, seed):
        g = torch.Generator(device=dev).manual_seed(seed)
        y = torch.randint(0, 10, (n,), device=dev, generator=g)
        return proto[y] + 0.7 * torch.randn(n, 3, 16, 16, device=dev, generator=g), y

    model = nn.Sequential(nn.Conv2d(3, channels, 3, padding=1), nn.ReLU(), CanvasConv2d(task.kernel_ir, channels, channels, 3), nn.BatchNorm2d(channels), nn.ReLU(), nn.AdaptiveAvgPool2d(1), nn.Flatten(), nn.Linear(channels, 10)).to(dev)
    opt = torch.optim.SGD(model.parameters(), lr=0.05, momentum=0.9)
    xv, yv = data(512, 999)
    acc = 0.0
    for ep in range(task.epochs):
        model.train()
        for it in range(steps_per_epoch):
            x, y = data(batch, ep * 1000 + it)
            opt.zero_grad(set_to_none=True)
            F.cross_entropy(model(x), y).backward()
            opt.step()
        model.eval()
        with torch.no_grad():
            acc = float((model(xv).argmax(1) == yv).float().mean())
        report(ep, acc)
    conv = model[2]
    x = torch.randn(batch, channels, 16, 16, device=dev, requires_grad=True)
    for _ in range(3):
        conv(x).sum().backward()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(10):
        conv(x).sum().backward()
    ev[1].record()
    torch.cuda.synchronize(dev)
    return {"accuracy": acc, "latency_ms": ev[0].elapsed_time(ev[1]) / 10}
