"""Candidate-parallel dispatcher (config 4) host logic, with fake workers on CPU.

Covers: every task completes exactly once across 2 worker processes, results
come back in task order with the worker that ran them, a failing task is
re-queued once then reported failed, a worker that dies
mid-task has its task re-queued to a surviving worker.
"""

import hashlib
import os

from paper_2304_07741_b200.evaluator import CandidateEvaluator

MARK = os.environ.get("CANVAS_TEST_MARK", "/tmp/canvas_eval_marks")


def _mark(ir: str, tag: str) -> str:
    os.makedirs(MARK, exist_ok=True)
    return os.path.join(MARK, tag + hashlib.sha1(ir.encode()).hexdigest()[:12])


def fake_ok(ir, device, **kw):
    return {"status": "ok", "plan_ms": 0.0, "fwd_ms": len(ir) / 1000.0, "bwd_ms": 1.0, "fc_macs_per_image": 0, "extra": {"device": device, "pid": os.getpid()}}


def fake_flaky(ir, device, **kw):
    m = _mark(ir, f"flaky{kw.get('salt', '')}")
    if "BAD" in ir and not os.path.exists(m):
        open(m, "w").close()
        raise RuntimeError("transient")
    return fake_ok(ir, device)


def fake_always_fail(ir, device, **kw):
    if "BAD" in ir:
        raise ValueError("kernel does not lower")
    return fake_ok(ir, device)


def fake_die(ir, device, **kw):
    m = _mark(ir, f"die{kw.get('salt', '')}")
    if "DIE" in ir and not os.path.exists(m):
        open(m, "w").close()
        os._exit(3)
    return fake_ok(ir, device)


def fake_prepare(ir, device, **kw):
    return {"ir": ir, "prepared_in_thread": True}


def fake_pipelined(ir, device, prepared=None, **kw):
    """evaluate_fn with a ``prepare`` half: the worker compiles ahead on threads."""
    assert prepared is not None and prepared["ir"] == ir
    if "DIE" in ir:
        m = _mark(ir, f"pdie{kw.get('salt', '')}")
        if not os.path.exists(m):
            open(m, "w").close()
            os._exit(3)
    if "BAD" in ir:
        raise ValueError("kernel does not lower")
    return fake_ok(ir, device)


fake_pipelined.prepare = fake_prepare


def fake_sticky(ir, device, **kw):
    """A kernel that faults and leaves the process's device context broken
    (like an illegal address): every later task in that process fails too."""
    flag = _sticky_flag()
    if os.path.exists(flag):
        raise RuntimeError("CUDA error: an illegal memory access was encountered (sticky)")
    if "FAULT" in ir:
        open(flag, "w").close()
        raise RuntimeError("CUDA error: an illegal memory access was encountered")
    return fake_ok(ir, device)


def _sticky_flag():
    return _mark("sticky", f"proc{os.getpid()}-{os.environ.get('CANVAS_STICKY_SALT', '')}")


fake_sticky.healthy = lambda device: not os.path.exists(_sticky_flag())


def fake_parity(ir, device, **kw):
    r = fake_ok(ir, device)
    verdict = kw["checker"](ir, {}, None, None, [])
    r["extra"]["parity"] = verdict
    if not verdict["ok"]:
        r["status"] = "parity_fail"
    return r


def check_no_odd(ir, shapes, y, dx, dws):
    return {"ok": "odd" not in ir}

TEXTS = [f"kernel {i}" + ("x" * i) for i in range(12)]


def test_all_tasks_complete_in_order():
    res = CandidateEvaluator([0, 1], fake_ok).run(TEXTS, timeout_s=600)
    assert [r.task_id for r in res] == list(range(12))
    assert all(r.status == "ok" for r in res)
    assert {r.worker for r in res} <= {0, 1}
    assert res[5].fwd_ms == len(TEXTS[5]) / 1000.0


def test_transient_failure_is_requeued(tmp_path):
    texts = TEXTS[:4] + ["BAD one"]
    res = CandidateEvaluator([0, 1], fake_flaky, salt=str(tmp_path).replace("/", "_")).run(texts, timeout_s=600)
    assert all(r.status == "ok" for r in res)


def test_permanent_failure_reported():
    res = CandidateEvaluator([0, 1], fake_always_fail).run(TEXTS[:3] + ["BAD kernel"], timeout_s=600)
    assert [r.status for r in res] == ["ok", "ok", "ok", "failed"]
    assert "does not lower" in res[3].error


def test_worker_death_requeues(tmp_path):
    res = CandidateEvaluator([0, 1], fake_die, salt=str(tmp_path).replace("/", "_")).run(TEXTS[:6] + ["DIE here"] + TEXTS[6:8], timeout_s=600)
    assert len(res) == 9
    # every task completes: the dead worker's held task AND results it had queued
    # but not flushed (tracked in shared memory, released only on arrival)
    assert all(r.status == "ok" for r in res), [(r.task_id, r.status, r.error) for r in res]


def test_compile_ahead_pipeline():
    """prefetch > 0: tasks held ahead by a worker are all accounted for — every
    task exactly once, a failing one retried then failed, and every task held by a
    worker that dies (not just the running one) re-queued."""
    texts = TEXTS[:5] + ["BAD one"] + TEXTS[5:9] + ["DIE here"] + TEXTS[9:]
    salt = str(os.getpid())
    res = CandidateEvaluator([0, 1], fake_pipelined, prefetch=3, salt=salt).run(texts, timeout_s=600)
    assert [r.task_id for r in res] == list(range(len(texts)))
    st = {texts[r.task_id]: r.status for r in res}
    assert st.pop("BAD one") == "failed"
    assert all(v == "ok" for v in st.values()), st


def test_single_device_survives_worker_crash(tmp_path):
    """One device: a worker that dies is replaced by a fresh process, so the
    sweep still completes (a dead worker used to end a 1-GPU sweep)."""
    res = CandidateEvaluator([0], fake_die, salt=str(tmp_path).replace("/", "_")).run(TEXTS[:3] + ["DIE here"] + TEXTS[3:6], timeout_s=600)
    assert all(r.status == "ok" for r in res), [(r.task_id, r.status, r.error) for r in res]


def test_broken_context_worker_exits_and_is_replaced(monkeypatch):
    """After a fault that breaks the device context, the worker exits instead of
    failing every later task; the faulting task is retried on a fresh worker
    (and fails again there), every other task succeeds."""
    monkeypatch.setenv("CANVAS_STICKY_SALT", f"{os.getpid()}-{os.urandom(4).hex()}")  # inherited by the workers
    texts = TEXTS[:3] + ["FAULT kernel"] + TEXTS[3:8]
    res = CandidateEvaluator([0], fake_sticky, respawns=4).run(texts, timeout_s=600)
    st = [r.status for r in res]
    assert st[3] == "failed" and "illegal" in res[3].error
    assert st[:3] + st[4:] == ["ok"] * 8, [(r.task_id, r.status, r.error) for r in res]


def test_parity_checker_injected():
    """The caller's checker decides parity; failures are reported as parity_fail."""
    res = CandidateEvaluator([0, 1], fake_parity, checker=check_no_odd).run(["k even", "k odd", "k even2"], timeout_s=600)
    assert [r.status for r in res] == ["ok", "parity_fail", "ok"]
    assert res[1].extra["parity"] == {"ok": False}
