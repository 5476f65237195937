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

TEXTS = [f"kernel {i}" + ("x" * i) for i in range(12)]


def test_all_tasks_complete_in_order():
    res = CandidateEvaluator([0, 1], fake_ok).run(TEXTS, timeout_s=120)
    assert [r.task_id for r in res] == list(range(12))
    assert all(r.status == "ok" for r in res)
    assert {r.worker for r in res} <= {0, 1}
    assert res[5].fwd_ms == len(TEXTS[5]) / 1000.0


def test_transient_failure_is_requeued(tmp_path):
    texts = TEXTS[:4] + ["BAD one"]
    res = CandidateEvaluator([0, 1], fake_flaky, salt=str(tmp_path).replace("/", "_")).run(texts, timeout_s=120)
    assert all(r.status == "ok" for r in res)


def test_permanent_failure_reported():
    res = CandidateEvaluator([0, 1], fake_always_fail).run(TEXTS[:3] + ["BAD kernel"], timeout_s=120)
    assert [r.status for r in res] == ["ok", "ok", "ok", "failed"]
    assert "does not lower" in res[3].error


def test_worker_death_requeues(tmp_path):
    res = CandidateEvaluator([0, 1], fake_die, salt=str(tmp_path).replace("/", "_")).run(TEXTS[:6] + ["DIE here"] + TEXTS[6:8], timeout_s=120)
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
    res = CandidateEvaluator([0, 1], fake_pipelined, prefetch=3, salt=salt).run(texts, timeout_s=120)
    assert [r.task_id for r in res] == list(range(len(texts)))
    st = {texts[r.task_id]: r.status for r in res}
    assert st.pop("BAD one") == "failed"
    assert all(v == "ok" for v in st.values()), st
