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
    assert res[6].status == "ok"
