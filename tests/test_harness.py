"""Search harness: the prune rule's SPEC examples, leaderboard
idempotency and ordering, and the dispatcher with scripted workers — pruning
mid-training, worker loss (task re-run elsewhere, one entry), scaling with
simulated fixed-latency workers."""

import os
import time

import pytest

from paper_2304_07741_b200.harness import Dispatcher, Entry, HarnessTask, Leaderboard, PruneRule, final_epoch_index, prune_decision, prune_threshold


def test_spec_examples():
    # theta = 0.5, epoch 0: candidate needs >= 0.5 * best[0]
    r = PruneRule(0.5, [0.4, 0.5, 0.6])
    assert prune_threshold(r, 0, 3) == pytest.approx(0.2)
    assert prune_decision(r, [0.19], 0, 3) == "prune" and prune_decision(r, [0.2], 0, 3) == "continue"
    # final epoch: threshold = best[last] exactly (lambda(1) = 1)
    r = PruneRule(0.5, [0.1, 0.3, 0.6])
    assert prune_threshold(r, 2, 2) == pytest.approx(0.6)
    # theta = 0.5, total = 300, epoch 150, best = 0.60 -> threshold 0.45
    r = PruneRule(0.5, [0.0] * 150 + [0.60])
    assert prune_threshold(r, 150, 300) == pytest.approx(0.45)
    # cold start: no best curve -> never prune
    assert prune_decision(PruneRule(), [0.0], 0, 10) == "continue"


def test_final_reported_epoch_uses_full_best():
    """Workers report epochs 0 .. E-1: with the dispatcher's normalisation the
    last reported epoch compares against best[last] exactly (lambda = 1) and
    epoch 0 against theta * best[0] (lambda used to stop short of 1)."""
    for E in (2, 3, 10):
        r = PruneRule(0.5, [0.1 * (i + 1) for i in range(E)])
        assert prune_threshold(r, E - 1, final_epoch_index(E)) == pytest.approx(r.best_curve[-1])
        assert prune_threshold(r, 0, final_epoch_index(E)) == pytest.approx(0.5 * r.best_curve[0])
        just_below = [0.0] * (E - 1) + [r.best_curve[-1] - 1e-9]
        assert prune_decision(r, just_below, E - 1, final_epoch_index(E)) == "prune"


def test_prune_monotonicity():
    """A pointwise-lower curve is pruned no later than the original."""
    import random

    rng = random.Random(0)
    for _ in range(200):
        best = [rng.random() for _ in range(8)]
        r = PruneRule(rng.random(), best)
        cand = [rng.random() for _ in range(8)]
        lower = [c * rng.random() for c in cand]

        def first(c):
            return next((e for e in range(8) if prune_decision(r, c, e, 8) == "prune"), 99)

        assert first(lower) <= first(cand)


def test_leaderboard_idempotent_and_ordered():
    b = Leaderboard()
    assert b.record(Entry(1, "completed", [0.5, 0.7], 0.7, 3.0))
    assert not b.record(Entry(1, "completed", [0.9], 0.9, 1.0))  # duplicate delivery
    b.record(Entry(2, "completed", [0.6, 0.7], 0.7, 2.0))
    b.record(Entry(3, "completed", [0.8], 0.8, 9.0, within_budget=False))
    b.record(Entry(4, "pruned", [0.1], 0.1))
    assert [e.task_id for e in b.ranking()] == [2, 1, 3]
    assert b.rule.best_curve == [0.8]  # a completed candidate ending higher replaces the best curve
    b.record(Entry(5, "completed", [0.2, 0.95], 0.95, 5.0))
    assert b.rule.best_curve == [0.2, 0.95]


# scripted workers (module level: spawned processes import them)
CURVES = {0: [0.5, 0.6, 0.7, 0.8], 1: [0.1, 0.1, 0.1, 0.1], 2: [0.45, 0.55, 0.75, 0.85], 3: [0.3, 0.2, 0.1, 0.0]}


def scripted(task, report, delay=0.0, die_on=None):
    if die_on is not None and task.task_id == die_on and task.attempts == 0:
        os._exit(1)  # worker lost mid-task
    for e, a in enumerate(CURVES[task.task_id % 4][: task.epochs]):
        time.sleep(delay)
        report(e, a)
    return {"accuracy": CURVES[task.task_id % 4][task.epochs - 1], "latency_ms": 1.0 + task.task_id}


def always_fails(task, report):
    raise RuntimeError("boom")


def fixed_latency(task, report, latency=0.5):
    time.sleep(latency)
    return {"accuracy": 0.5, "latency_ms": latency * 1e3}


def test_dispatch_prunes_bad_candidates():
    tasks = [HarnessTask(i, "ir", epochs=4) for i in range(4)]
    # task 0 runs first alone so its curve becomes the baseline
    d = Dispatcher(1, scripted)
    board = d.run(tasks, timeout_s=120)
    st = {e.task_id: e.status for e in board.entries.values()}
    assert st[0] == "completed" and st[2] == "completed"
    assert st[1] == "pruned" and st[3] == "pruned"
    assert board.best().task_id == 2 and board.rule.best_curve == CURVES[2]
    assert all(m["type"] == "prune" for m in d.messages) and len(d.messages) == 2


def test_worker_lost_task_rerun_once():
    tasks = [HarnessTask(i, "ir", epochs=1) for i in range(4)]
    board = Dispatcher(2, scripted, rule=PruneRule(0.0), die_on=1).run(tasks, timeout_s=120)  # theta 0: no pruning at epoch 0
    assert sorted(board.entries) == [0, 1, 2, 3]
    assert all(e.status == "completed" for e in board.entries.values())


def test_retry_limit_marks_failed():
    board = Dispatcher(1, always_fails, max_attempts=2).run([HarnessTask(0, "ir")], timeout_s=60)
    assert board.entries[0].status == "failed" and "RuntimeError" in board.entries[0].reason


def test_simulated_worker_scaling():
    """16 simulated workers within 10% of linear.  Steady-state
    throughput: every worker process is started and reports ready before the
    first task (warm_start), each worker then runs 8 fixed-latency tasks."""
    per, lat = 8, 0.1

    def throughput(w):
        d = Dispatcher(w, fixed_latency, warm_start=True, latency=lat)
        board = d.run([HarnessTask(i, "ir") for i in range(per * w)], timeout_s=300)
        assert all(e.status == "completed" for e in board.entries.values())
        return per * w / d.timing["run_s"]

    one = throughput(1)
    for w in (4, 16):
        eff = throughput(w) / (w * one)
        assert eff >= 0.9, (w, eff)


@pytest.mark.gpu
def test_synthetic_accuracy_worker_on_gpu():
    """End to end: two candidates trained by a worker process on the B200
    (CanvasConv2d through the C ABI), accuracy above chance (0.1), latency measured."""
    from paper_2304_07741_b200 import zoo
    from paper_2304_07741_b200.harness import synthetic_accuracy_worker

    tasks = [HarnessTask(0, zoo.SEED7_K1, epochs=3), HarnessTask(1, zoo.SEED7_K1, epochs=3)]
    board = Dispatcher(1, synthetic_accuracy_worker, rule=PruneRule(0.0), steps_per_epoch=20).run(tasks, timeout_s=600)
    for e in board.entries.values():
        assert e.status == "completed", e
        assert e.accuracy > 0.15 and len(e.curve) == 3 and 0 < e.latency_ms < 100
