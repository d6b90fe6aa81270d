"""GPU parity of the Hogwild kernels against the CPU oracle.

Mirrors proj/tests/test_async_engine.cpp and acceptance criteria 4-6
(proj/tests/acceptance.cpp:170-312). One worker (one lane group) reproduces
sequential Alg. 3 up to fp32 arithmetic; independent replicas (thread scope,
dual instances) are deterministic and match the serialized oracle; racing
workers are checked on the loss curve (acceptance 5's template).

Tolerances: model rel-L2 <= 1e-4 and loss rel <= 1e-5 for deterministic
schedules (the device keeps the Hogwild model in fp32, as the paper's GPU
kernel does, so rounding accumulates per update; measured ~1e-6).
"""
import numpy as np
import pytest

from conftest import rel, rel_l2

pytestmark = pytest.mark.gpu

MODEL_TOL = 1e-4
LOSS_TOL = 1e-5

RR = {"row-rr": 1, "row-ch": 0, "col-rr": 1, "col-ch": 0}
REPL = {"kernel": 0, "block": 1, "thread": 2}


def _inc(S, task, alpha, epochs, decay=1.0):
    return S.Hyperparams(alpha=alpha, batch_b=1, epochs=epochs, task=task, step_decay=decay)


@pytest.fixture(scope="module")
def datasets(sgdb):
    S = sgdb
    csr = S.fixtures.sparse_classification(60, 20, 4.0, 3).rounded_f32()
    dense_row = S.fixtures.dense_classification(50, 7, 4).rounded_f32()
    return {
        "csr": csr,
        "padded": S.convert_layout(csr, S.Layout.PaddedDense),
        "dense_row": dense_row,
        "dense_col": S.convert_layout(dense_row, S.Layout.DenseColMajor),
    }


CASES = [("csr", "row-rr:kernel:0"), ("csr", "row-ch:kernel:0"), ("csr", "row-rr:thread:0"),
         ("csr", "row-ch:block:0"), ("padded", "col-rr:kernel:0"), ("padded", "col-ch:kernel:0"),
         ("dense_row", "row-rr:kernel:0"), ("dense_row", "row-ch:thread:0"),
         ("dense_col", "col-rr:kernel:0"), ("dense_col", "col-ch:block:0"),
         ("csr", "row-ch:kernel:3"), ("dense_row", "row-rr:block:2")]


@pytest.mark.parametrize("name,plan_text", CASES)
@pytest.mark.parametrize("task", [0, 1])
@pytest.mark.parametrize("lanes", [0, 1, 32])
def test_one_worker_equals_sequential(sgdb, dev, orc, datasets, name, plan_text, task, lanes):
    """test_async_engine.cpp:99-128 / acceptance 4 (bitwise there, fp32 tolerance here)."""
    S = sgdb
    ds = datasets[name]
    plan = S.parse_plan(plan_text)
    plan.workers = 1
    plan.lanes_per_worker = lanes
    r = S.hogwild.train(S.Task(task), ds, _inc(S, S.Task(task), 0.05, 3), plan, 0, device=dev)
    access, repl, k = plan_text.split(":")
    om, ol, ev = orc.hogwild_serial(ds, task, 0.05, 3, RR[access], REPL[repl], int(k), 1)
    assert rel_l2(r.model, om[-1]) <= MODEL_TOL
    for e in range(3):
        assert rel(r.trace.epochs[e].loss, ol[e]) <= LOSS_TOL
    assert r.evals_per_epoch == [int(x) for x in ev]


@pytest.mark.parametrize("workers,gs", [(2, 32), (7, 32), (64, 8), (300, 32)])
def test_thread_scope_equals_serialized_partitions(sgdb, dev, orc, workers, gs):
    """test_async_engine.cpp:187-215: per-worker replicas never interact within an
    epoch, so T workers equal T sequential partition runs merged by mean."""
    S = sgdb
    ds = S.fixtures.sparse_classification(2000, 300, 12.0, 8).rounded_f32()
    plan = S.parse_plan("row-ch:thread:0")
    plan.workers = workers
    r = S.hogwild.train(S.Task.LR, ds, _inc(S, S.Task.LR, 0.07, 3), plan, 0, device=dev)
    om, ol, _ = orc.hogwild_serial(ds, 0, 0.07, 3, 0, 2, 0, workers)
    assert rel_l2(r.model, om[-1]) <= MODEL_TOL
    for e in range(3):
        assert rel(r.trace.epochs[e].loss, ol[e]) <= LOSS_TOL


@pytest.mark.parametrize("plan_text", ["row-ch:block:0", "row-rr:block:2"])
def test_block_scope_one_worker_per_group_is_deterministic(sgdb, dev, orc, plan_text):
    """group_size 1: every replica has a single worker -> equals the serialized oracle."""
    S = sgdb
    ds = S.fixtures.sparse_classification(3000, 47236 // 4, 30.0, 9).rounded_f32()
    plan = S.parse_plan(plan_text)
    plan.workers, plan.group_size = 40, 1
    r = S.hogwild.train(S.Task.SVM, ds, _inc(S, S.Task.SVM, 0.05, 2), plan, 0, device=dev)
    om, ol, _ = orc.hogwild_serial(ds, 1, 0.05, 2, RR[plan_text.split(":")[0]], 1,
                                   int(plan_text.split(":")[2]), 40, group_size=1)
    assert rel_l2(r.model, om[-1]) <= MODEL_TOL
    assert rel(r.trace.final_loss(), ol[-1]) <= LOSS_TOL


def test_block_scope_global_replicas(sgdb, dev, orc):
    """A model too large for shared memory takes the global-replica path."""
    S = sgdb
    ds = S.fixtures.sparse_classification(800, 200000, 30.0, 10).rounded_f32()
    plan = S.parse_plan("row-ch:block:0")
    plan.workers, plan.group_size = 16, 1
    r = S.hogwild.train(S.Task.LR, ds, _inc(S, S.Task.LR, 0.1, 2), plan, 0, device=dev)
    om, ol, _ = orc.hogwild_serial(ds, 0, 0.1, 2, 0, 1, 0, 16, group_size=1)
    assert rel_l2(r.model, om[-1]) <= MODEL_TOL


def test_evals_per_epoch(sgdb, dev):
    """test_async_engine.cpp:301-311 / acceptance 6: evals = n + T*k."""
    S = sgdb
    ds = S.fixtures.sparse_classification(64, 16, 3.0, 16)
    for k in (0, 2, 5, 10):
        plan = S.parse_plan(f"row-ch:kernel:{k}")
        plan.workers = 4
        r = S.hogwild.train(S.Task.LR, ds, _inc(S, S.Task.LR, 0.02, 3), plan, 0, device=dev)
        assert r.evals_per_epoch == [64 + 4 * k] * 3


def test_dual_equals_single(sgdb, dev):
    """test_async_engine.cpp:273-299."""
    S = sgdb
    ds = S.fixtures.sparse_classification(40, 12, 3.0, 14)
    plan = S.parse_plan("row-ch:kernel:0")
    dual = S.hogwild.numa_dual_train(S.Task.LR, ds, _inc(S, S.Task.LR, 0.08, 4), plan, 0, device=dev)
    single = S.hogwild.train(S.Task.LR, ds, _inc(S, S.Task.LR, 0.08, 4), plan, 0, device=dev)
    np.testing.assert_array_equal(dual.model, single.model)
    assert dual.trace.losses() == single.trace.losses()
    assert dual.evals_per_epoch[0] == 2 * ds.n_examples
    plan.merge_period_epochs = 0
    dual = S.hogwild.numa_dual_train(S.Task.SVM, ds, _inc(S, S.Task.SVM, 0.05, 3), plan, 0, device=dev)
    single = S.hogwild.train(S.Task.SVM, ds, _inc(S, S.Task.SVM, 0.05, 3), plan, 0, device=dev)
    np.testing.assert_array_equal(dual.model, single.model)


def test_invalid_plan_layout_rejected(sgdb, dev):
    S = sgdb
    csr = S.fixtures.sparse_classification(10, 5, 2.0, 19)
    plan = S.parse_plan("col-rr:kernel:0")
    with pytest.raises(ValueError):
        S.hogwild.train(S.Task.LR, csr, _inc(S, S.Task.LR, 0.1, 1), plan, 0, device=dev)


@pytest.mark.parametrize("name,plan_text", [("csr", "row-ch:example:0"), ("csr", "row-rr:example:0"),
                                             ("padded", "row-ch:example:0"), ("csr", "row-ch:example:3")])
@pytest.mark.parametrize("task", [0, 1])
@pytest.mark.parametrize("lanes", [1, 32])
def test_example_scope_one_worker_matches_reference(sgdb, dev, ref, datasets, name, plan_text, task,
                                                    lanes):
    """Example-scope replication (async_engine.cpp:266-370) with one worker is
    deterministic: every example's replica starts from the epoch-start model,
    and the shared model takes the replicas in list order at the end of the
    epoch. Compared with the unmodified reference's hogwild::train."""
    S = sgdb
    ds = datasets[name]
    plan = S.parse_plan(plan_text)
    plan.workers = 1
    plan.lanes_per_worker = lanes
    alpha, epochs = 0.1, 4
    r = S.hogwild.train(S.Task(task), ds, _inc(S, S.Task(task), alpha, epochs), plan, 0, device=dev)
    model, losses, _, evals = ref.hogwild_train(ds, task, alpha, epochs, plan_text, workers=1)
    assert rel_l2(r.model, model) <= MODEL_TOL, rel_l2(r.model, model)
    for e in range(epochs):
        assert rel(r.trace.epochs[e].loss, losses[e]) <= LOSS_TOL
    assert list(r.evals_per_epoch) == [int(x) for x in evals]


def test_example_scope_racing_workers_converge(sgdb, dev, ref):
    """Racing workers with example replicas (and k-rep duplicates claimed by
    two workers). The result depends on when replicas are initialised relative
    to other workers' end-of-list stores: a single worker initialises every
    replica from the epoch-start model, the reference's staggered threads let
    later replicas see earlier stores. Every interleaving is legal, so the
    device's final loss must fall within that range (10 % slack either side)."""
    S = sgdb
    ds = S.fixtures.sparse_classification(3000, 400, 12.0, 23).rounded_f32()
    plan = S.parse_plan("row-ch:example:2")
    plan.workers = 8
    hp = _inc(S, S.Task.SVM, 0.05, 8)
    r = S.hogwild.train(S.Task.SVM, ds, hp, plan, 0, device=dev)
    _, ref1, _, _ = ref.hogwild_train(ds, 1, 0.05, 8, "row-ch:example:2", workers=1)
    _, ref8, _, _ = ref.hogwild_train(ds, 1, 0.05, 8, "row-ch:example:2", workers=8)
    losses = r.trace.losses()
    assert all(np.isfinite(losses)) and losses[-1] < losses[0]
    lo, hi = min(ref1[-1], ref8[-1]), max(ref1[-1], ref8[-1])
    assert 0.9 * lo <= losses[-1] <= 1.1 * hi, (losses[-1], ref1[-1], ref8[-1])
    assert r.evals_per_epoch[0] == ds.n_examples + 8 * 2


@pytest.fixture(scope="module")
def acceptance5(sgdb, dev):
    """Acceptance 5's fixture and L* (acceptance.cpp:222-240): sparse 20000x10000
    avg 50, L* = best sync batch-GD loss over alpha in {1e-4..1}, 60 epochs."""
    S = sgdb
    ds = S.fixtures.sparse_classification(20000, 10000, 50.0, 20250810, 0.1)
    dds = S.DeviceDataset(dev, ds)
    l_star = np.inf
    for alpha in (1e-4, 1e-3, 1e-2, 1e-1, 1.0):
        hp = S.Hyperparams(alpha=alpha, batch_b=ds.n_examples, epochs=60, task=S.Task.SVM)
        r = S.sync.train(S.Task.SVM, dds, hp, 0)
        l_star = min([l_star] + [x for x in r.trace.losses() if np.isfinite(x)])
    hp = _inc(S, S.Task.SVM, 0.5, 60, 0.93)
    e1 = _epochs_to(S.hogwild.train(S.Task.SVM, dds, hp, S.parse_plan("row-ch:kernel:0"),
                                    0).trace.losses(), l_star)
    assert e1 is not None
    return dds, l_star, e1


def _epochs_to(losses, l_star, tol=0.01):
    for i, loss in enumerate(losses):
        if loss <= (1 + tol) * l_star:
            return i + 1
    return None


@pytest.mark.parametrize("plan_text,lanes", [("row-ch:kernel:0", 0), ("row-ch:kernel:0", 8),
                                             ("row-rr:kernel:0", 0), ("row-ch:kernel:10", 0)])
def test_acceptance5_eight_workers(sgdb, acceptance5, plan_text, lanes):
    """Acceptance 5 verbatim: SVM alpha 0.5 decay 0.93, 60 epochs, 8 racing
    workers reach 1% of L* within 3x the epochs one worker needs."""
    S = sgdb
    dds, l_star, e1 = acceptance5
    plan = S.parse_plan(plan_text)
    plan.workers = 8
    plan.lanes_per_worker = lanes
    r = S.hogwild.train(S.Task.SVM, dds, _inc(S, S.Task.SVM, 0.5, 60, 0.93), plan, 0)
    en = _epochs_to(r.trace.losses(), l_star)
    assert en is not None and en <= 3 * e1, (en, e1)


@pytest.mark.parametrize("workers,gs,lanes", [(4096, 2048, 0), (4096, 2048, 32), (64, 32, 0),
                                              (8, 4, 0), (4736, 32, 0)])
def test_block_scope_loss_curve_tracks_oracle(sgdb, dev, orc, workers, gs, lanes):
    """Block scope with racing workers per replica (async_engine.cpp:293-331):
    the per-epoch loss curve stays within 2% above the serialized-worker oracle
    (one legal Hogwild interleaving) on acceptance 5's fixture. R = workers /
    gs replicas: 148 (one per SM, shared-memory replicas, K6) or fewer
    (replicas in L2 shared by all resident warps, K6g)."""
    S = sgdb
    ds = S.fixtures.sparse_classification(20000, 10000, 50.0, 20250810).rounded_f32()
    plan = S.parse_plan("row-ch:block:0")
    plan.workers, plan.group_size, plan.lanes_per_worker = workers, gs, lanes
    r = S.hogwild.train(S.Task.SVM, ds, _inc(S, S.Task.SVM, 0.1, 5, 0.97), plan, 0, device=dev)
    _, ol, _ = orc.hogwild_serial(ds, 1, 0.1, 5, 0, 1, 0, workers, group_size=gs, decay=0.97)
    for e in range(5):
        # red.add replicas lose no updates, so racing runs may converge faster
        # than the serialized interleaving: the bound is one-sided.
        assert r.trace.epochs[e].loss <= 1.02 * ol[e], (e, r.trace.losses(), list(ol))


@pytest.mark.parametrize("plan_text,workers,gs", [("row-ch:kernel:0", 4096, 32),
                                                  ("row-rr:kernel:0", 4096, 32)])
def test_gpu_scale_workers_converge(sgdb, acceptance5, plan_text, workers, gs):
    """GPU-scale concurrency (thousands of lane groups racing on one model) is
    a different operating point from 8 CPU threads: as the paper reports
    (§6, Table tbl:asynch-sgd), the step size must be re-tuned. With
    the best alpha of a small grid the run reaches 1% of L* within 60 epochs."""
    S = sgdb
    dds, l_star, e1 = acceptance5
    best = None
    for alpha in (0.5, 0.1, 0.02, 0.005):
        plan = S.parse_plan(plan_text)
        plan.workers, plan.group_size = workers, gs
        r = S.hogwild.train(S.Task.SVM, dds, _inc(S, S.Task.SVM, alpha, 60, 0.93), plan, 0)
        en = _epochs_to(r.trace.losses(), l_star)
        if en is not None and (best is None or en < best):
            best = en
    assert best is not None and best <= 60


@pytest.mark.parametrize("task", [0, 1])
def test_long_rows_one_worker_equals_sequential(sgdb, dev, orc, task):
    """Rows of hundreds of slots select the LONG kernel variant (two slot
    batches per round trip, K5); one worker is still sequential
    Alg. 3 (same tolerance as the other one-worker cases)."""
    S = sgdb
    ds = S.fixtures.sparse_classification(120, 3000, 400.0, 41).rounded_f32()
    assert ds.values.size / ds.n_examples >= 256
    plan = S.parse_plan("row-ch:kernel:0")
    plan.workers = 1
    hp = _inc(S, S.Task(task), 0.01, 3)
    r = S.hogwild.train(S.Task(task), ds, hp, plan, 0, device=dev)
    om, ol, _ = orc.hogwild_serial(ds, task, 0.01, 3, 0, 0, 0, 1)
    for e in range(3):
        assert rel(r.trace.epochs[e].loss, ol[e]) <= LOSS_TOL, (e, r.trace.epochs[e].loss, ol[e])
    assert rel_l2(r.model, om[-1]) <= MODEL_TOL
