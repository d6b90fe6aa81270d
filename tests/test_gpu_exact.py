"""Exact-fp64 mode (SGDB_UPLOAD_EXACT_FP64) against the reference itself
(oracle/_ref), on the reference's fp64 fixtures — no fp32 rounding of the
inputs. The device runs the reference's own operation order (the §4
primitive chain for sync, process_examples for Hogwild, glibc's exp), so the
comparisons are BITWISE:

* sync::train / batch_gradient / epoch_batch: models, gradients, norms and
  SVM losses bit-identical; LR losses within 1e-14 (log1p is CUDA's, not
  glibc's).
* hogwild::train with one worker: bit-identical for every access path and
  scope of acceptance criterion 4 (proj/tests/acceptance.cpp:183-220), with
  k-replication, and for numa_dual_train.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LR_LOSS_TOL = 1e-14


def _data(S, layout, n, d, seed, avg=None):
    ds = (S.fixtures.dense_classification(n, d, seed) if avg is None
          else S.fixtures.sparse_classification(n, d, avg, seed))
    return ds if ds.layout == layout else S.convert_layout(ds, layout)


def _exact(S, dev, ds):
    return S.DeviceDataset(dev, ds, exact=True)


def _losses_match(task, got, want):
    got, want = np.asarray(got), np.asarray(want)
    assert got.shape == want.shape
    if task == 1:
        assert np.array_equal(got, want)
    else:
        assert np.all(np.abs(got - want) <= LR_LOSS_TOL * np.abs(want))


SYNC_CASES = [
    # layout, n, d, avg, batch, epochs, decay
    (0, 900, 54, None, 128, 4, 1.0),
    (0, 700, 20, None, 700, 5, 0.9),     # full batch, dense through its transpose
    (1, 600, 30, None, 64, 3, 1.0),
    (2, 1500, 300, 11.0, 256, 3, 0.95),
    (2, 800, 2000, 40.0, 800, 3, 1.0),
    (3, 500, 120, 6.0, 100, 3, 1.0),
]


@pytest.mark.parametrize("layout,n,d,avg,b,epochs,decay", SYNC_CASES)
@pytest.mark.parametrize("task", [0, 1])
def test_sync_train_bitwise(sgdb, ref, dev, layout, n, d, avg, b, epochs, decay, task):
    S = sgdb
    ds = _data(S, S.Layout(layout), n, d, 40 + n, avg)
    alpha = 0.05 if task == 0 else 0.01
    hp = S.Hyperparams(alpha=alpha, batch_b=b, epochs=epochs, task=S.Task(task), step_decay=decay)
    r = S.sync.train(S.Task(task), _exact(S, dev, ds), hp, 1234)
    model, losses, _, div = ref.sync_train(ds, task, alpha, b, epochs, 1234, decay=decay)
    assert not div and not r.trace.diverged
    assert np.array_equal(r.model, model)
    _losses_match(task, r.trace.losses(), losses)


@pytest.mark.parametrize("layout,avg", [(0, None), (1, None), (2, 9.0), (3, 5.0)])
@pytest.mark.parametrize("task", [0, 1])
def test_batch_gradient_and_epoch_batch_bitwise(sgdb, ref, dev, layout, avg, task):
    S = sgdb
    ds = _data(S, S.Layout(layout), 1100, 70, 5, avg)
    dds = _exact(S, dev, ds)
    rng = np.random.default_rng(layout)
    w = rng.standard_normal(70) * 0.2
    rows = np.sort(rng.choice(1100, 300, replace=False)).astype(np.uint32)
    # ref.batch_gradient passes the materialised transpose for DenseRowMajor,
    # as sync::train does.
    transposed = True if layout == 0 else None
    g = S.sync.batch_gradient(S.Task(task), dds, rows, w, transposed=transposed)
    assert np.array_equal(g, ref.batch_gradient(ds, task, rows, w))
    w2 = w.copy()
    norm = S.sync.epoch_batch(S.Task(task), dds, w2, 0.125)
    rw, rnorm = ref.epoch_batch(ds, task, w, 0.125)
    assert np.array_equal(w2, rw) and norm == rnorm


def test_pipeline_criterion_2(sgdb, ref, dev):
    """acceptance criterion 2 (acceptance.cpp:95-136): random fp64 CSR with
    values in (-2, 2), LR batch gradient of the whole set; here bitwise vs the
    reference and within 1e-12 of the summed per-example oracle."""
    S = sgdb
    rng = np.random.default_rng(202)
    for trial in range(3):
        mask = rng.random((50, 20)) < 0.35
        vals = np.where(mask, rng.uniform(-2, 2, (50, 20)), 0.0)
        idx, offs, v = [], [0], []
        for e in range(50):
            nz = np.nonzero(mask[e])[0]
            idx += nz.tolist()
            v += vals[e, nz].tolist()
            offs.append(len(idx))
        labels = np.where(rng.random(50) < 0.5, 1.0, -1.0)
        csr = S.Dataset(50, 20, S.Layout.Csr, labels, np.array(v), np.array(idx, np.uint32),
                        np.array(offs, np.uint64))
        dense = S.convert_layout(csr, S.Layout.DenseRowMajor)
        w = rng.standard_normal(20)
        for ds in (csr, dense):
            g = S.sync.batch_gradient(S.Task.LR, _exact(S, dev, ds), None, w)
            assert np.array_equal(g, ref.batch_gradient(ds, 0, None, w))
            z = vals @ w
            oracle = (vals * (-labels / (1 + np.exp(labels * z)))[:, None]).sum(0)
            assert np.all(np.abs(g - oracle) <= 1e-12 * np.maximum(1, np.abs(oracle)))


# acceptance criterion 4's cases + k-replication.
HOG_CASES = [(0, "row-rr"), (0, "row-ch"), (1, "col-rr"), (1, "col-ch"), (2, "row-rr"),
             (2, "row-ch"), (3, "col-rr"), (3, "col-ch")]


@pytest.mark.parametrize("layout,access", HOG_CASES)
@pytest.mark.parametrize("scope", ["kernel", "thread", "block"])
def test_hogwild_one_worker_bitwise(sgdb, ref, dev, layout, access, scope):
    S = sgdb
    avg = None if layout in (0, 1) else 8.0
    ds = _data(S, S.Layout(layout), 400, 40, 77, avg)
    dds = _exact(S, dev, ds)
    for task, k in ((0, 0), (1, 2)):
        rep = "0" if k == 0 else f"rep-{k}"
        plan = S.parse_plan(f"{access}:{scope}:{rep}")
        plan.workers = 1
        hp = S.Hyperparams(alpha=0.05, batch_b=1, epochs=2, task=S.Task(task))
        r = S.hogwild.train(S.Task(task), dds, hp, plan)
        model, losses, _, evals = ref.hogwild_train(ds, task, 0.05, 2, f"{access}:{scope}:{rep}")
        assert np.array_equal(r.model, model), (task, k)
        _losses_match(task, r.trace.losses(), losses)
        assert r.evals_per_epoch == [int(e) for e in evals]


@pytest.mark.parametrize("layout", [2, 3])
@pytest.mark.parametrize("access", ["row-rr", "row-ch"])
def test_hogwild_example_scope_one_worker_bitwise(sgdb, ref, dev, layout, access):
    """Example-scope replication (async_engine.cpp:266-370), one worker, exact mode."""
    S = sgdb
    ds = _data(S, S.Layout(layout), 400, 40, 78, 8.0)
    dds = _exact(S, dev, ds)
    for task, k in ((0, 0), (1, 2)):
        rep = "0" if k == 0 else f"rep-{k}"
        plan = S.parse_plan(f"{access}:example:{rep}")
        plan.workers = 1
        hp = S.Hyperparams(alpha=0.05, batch_b=1, epochs=3, task=S.Task(task))
        r = S.hogwild.train(S.Task(task), dds, hp, plan)
        model, losses, _, evals = ref.hogwild_train(ds, task, 0.05, 3, f"{access}:example:{rep}")
        assert np.array_equal(r.model, model), (task, k)
        _losses_match(task, r.trace.losses(), losses)
        assert r.evals_per_epoch == [int(e) for e in evals]


def test_numa_dual_one_worker_bitwise(sgdb, ref, dev):
    S = sgdb
    ds = _data(S, S.Layout.Csr, 600, 50, 91, 6.0)
    plan = S.parse_plan("row-rr:kernel:0")
    plan.workers = 1
    hp = S.Hyperparams(alpha=0.02, batch_b=1, epochs=3, task=S.Task.SVM)
    r = S.hogwild.numa_dual_train(S.Task.SVM, _exact(S, dev, ds), hp, plan)
    model, losses, _, _ = ref.hogwild_train(ds, 1, 0.02, 3, "row-rr:kernel:0", dual=True)
    assert np.array_equal(r.model, model)
    assert np.array_equal(np.array(r.trace.losses()), losses)


def test_exact_many_workers_converges(sgdb, ref, dev):
    """With many workers the exact mode is Hogwild in fp64 (racy like the
    reference's relaxed atomics): not bitwise; the final loss must be no
    worse than the reference's multi-threaded run at the same epoch budget
    (+2%; measured ~2.6% lower)."""
    S = sgdb
    ds = _data(S, S.Layout.Csr, 4000, 300, 8, 11.5)
    plan = S.parse_plan("row-ch:kernel:0")
    plan.workers = 8
    hp = S.Hyperparams(alpha=0.01, batch_b=1, epochs=4, task=S.Task.SVM)
    r = S.hogwild.train(S.Task.SVM, _exact(S, dev, ds), hp, plan)
    _, losses, _, _ = ref.hogwild_train(ds, 1, 0.01, 4, "row-ch:kernel:0", workers=8)
    assert r.trace.losses()[-1] <= 1.02 * losses[-1]
