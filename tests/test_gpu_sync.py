"""GPU parity of the synchronous engine against the CPU oracle.

Mirrors proj/tests/test_sync_engine.cpp and acceptance criteria 2-3
(proj/tests/acceptance.cpp:95-166). The reference asserts bitwise equality
between CPU code paths; the device computes in fp32 with fp64 reductions, so
each bitwise check becomes the stated fp32 tolerance below (DESIGN.md
§Numerics). All inputs are rounded to fp32 before the oracle sees them, so
only arithmetic differs.

Tolerances (BASELINE.json north star: "rel 1e-4"; we hold the tighter):
  per-epoch model rel-L2 <= 1e-5, per-epoch loss rel <= 1e-6.
"""
import numpy as np
import pytest

from conftest import rel, rel_l2

pytestmark = pytest.mark.gpu

MODEL_TOL = 1e-5
LOSS_TOL = 1e-6


def _run_epochs(S, dev, ds, task, alpha, batch_b, epochs, seed, shuffle=True):
    """sync::train's loop driven through the device ops, capturing every epoch's model."""
    dds = S.DeviceDataset(dev, ds)
    model = S.DeviceModel(dev, ds.n_features)
    sched = S.Schedule(seed, ds.n_examples, shuffle)
    models, losses = [], []
    for e in range(1, epochs + 1):
        order = sched.next()
        a = S.Hyperparams(alpha=alpha).step_size(e)
        finite = S.sync_epoch(dds, model, task, a, order if batch_b < ds.n_examples else None,
                              batch_b)
        assert finite
        models.append(model.get())
        losses.append(S.device_loss(dds, model, task))
    return np.array(models), np.array(losses)


CASES = [
    # (kind, n, d, avg_nnz, seed)
    ("dense", 2000, 54, None, 11),
    ("dense", 777, 7, None, 12),
    ("dense", 1500, 300, None, 13),
    ("dense", 600, 1000, None, 14),
    ("sparse", 3000, 300, 11.65, 15),
    ("sparse", 2000, 2000, 50.0, 16),
    ("sparse", 500, 40000, 200.0, 17),
]


def _make(S, kind, n, d, avg, seed):
    if kind == "dense":
        return S.fixtures.dense_classification(n, d, seed).rounded_f32()
    return S.fixtures.sparse_classification(n, d, avg, seed).rounded_f32()


@pytest.mark.parametrize("kind,n,d,avg,seed", CASES)
@pytest.mark.parametrize("task", [0, 1])
@pytest.mark.parametrize("batch", ["N", 64])
def test_per_epoch_parity(sgdb, dev, orc, kind, n, d, avg, seed, task, batch):
    S = sgdb
    ds = _make(S, kind, n, d, avg, seed)
    b = ds.n_examples if batch == "N" else batch
    alpha = 1.0 / b  # well inside the 2/L stability bound for these fixtures
    epochs = 6
    gm, gl = _run_epochs(S, dev, ds, S.Task(task), alpha, b, epochs, seed=7)
    om, ol, div = orc.sync_train(ds, task, alpha, b, epochs, 7)
    assert not div
    for e in range(epochs):
        assert rel_l2(gm[e], om[e]) <= MODEL_TOL, (e, rel_l2(gm[e], om[e]))
        assert rel(gl[e], ol[e]) <= LOSS_TOL, (e, gl[e], ol[e])


def test_whole_run_train_matches_oracle(sgdb, orc):
    S = sgdb
    ds = S.fixtures.dense_classification(5000, 54, 20250810).rounded_f32()
    hp = S.Hyperparams(alpha=2e-4, batch_b=256, epochs=8, task=S.Task.LR)
    r = S.sync.train(S.Task.LR, ds, hp, 4242)
    om, ol, _ = orc.sync_train(ds, 0, 2e-4, 256, 8, 4242)
    assert len(r.trace.epochs) == 8
    assert rel_l2(r.model, om[-1]) <= MODEL_TOL
    for e in range(8):
        assert rel(r.trace.epochs[e].loss, ol[e]) <= LOSS_TOL
        assert r.trace.epochs[e].seconds > 0.0


def test_reference_binary_parity(sgdb, ref):
    """The restatement is pinned to the reference elsewhere; here the device is
    compared straight against the unmodified reference's sync::train."""
    S = sgdb
    ds = S.fixtures.sparse_classification(4000, 500, 20.0, 99).rounded_f32()
    hp = S.Hyperparams(alpha=0.02, batch_b=100, epochs=5, task=S.Task.SVM)
    r = S.sync.train(S.Task.SVM, ds, hp, 99)
    model, losses, _, div = ref.sync_train(ds, 1, 0.02, 100, 5, 99)
    assert rel_l2(r.model, model) <= MODEL_TOL
    for e in range(5):
        assert rel(r.trace.epochs[e].loss, losses[e]) <= LOSS_TOL


@pytest.mark.parametrize("kind", ["dense", "sparse"])
def test_batch_gradient_matches_oracle(sgdb, dev, orc, kind):
    S = sgdb
    ds = (S.fixtures.dense_classification(3000, 64, 3) if kind == "dense"
          else S.fixtures.sparse_classification(3000, 800, 30.0, 3)).rounded_f32()
    rng = np.random.default_rng(0)
    w = rng.normal(0, 0.3, ds.n_features)
    for task in (0, 1):
        for rows in (None, np.sort(rng.choice(ds.n_examples, 777, replace=False)).astype(np.uint32)):
            g = S.sync.batch_gradient(S.Task(task), ds, rows, w, device=dev)
            og = orc.batch_gradient(ds, task, rows, w)
            assert rel_l2(g, og) <= 1e-5


def test_epoch_batch_zero_model_closed_forms(sgdb, dev):
    """test_sync_engine.cpp:23-42: at w=0 the SVM step is alpha*sum(y x); LR carries 1/2."""
    S = sgdb
    ds = S.fixtures.sparse_classification(30, 12, 4.0, 5).rounded_f32()
    expected = np.zeros(ds.n_features)
    for e in range(ds.n_examples):
        for s in range(int(ds.row_offsets[e]), int(ds.row_offsets[e + 1])):
            expected[ds.indices[s]] += ds.labels[e] * ds.values[s]
    w = np.zeros(ds.n_features)
    S.sync.epoch_batch(S.Task.SVM, ds, w, 0.5, device=dev)
    np.testing.assert_allclose(w, 0.5 * expected, rtol=1e-6, atol=1e-7)
    wlr = np.zeros(ds.n_features)
    S.sync.epoch_batch(S.Task.LR, ds, wlr, 0.5, device=dev)
    np.testing.assert_allclose(wlr, 0.25 * expected, rtol=1e-6, atol=1e-7)


def test_epoch_batch_norm(sgdb, dev, ref):
    S = sgdb
    ds = S.fixtures.dense_classification(900, 20, 8).rounded_f32()
    w0 = np.random.default_rng(1).normal(0, 0.5, ds.n_features)
    w = w0.copy()
    norm = S.sync.epoch_batch(S.Task.LR, ds, w, 0.125, device=dev)
    rw, rnorm = ref.epoch_batch(ds, 0, w0, 0.125)
    assert rel(norm, rnorm) <= 1e-5
    assert rel_l2(w, rw) <= 1e-6


def test_train_b_equals_n_reduces_to_epoch_batch(sgdb, dev):
    """test_sync_engine.cpp:69-82 (bitwise there; identical kernels here, so bitwise too)."""
    S = sgdb
    ds = S.fixtures.dense_classification(60, 8, 3).rounded_f32()
    hp = S.Hyperparams(alpha=0.05, batch_b=ds.n_examples, epochs=4, task=S.Task.LR)
    r = S.sync.train(S.Task.LR, ds, hp, 123, device=dev)
    w = np.zeros(ds.n_features)
    for _ in range(4):
        S.sync.epoch_batch(S.Task.LR, ds, w, 0.05, device=dev)
    np.testing.assert_array_equal(r.model, w)


def test_divergence_is_reported(sgdb, dev):
    """test_sync_engine.cpp:159-170."""
    S = sgdb
    ds = S.fixtures.dense_classification(50, 6, 23)
    hp = S.Hyperparams(alpha=1e308, batch_b=ds.n_examples, epochs=200, task=S.Task.LR)
    r = S.sync.train(S.Task.LR, ds, hp, 3, device=dev)
    assert r.trace.diverged
    assert r.trace.divergence_note
    assert len(r.trace.epochs) < 200


def test_divergence_stops_minibatch_epoch(sgdb, dev):
    S = sgdb
    ds = S.fixtures.sparse_classification(400, 50, 5.0, 2)
    hp = S.Hyperparams(alpha=1e308, batch_b=16, epochs=50, task=S.Task.LR)
    r = S.sync.train(S.Task.LR, ds, hp, 3, device=dev)
    assert r.trace.diverged and len(r.trace.epochs) < 50


def test_divergence_stops_dense_minibatch_epoch(sgdb, dev):
    """Dense mini-batch epochs run as one persistent kernel (K1c): a non-finite
    gradient must stop every CTA at the same step and be reported."""
    S = sgdb
    ds = S.fixtures.dense_classification(3000, 40, 4)
    hp = S.Hyperparams(alpha=1e308, batch_b=64, epochs=50, task=S.Task.LR)
    r = S.sync.train(S.Task.LR, ds, hp, 3, device=dev)
    assert r.trace.diverged and len(r.trace.epochs) < 50
    assert "non-finite" in r.trace.divergence_note


def test_epoch_timing_excludes_loss_and_hook(sgdb, dev):
    """test_sync_engine.cpp:172-192: every clock read advances 0.25 s; the hook 1000 s."""
    S = sgdb
    ds = S.fixtures.dense_classification(40, 6, 29)
    now = [0.0]

    def clock():
        now[0] += 0.25
        return now[0]

    def hook(epoch, loss):
        now[0] += 1000.0

    hp = S.Hyperparams(alpha=0.01, batch_b=ds.n_examples, epochs=3, task=S.Task.SVM)
    r = S.sync.train(S.Task.SVM, ds, hp, 0, S.TrainOptions(clock=clock, epoch_hook=hook),
                     device=dev)
    assert len(r.trace.epochs) == 3
    assert all(e.seconds == 0.25 for e in r.trace.epochs)


def test_empty_dataset_is_an_error(sgdb, dev):
    S = sgdb
    empty = S.Dataset(0, 0, S.Layout.Csr, row_offsets=np.zeros(1, np.uint64))
    with pytest.raises(ValueError):
        S.sync.train(S.Task.LR, empty, S.Hyperparams(batch_b=1), 0, device=dev)


def test_monotone_batch_gd(sgdb, dev):
    """test_sync_engine.cpp:132-157: batch GD is non-increasing once alpha is small."""
    S = sgdb
    ds = S.fixtures.sparse_classification(50, 10, 3.0, 31)
    for task in (S.Task.LR, S.Task.SVM):
        alpha, ok = 1.0, False
        for _ in range(40):
            hp = S.Hyperparams(alpha=alpha, batch_b=ds.n_examples, epochs=25, task=task)
            r = S.sync.train(task, ds, hp, 1, device=dev)
            alpha /= 2
            if r.trace.diverged:
                continue
            prev = S.dataset_loss(task, ds, np.zeros(ds.n_features), device=dev)
            ok = all(e.loss <= prev + 1e-9 * max(1, abs(prev)) or False for e in r.trace.epochs[:1])
            losses = [prev] + r.trace.losses()
            ok = all(b <= a + 1e-6 * abs(a) for a, b in zip(losses, losses[1:]))
            if ok:
                break
        assert ok


def test_loss_matches_oracle(sgdb, dev, orc):
    S = sgdb
    for ds in (S.fixtures.dense_classification(3333, 54, 1).rounded_f32(),
               S.fixtures.sparse_classification(2222, 5000, 40.0, 2).rounded_f32()):
        w = np.random.default_rng(3).normal(0, 1, ds.n_features)
        for task in (0, 1):
            gl = S.dataset_loss(S.Task(task), ds, w, device=dev)
            assert rel(gl, orc.dataset_loss(ds, task, w)) <= 1e-12


def test_padded_and_colmajor_inputs(sgdb, dev, orc):
    """Every input layout trains to the same result (conversion preserves content)."""
    S = sgdb
    csr = S.fixtures.sparse_classification(700, 90, 8.0, 4).rounded_f32()
    padded = S.convert_layout(csr, S.Layout.PaddedDense)
    dense = S.fixtures.dense_classification(500, 30, 5).rounded_f32()
    dcol = S.convert_layout(dense, S.Layout.DenseColMajor)
    for a, b in ((csr, padded), (dense, dcol)):
        hp = S.Hyperparams(alpha=0.01, batch_b=50, epochs=3, task=S.Task.LR)
        ra = S.sync.train(S.Task.LR, a, hp, 5, device=dev)
        rb = S.sync.train(S.Task.LR, b, hp, 5, device=dev)
        assert rel_l2(ra.model, rb.model) <= 1e-6


def _heavy_tailed(S, n, d, seed):
    """CSR rows with a heavy tail (a few rows many chunks long) and empty rows:
    the chunked mini-batch kernels (K3c) cut rows into chunks of G*4 slots."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, 40, n)
    lens[rng.choice(n, 6, replace=False)] = rng.integers(600, 3000, 6)
    lens[rng.choice(n, 25, replace=False)] = 0
    idx, val, offs = [], [], [0]
    for ln in lens:
        cols = np.sort(rng.choice(d, int(ln), replace=False))
        idx.extend(cols.tolist())
        val.extend(rng.normal(0, 0.5, int(ln)).tolist())
        offs.append(len(idx))
    labels = np.where(rng.random(n) < 0.5, 1.0, -1.0)
    return S.Dataset(n, d, S.Layout.Csr, labels, np.array(val), np.array(idx, np.uint32),
                     np.array(offs, np.uint64)).rounded_f32()


@pytest.mark.parametrize("batch", [37, 256])
@pytest.mark.parametrize("task", [0, 1])
def test_minibatch_heavy_tailed_rows(sgdb, dev, orc, batch, task):
    S = sgdb
    ds = _heavy_tailed(S, 1500, 5000, 29 + task)
    alpha = 0.5 / batch
    gm, gl = _run_epochs(S, dev, ds, S.Task(task), alpha, batch, 4, seed=3)
    om, ol, div = orc.sync_train(ds, task, alpha, batch, 4, 3)
    assert not div
    for e in range(4):
        assert rel_l2(gm[e], om[e]) <= MODEL_TOL, (e, rel_l2(gm[e], om[e]))
        assert rel(gl[e], ol[e]) <= LOSS_TOL, (e, gl[e], ol[e])


def test_minibatch_heavy_tailed_batch_gradient_repeats(sgdb, dev, orc):
    """Operator API with repeated and unsorted ids over heavy-tailed rows."""
    S = sgdb
    ds = _heavy_tailed(S, 900, 3000, 41)
    rng = np.random.default_rng(5)
    w = rng.normal(0, 0.2, ds.n_features)
    lens = np.diff(ds.row_offsets.astype(np.int64))
    heavy = np.argsort(lens)[-3:].astype(np.uint32)
    # random repeats (fits the per-chunk table) and the longest rows repeated
    # past the table's capacity (the kernels fall back to the owner search)
    for rows in (rng.integers(0, ds.n_examples, 700).astype(np.uint32), np.tile(heavy, 150)):
        for task in (0, 1):
            g = S.sync.batch_gradient(S.Task(task), ds, rows, w, device=dev)
            og = orc.batch_gradient(ds, task, rows, w)
            assert rel_l2(g, og) <= 1e-5
