"""Edge cases of the full-batch sparse passes (K2s / K2w / K3s, kernels_sparse.cu;
with the model in SMEM, K2s and K3s run as the phases of one launch, K23g).

The margin pass and the blocked-CSC gradient pass walk each warp's nonzeros
in 256-slot tiles, find segment boundaries in a head bitmap and recover
per-row / per-(block, column) sums with a segmented warp scan; segments cut
between warps are finished in SMEM, empty segments go through ordinal maps.
These inputs put boundaries where that bookkeeping can go wrong: empty rows
(single, in long runs, leading and trailing), one-slot rows (several heads
per lane), rows spanning many tiles and warps, tiny inputs (most warps
empty), a model too wide to stage in shared memory (its margins through the
column-blocked pass K2w, where an empty row is empty in every column block),
and more row blocks than SMs. Full-batch gradients are compared with the CPU
oracle (proj/src/sync_engine.cpp:22-42 restated) at the sync tolerance of
DESIGN.md §Numerics.
"""
import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu


def _csr(S, lengths, d, seed):
    rng = np.random.default_rng(seed)
    rows, idx, val = [0], [], []
    for ln in lengths:
        cols = np.sort(rng.choice(d, size=ln, replace=False)) if ln else np.zeros(0, np.int64)
        idx.extend(cols.tolist())
        val.extend(rng.uniform(-1, 1, ln).astype(np.float32).astype(np.float64).tolist())
        rows.append(rows[-1] + ln)
    n = len(lengths)
    y = np.where(rng.random(n) < 0.5, -1.0, 1.0)
    return S.Dataset(n, d, S.Layout.Csr, labels=y, values=np.array(val, np.float64),
                     indices=np.array(idx, np.uint32), row_offsets=np.array(rows, np.uint64))


def _shapes():
    rng = np.random.default_rng(3)
    out = {}
    out["empty_runs"] = [0] * 40 + [5, 0, 0, 3] + [0] * 70 + [1] * 100 + [0] * 33
    out["one_slot_rows"] = [1] * 3000
    out["mixed_pareto"] = np.minimum(
        (rng.pareto(2.0, 5000) + 1) * 6, 900).astype(int).tolist()
    out["long_rows"] = [700, 0, 1300, 2, 129, 128, 127, 0, 511, 513] * 5
    out["tiny_n"] = [3, 0, 7]
    out["single_row"] = [37]
    out["many_short"] = rng.integers(0, 4, 20000).tolist()
    return out


SHAPES = _shapes()


@pytest.mark.parametrize("name", sorted(SHAPES))
@pytest.mark.parametrize("d", [600, 100_000])
def test_full_batch_gradient_segments(sgdb, dev, orc, name, d):
    """d = 600: K2s (model in SMEM); d = 100,000: the model does not fit in
    SMEM, margins through the column-blocked pass K2w (4 column blocks)."""
    S = sgdb
    lengths = [min(ln, d) for ln in SHAPES[name]]
    ds = _csr(S, lengths, d, seed=len(lengths) + d)
    rng = np.random.default_rng(1)
    w = rng.normal(0, 0.5, d)
    for task in (0, 1):
        g = S.sync.batch_gradient(S.Task(task), ds, None, w, device=dev)
        og = orc.batch_gradient(ds, task, None, w)
        if np.linalg.norm(og) == 0.0:
            assert np.linalg.norm(g) == 0.0
        else:
            assert rel_l2(g, og) <= 1e-5, (name, d, task, rel_l2(g, og))


@pytest.mark.parametrize("name", ["mixed_pareto", "empty_runs", "long_rows"])
@pytest.mark.parametrize("d", [3000, 100_000])
def test_full_batch_epochs_segments(sgdb, dev, orc, name, d):
    """Several B = N epochs (margin pass reads the updated model each time;
    d = 100,000 through K2w's model slices)."""
    S = sgdb
    ds = _csr(S, SHAPES[name], d, seed=5)
    dds = S.DeviceDataset(dev, ds)
    model = S.DeviceModel(dev, ds.n_features)
    om, ol, _ = orc.sync_train(ds, 0, 0.05, ds.n_examples, 4, 7)
    for e in range(4):
        assert S.sync_epoch(dds, model, S.Task.LR, 0.05, None, ds.n_examples)
        assert rel_l2(model.get(), om[e]) <= 1e-5


@pytest.mark.parametrize("d", [500, 100_000])
def test_refresh_rebuilds_full_batch_structures(sgdb, dev, orc, d):
    """sgdb_dataset_refresh_f32 with new values, column ids and row offsets
    (same n, nnz): the head bitmaps, 16-bit ids, the blocked CSC and (d =
    100,000) the column-blocked copy of K2w are rebuilt on the device, so
    full-batch gradients, the mini-batch chunk plan (longest row recomputed)
    and Hogwild all see the new data."""
    S = sgdb
    a = S.fixtures.sparse_classification(3000, d, 12.0, 31).rounded_f32()
    dds = S.DeviceDataset(dev, a)
    model = S.DeviceModel(dev, a.n_features)
    assert S.sync_epoch(dds, model, S.Task.LR, 0.1, None, a.n_examples)
    # Same nnz, different rows: rotate the slots by one row's worth so every
    # row boundary moves, and make one row much longer than any before.
    rng = np.random.default_rng(4)
    nnz = a.values.size
    lens = np.diff(a.row_offsets.astype(np.int64))
    lens = np.roll(lens, 7)
    lens[0] += 200
    lens[1:201] -= np.minimum(lens[1:201] - 1, 1)
    lens[-1] += nnz - lens.sum()
    assert lens.min() >= 0 and lens.sum() == nnz
    rows = np.zeros(a.n_examples + 1, np.uint64)
    np.cumsum(lens, out=rows[1:])
    idx = np.empty(nnz, np.uint32)
    for r in range(a.n_examples):
        lo, hi = int(rows[r]), int(rows[r + 1])
        idx[lo:hi] = np.sort(rng.choice(a.n_features, hi - lo, replace=False))
    vals = rng.uniform(-1, 1, nnz).astype(np.float32)
    labs = np.where(rng.random(a.n_examples) < 0.5, -1.0, 1.0).astype(np.float32)
    b = S.Dataset(a.n_examples, a.n_features, S.Layout.Csr, labels=labs.astype(np.float64),
                  values=vals.astype(np.float64), indices=idx, row_offsets=rows)
    dds.refresh_f32(vals, labs, idx, rows.astype(np.uint32))
    dev.synchronize()
    w = rng.normal(0, 0.3, a.n_features)
    for task in (0, 1):
        g = S.sync.batch_gradient(S.Task(task), dds, None, w, device=dev)
        assert rel_l2(g, orc.batch_gradient(b, task, None, w)) <= 1e-5
        rows_b = np.sort(rng.choice(a.n_examples, 400, replace=False)).astype(np.uint32)
        g = S.sync.batch_gradient(S.Task(task), dds, rows_b, w, device=dev)
        assert rel_l2(g, orc.batch_gradient(b, task, rows_b, w)) <= 1e-5
    m2 = S.DeviceModel(dev, a.n_features)
    sched = S.Schedule(3, a.n_examples)
    om, ol, _ = orc.sync_train(b, 1, 0.05, 256, 2, 3)
    for e in range(2):
        assert S.sync_epoch(dds, m2, S.Task.SVM, 0.05, sched.next(), 256)
        assert rel_l2(m2.get(), om[e]) <= 1e-5


def test_refresh_dense_rebuilds_column_copy(sgdb, dev, orc):
    """Dense refresh invalidates the column-major copy the col-* Hogwild paths
    read: a one-worker col-rr epoch after the refresh trains on
    the new values."""
    S = sgdb
    a = S.fixtures.dense_classification(400, 16, 8).rounded_f32()
    b = S.fixtures.dense_classification(400, 16, 9).rounded_f32()
    col_a = S.convert_layout(a, S.Layout.DenseColMajor)
    dds = S.DeviceDataset(dev, col_a)
    plan = S.parse_plan("col-rr:kernel:0")
    plan.workers = 1
    m = S.DeviceModel(dev, a.n_features)
    S.hogwild_epoch(dds, m, S.Task.LR, 0.05, plan)  # builds the column copy from a
    dds.refresh_f32(np.ascontiguousarray(b.values.astype(np.float32)),
                    np.ascontiguousarray(b.labels.astype(np.float32)))
    m.set(np.zeros(a.n_features))
    S.hogwild_epoch(dds, m, S.Task.LR, 0.05, plan)
    om, _, _ = orc.hogwild_serial(S.convert_layout(b, S.Layout.DenseColMajor), 0, 0.05, 1, 1, 0, 0, 1)
    assert rel_l2(m.get(), om[-1]) <= 1e-4


def test_refresh_rejects_exact_and_padded(sgdb, dev):
    S = sgdb
    a = S.fixtures.sparse_classification(200, 50, 5.0, 2).rounded_f32()
    exact = S.DeviceDataset(dev, a, exact=True)
    with pytest.raises(S.UnsupportedError):
        exact.refresh_f32(np.ascontiguousarray(a.values.astype(np.float32)))
    padded = S.DeviceDataset(dev, S.convert_layout(a, S.Layout.PaddedDense))
    with pytest.raises(S.UnsupportedError):
        padded.refresh_f32(np.ascontiguousarray(a.values.astype(np.float32)))


@pytest.mark.parametrize("nnz_tail", [0, 3])
def test_refresh_idx16_matches_idx32(sgdb, dev, nnz_tail):
    """sgdb_dataset_refresh_idx16 (16-bit ids widened on the device) leaves the
    dataset identical to a 32-bit refresh: one-worker Hogwild epochs and the
    mini-batch sync epochs give bit-identical models."""
    S = sgdb
    ds = S.fixtures.sparse_classification(997 + nnz_tail, 300, 11.65, 57).rounded_f32()
    vals = np.ascontiguousarray(ds.values.astype(np.float32)[::-1].copy())
    idx = np.ascontiguousarray(ds.indices[::-1].astype(np.uint32))
    idx = np.minimum(idx, ds.n_features - 1).astype(np.uint32)
    a, b = S.DeviceDataset(dev, ds), S.DeviceDataset(dev, ds)
    a.refresh_f32(vals, None, idx)
    b.refresh_f32(vals)
    b.refresh_idx16(np.ascontiguousarray(idx.astype(np.uint16)))
    dev.synchronize()
    plan = S.parse_plan("row-ch:kernel:0")
    plan.workers = 1
    ma, mb = S.DeviceModel(dev, ds.n_features), S.DeviceModel(dev, ds.n_features)
    for _ in range(2):
        S.hogwild_epoch(a, ma, S.Task.SVM, 0.01, plan)
        S.hogwild_epoch(b, mb, S.Task.SVM, 0.01, plan)
    np.testing.assert_array_equal(ma.get(), mb.get())
    assert S.sync_epoch(a, ma, S.Task.LR, 0.01, None, 64)
    assert S.sync_epoch(b, mb, S.Task.LR, 0.01, None, 64)
    np.testing.assert_allclose(ma.get(), mb.get(), rtol=1e-12, atol=1e-14)


def test_refresh_idx16_rejects_wide_models(sgdb, dev):
    S = sgdb
    ds = S.fixtures.sparse_classification(50, 70000, 5.0, 3).rounded_f32()
    dds = S.DeviceDataset(dev, ds)
    with pytest.raises(Exception):
        dds.refresh_idx16(np.zeros(ds.nnz, np.uint16))


def test_more_row_blocks_than_sms(sgdb, dev, orc):
    """7.5M rows: more row blocks of the CSC (<= 49,152 rows each) than SMs, so
    the gradient pass runs several waves of CTAs (no co-residency assumed)."""
    S = sgdb
    rng = np.random.default_rng(9)
    n, d = 7_500_000, 40
    lens = rng.integers(1, 4, n)
    rows = np.zeros(n + 1, np.uint64)
    np.cumsum(lens, out=rows[1:])
    nnz = int(rows[-1])
    idx = rng.integers(0, d, nnz).astype(np.uint32)
    # column ids must be unique within a row: take distinct offsets per slot
    pos = np.arange(nnz) - np.repeat(rows[:-1].astype(np.int64), lens)
    idx = ((np.repeat(rng.integers(0, d, n), lens) + pos * 7) % d).astype(np.uint32)
    val = rng.uniform(-1, 1, nnz).astype(np.float32).astype(np.float64)
    y = np.where(rng.random(n) < 0.5, -1.0, 1.0)
    ds = S.Dataset(n, d, S.Layout.Csr, labels=y, values=val, indices=idx, row_offsets=rows)
    w = rng.normal(0, 0.5, d)
    for task in (0, 1):
        g = S.sync.batch_gradient(S.Task(task), ds, None, w, device=dev)
        og = orc.batch_gradient(ds, task, None, w)
        assert rel_l2(g, og) <= 1e-5, (task, rel_l2(g, og))


@pytest.mark.parametrize("n,d", [
    (49_153, 600),      # two row blocks, the second holding one row
    (3_000, 57_000),    # K2s with the model just inside shared memory
    (3_000, 57_700),    # just past it: K2w
    (3_000, 98_305),    # K2w, the last column block holding one column
    (2_000, 1_000_003)])  # K2w, many column blocks, most segments empty (seg_of_ord)
def test_full_batch_block_boundaries(sgdb, dev, orc, n, d):
    """Row / column block boundaries of the blocked passes and the K2s / K2w
    switch, against the oracle for both tasks."""
    S = sgdb
    rng = np.random.default_rng(n + d)
    lengths = rng.integers(0, 9, n).tolist()
    lengths[0], lengths[-1] = 8, 8  # the first and last rows and columns take part
    ds = _csr(S, lengths, d, seed=n + d)
    w = rng.normal(0, 0.5, d)
    for task in (0, 1):
        g = S.sync.batch_gradient(S.Task(task), ds, None, w, device=dev)
        og = orc.batch_gradient(ds, task, None, w)
        assert rel_l2(g, og) <= 1e-5, (n, d, task, rel_l2(g, og))


@pytest.mark.parametrize("d,n,kernels", [
    (600, 5_000, {"k23g_step_kernel"}),                       # model in SMEM: one launch
    (100_000, 5_000, {"k2w_margin_kernel", "k3s_grad_kernel"}),  # wide model: two launches
])
def test_full_batch_step_kernels(sgdb, dev, orc, d, n, kernels):
    """Which kernels one full-batch step launches (the library's per-launch
    profiler), and that the step's model equals the oracle's: the one-launch
    K23g for models that fit in SMEM, K2w -> K3s otherwise. (More row blocks
    than SMs take K2s -> K3s: test_more_row_blocks_than_sms.)"""
    S = sgdb
    rng = np.random.default_rng(21)
    ds = _csr(S, np.minimum((rng.pareto(2.0, n) + 1) * 6, 400).astype(int).tolist(), d, 22)
    w0 = rng.normal(0, 0.3, d)
    dds = S.DeviceDataset(dev, ds)
    m = S.DeviceModel(dev, d, init=w0)
    S.sync_epoch(dds, m, S.Task.LR, 0.05, None, n)  # builds the structures
    m.set(w0)
    dev.set_profiling(True)
    S.sync_epoch(dds, m, S.Task.LR, 0.05, None, n)
    stats = dev.kernel_stats()
    dev.set_profiling(False)
    step = {k for k in stats if k.startswith(("k2", "k3"))}
    assert step == kernels, stats
    om, _, _ = orc.sync_train(ds, 0, 0.05, n, 1, 5, init=w0)
    assert rel_l2(m.get(), om[0]) <= 1e-5
