"""Edge cases of the full-batch sparse passes (segmented warp stream, K2t/K3t).

The margin pass and the blocked-CSC gradient pass walk each warp's nonzeros
in 128-slot tiles and recover per-row / per-column sums with a segmented warp
scan (paper_1802_08800_b200/csrc/segstream.cuh). These inputs put segment
boundaries where that bookkeeping can go wrong: empty rows (single, in runs
longer than the 32-entry pointer chunk, leading and trailing), one-slot rows,
more rows in one tile than a chunk holds, rows spanning many tiles, and a
model too wide to stage in shared memory. Full-batch gradients are compared
with the CPU oracle (proj/src/sync_engine.cpp:22-42 restated) at the sync
tolerance of DESIGN.md §Numerics.
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
@pytest.mark.parametrize("split", ["0", "1"])
def test_full_batch_gradient_segments(sgdb, dev, orc, name, d, split, monkeypatch):
    """split=1: warps take equal nonzero ranges and rows cut by warp boundaries
    are finished from per-warp pieces; split=0: whole rows per warp."""
    monkeypatch.setenv("SGDB_SEG_SPLIT", split)
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
def test_full_batch_epochs_segments(sgdb, dev, orc, name):
    """Several B = N epochs (margin pass reads the updated model each time)."""
    S = sgdb
    ds = _csr(S, SHAPES[name], 3000, seed=5)
    dds = S.DeviceDataset(dev, ds)
    model = S.DeviceModel(dev, ds.n_features)
    om, ol, _ = orc.sync_train(ds, 0, 0.05, ds.n_examples, 4, 7)
    for e in range(4):
        assert S.sync_epoch(dds, model, S.Task.LR, 0.05, None, ds.n_examples)
        assert rel_l2(model.get(), om[e]) <= 1e-5


def test_refresh_drops_csc_copy(sgdb, dev):
    """sgdb_dataset_refresh_f32 re-copies CSR arrays but not the row-blocked CSC
    copy built at upload: full-batch sync must fail loudly afterwards (not read
    stale values), while Hogwild and a fresh upload keep working."""
    S = sgdb
    ds = S.fixtures.sparse_classification(500, 80, 6.0, 31).rounded_f32()
    dds = S.DeviceDataset(dev, ds)
    model = S.DeviceModel(dev, ds.n_features)
    assert S.sync_epoch(dds, model, S.Task.LR, 0.1, None, ds.n_examples)
    new_vals = np.ascontiguousarray(ds.values.astype(np.float32) * 2.0)
    dds.refresh_f32(new_vals)
    dev.synchronize()
    with pytest.raises(S.UnsupportedError):
        S.sync_epoch(dds, model, S.Task.LR, 0.1, None, ds.n_examples)
    plan = S.parse_plan("row-ch:kernel:0")
    plan.workers = 4
    S.hogwild_epoch(dds, model, S.Task.LR, 0.1, plan)
    fresh = S.DeviceDataset(dev, ds)
    assert S.sync_epoch(fresh, model, S.Task.LR, 0.1, None, ds.n_examples)


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
