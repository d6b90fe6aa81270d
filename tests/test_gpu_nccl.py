"""The engine's own NCCL communicator (sgdb_ctx_init_nccl), on one B200.

NCCL does not allow two ranks of one communicator on the same GPU, so the
binding is checked with a 1-rank communicator: every exchange step (gradient
SUM all-reduce per mini-batch step, inside the CUDA-graph-replayed epoch;
the full-batch gradient; the loss; rank averaging of Hogwild replicas) runs
through ncclAllReduce on the context stream, and must leave results equal to
the collective-free path (a 1-rank SUM is the identity; mini-batch epochs of
dense data take the per-step kernels instead of the persistent epoch kernel,
so those agree to fp32 summation order) and the oracle. The multi-rank
semantics are covered by tests/test_gpu_multirank.py (two ranks on one GPU
through the host hook) and tests/test_distributed.py (gloo).
"""
import numpy as np
import pytest

from conftest import rel, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_dev(sgdb):
    import torch
    S = sgdb
    dev = S.Device(0, stream=torch.cuda.current_stream().cuda_stream)
    dev.init_nccl(1, 0, S.Device.nccl_unique_id())
    assert dev.world() == (0, 1)
    return dev


@pytest.mark.parametrize("kind", ["dense", "sparse"])
@pytest.mark.parametrize("batch", ["N", 256])
def test_sync_epochs_through_nccl_equal_plain(sgdb, dev, nccl_dev, orc, kind, batch):
    S = sgdb
    ds = (S.fixtures.dense_classification(3000, 54, 5) if kind == "dense"
          else S.fixtures.sparse_classification(3000, 800, 20.0, 5)).rounded_f32()
    b = ds.n_examples if batch == "N" else batch
    out = []
    for d in (dev, nccl_dev):
        dds = S.DeviceDataset(d, ds)
        m = S.DeviceModel(d, ds.n_features)
        sched = S.Schedule(3, ds.n_examples)
        for e in range(5):  # >= 4 steps per epoch: the graph-replayed path
            assert S.sync_epoch(dds, m, S.Task.LR, 1e-3, sched.next() if b < ds.n_examples else None, b)
        out.append((m.get(), S.device_loss(dds, m, S.Task.LR)))
    same_kernels = not (kind == "dense" and batch != "N")
    tol = 1e-12 if same_kernels else 1e-6
    assert rel_l2(out[1][0], out[0][0]) <= tol
    assert rel(out[1][1], out[0][1]) <= tol
    om, ol, _ = orc.sync_train(ds, 0, 1e-3, b, 5, 3)
    assert rel_l2(out[1][0], om[-1]) <= 1e-5
    assert rel(out[1][1], ol[-1]) <= 1e-6


def test_hogwild_rank_average_through_nccl(sgdb, nccl_dev, orc):
    S = sgdb
    from paper_1802_08800_b200 import distributed as SD
    ds = S.fixtures.sparse_classification(500, 60, 6.0, 9).rounded_f32()
    dds = S.DeviceDataset(nccl_dev, ds)
    m = S.DeviceModel(nccl_dev, ds.n_features)
    plan = S.parse_plan("row-ch:kernel:0")
    plan.workers = 1
    for _ in range(2):
        SD.hogwild_epoch_ranks(nccl_dev, dds, m, S.Task.SVM, 0.01, plan, 1, segments=3)
    om, _, _ = orc.hogwild_serial(ds, 1, 0.01, 2, 0, 0, 0, 1)
    assert rel_l2(m.get(), om[-1]) <= 1e-4
    # world = 1 with a communicator: the average is a SUM over one rank, x 1.
    S._lib.check(S._lib.load().sgdb_model_average_ranks(nccl_dev.handle, m.handle, 1))
