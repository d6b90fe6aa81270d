"""Multi-rank end to end on ONE GPU: two processes share cuda:0 and use the
gloo backend (which all-reduces CUDA tensors) as the engine's allreduce hook,
so the real device paths of SURVEY §8(e) run with world_size 2:

* sync SGD over contiguous row shards: each rank computes the partial
  gradient of its members of the global sorted batch, the hook SUM-reduces g,
  every rank applies the same update -> equals the single-process oracle run;
* Hogwild replicas averaged `segments` times per epoch
  (distributed.hogwild_epoch_ranks): with one worker per rank every segment is
  a serial pass over a contiguous row range, so the oracle reproduces the whole
  schedule (segment passes from the averaged model, then merge_models).

On a multi-GPU box the same code runs with NCCL, one GPU per rank.
Tolerance: fp32 device arithmetic, model rel-L2 <= 1e-5.
"""
import os
import socket

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu

WORLD = 2
SEGMENTS = 3
EPOCHS = 2
ALPHA_H = 0.05
N_SYNC, D_SYNC, B_SYNC, ALPHA_S, SEED_S = 1203, 60, 128, 0.1, 31


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _partition(S, rank):
    return S.fixtures.sparse_classification(500 + 37 * rank, 50, 5.0, 100 + rank).rounded_f32()


def _sync_data(S):
    return S.fixtures.sparse_classification(N_SYNC, D_SYNC, 6.0, 9).rounded_f32()


def _rank_main(rank, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    import paper_1802_08800_b200 as S
    from paper_1802_08800_b200 import distributed as SD

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    dev = S.Device(0, stream=torch.cuda.current_stream().cuda_stream)
    SD.attach(dev)
    out = {}

    # Sync SGD on row shards, global schedule on every rank.
    full = _sync_data(S)
    base, cnt = SD.shard_rows(full.n_examples, rank, WORLD)
    lo, hi = int(full.row_offsets[base]), int(full.row_offsets[base + cnt])
    shard = S.Dataset(cnt, full.n_features, S.Layout.Csr, full.labels[base:base + cnt],
                      full.values[lo:hi], full.indices[lo:hi],
                      full.row_offsets[base:base + cnt + 1] - full.row_offsets[base])
    dds = S.DeviceDataset(dev, shard, row_base=base, n_global=full.n_examples)
    model = S.DeviceModel(dev, full.n_features)
    sched = S.Schedule(SEED_S, full.n_examples, True)
    for e in range(1, EPOCHS + 1):
        assert S.sync_epoch(dds, model, S.Task.LR, ALPHA_S, sched.next(), B_SYNC)
    out["sync"] = model.get()
    out["sync_loss"] = S.device_loss(dds, model, S.Task.LR)

    # Hogwild replicas, averaged SEGMENTS times per epoch.
    part = _partition(S, rank)
    hds = S.DeviceDataset(dev, part)
    hm = S.DeviceModel(dev, part.n_features)
    plan = S.parse_plan("row-ch:kernel:0")
    plan.workers = 1
    evals = 0
    for _ in range(EPOCHS):
        evals += SD.hogwild_epoch_ranks(dev, hds, hm, S.Task.LR, ALPHA_H, plan, WORLD, SEGMENTS)
    out["hog"] = hm.get()
    out["evals"] = evals
    results[rank] = out
    dist.barrier()
    dist.destroy_process_group()


@pytest.fixture(scope="module")
def ranks():
    import torch.multiprocessing as mp
    port = _free_port()
    with mp.get_context("spawn").Manager() as mgr:
        results = mgr.dict()
        mp.spawn(_rank_main, args=(port, results), nprocs=WORLD, join=True)
        return dict(results)


def test_sharded_sync_matches_single_process(sgdb, orc, ranks):
    S = sgdb
    full = _sync_data(S)
    om, ol, _ = orc.sync_train(full, 0, ALPHA_S, B_SYNC, EPOCHS, SEED_S)
    for r in range(WORLD):
        assert rel_l2(ranks[r]["sync"], om[-1]) <= 1e-5
        assert abs(ranks[r]["sync_loss"] - ol[-1]) <= 1e-6 * abs(ol[-1])
    assert np.array_equal(ranks[0]["sync"], ranks[1]["sync"])  # replicated update


def _rows(ds, lo, hi):
    import oracle
    a, b = int(ds.row_offsets[lo]), int(ds.row_offsets[hi])
    return oracle.HostData(hi - lo, ds.n_features, 2, ds.labels[lo:hi], ds.values[a:b],
                           ds.indices[a:b], ds.row_offsets[lo:hi + 1] - ds.row_offsets[lo])


def test_hogwild_segment_averaging_matches_oracle(sgdb, orc, ranks):
    S = sgdb
    parts = [_partition(S, r) for r in range(WORLD)]
    avg = np.zeros(parts[0].n_features)
    for _ in range(EPOCHS):
        for s in range(SEGMENTS):
            own = []
            for ds in parts:
                t = ds.n_examples
                lo, hi = t * s // SEGMENTS, t * (s + 1) // SEGMENTS
                m, _, _ = orc.hogwild_serial(_rows(ds, lo, hi), 0, ALPHA_H, 1, 0, 0, 0, 1,
                                             init=avg)
                own.append(m[-1])
            avg = orc.merge_models(np.stack(own))
    for r in range(WORLD):
        assert rel_l2(ranks[r]["hog"], avg) <= 1e-5
        assert ranks[r]["evals"] == EPOCHS * parts[r].n_examples
    assert np.array_equal(ranks[0]["hog"], ranks[1]["hog"])  # every rank holds the mean


def test_segments_compose_to_one_epoch(sgdb, dev):
    """Single process: segments 0..S-1 back to back == one epoch when the
    schedule is sequential (1 worker), and the eval counts add up for many
    workers with k-replication."""
    S = sgdb
    ds = _partition(S, 0)
    plan = S.parse_plan("row-rr:kernel:2")
    plan.workers = 1
    a, b = S.DeviceModel(dev, ds.n_features), S.DeviceModel(dev, ds.n_features)
    dds = S.DeviceDataset(dev, ds)
    S.hogwild_epoch(dds, a, S.Task.SVM, 0.02, plan)
    for s in range(4):
        S.hogwild_epoch(dds, b, S.Task.SVM, 0.02, plan, s, 4)
    assert np.array_equal(a.get(), b.get())
    plan.workers = 37
    full = S.hogwild_epoch(dds, a, S.Task.SVM, 0.02, plan)
    parts = sum(S.hogwild_epoch(dds, b, S.Task.SVM, 0.02, plan, s, 5) for s in range(5))
    assert full == parts == ds.n_examples + 37 * 2
    with pytest.raises(ValueError, match="segment out of range"):
        S.hogwild_epoch(dds, b, S.Task.SVM, 0.02, plan, 5, 5)
