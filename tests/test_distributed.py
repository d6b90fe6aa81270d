"""Multi-process (world_size 2, gloo, CPU) coverage of the multi-GPU host logic:
row sharding, the SUM collective the engine's allreduce hook performs, the
row-sharded synchronous gradient (sum of per-shard gradients == the full
batch gradient) and per-rank replica averaging (the
numa_dual_train merge generalised to G ranks, async_engine.cpp:478-501).
The per-rank compute here is the CPU oracle; on GPUs the same collective runs
over NCCL inside sgdb_sync_epoch / sgdb_model_average_ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1802_08800_b200 import distributed as SD


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    O = oracle.oracle()
    out = {}
    # 1. row sharding covers [0, n) exactly once
    n = 1003
    base, cnt = SD.shard_rows(n, rank, world)
    out["shard"] = (base, cnt)
    # 2. sync: per-shard gradient of the global batch, summed across ranks
    ds = O.fixture_sparse(n, 80, 7.0, 5)
    w = np.random.default_rng(2).normal(0, 0.3, 80)
    batch = np.sort(np.random.default_rng(3).choice(n, 400, replace=False)).astype(np.uint32)
    mine = batch[(batch >= base) & (batch < base + cnt)]
    g = O.batch_gradient(ds, 0, mine, w) if mine.size else np.zeros(80)
    t = torch.from_numpy(g.copy())
    SD.sum_in_place(t)
    out["grad"] = t.numpy()
    # 3. Hogwild replicas: rank trains on its own partition, then averages
    part = O.fixture_sparse(500, 40, 5.0, 100 + rank)
    models, _, _ = O.hogwild_serial(part, 1, 0.05, 2, 0, 0, 0, 1)
    mt = torch.from_numpy(models[-1].copy())
    SD.sum_in_place(mt)
    out["avg"] = (mt / world).numpy()
    out["own"] = models[-1]
    results[rank] = out
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        results = mgr.dict()
        mp.spawn(_worker, args=(world, port, results), nprocs=world, join=True)
        res = dict(results)
    import oracle
    O = oracle.oracle()
    shards = [res[r]["shard"] for r in range(world)]
    covered = sorted(i for b, c in shards for i in range(b, b + c))
    assert covered == list(range(1003))
    ds = O.fixture_sparse(1003, 80, 7.0, 5)
    w = np.random.default_rng(2).normal(0, 0.3, 80)
    batch = np.sort(np.random.default_rng(3).choice(1003, 400, replace=False)).astype(np.uint32)
    full = O.batch_gradient(ds, 0, batch, w)
    for r in range(world):
        np.testing.assert_allclose(res[r]["grad"], full, rtol=1e-12, atol=1e-14)
    expected = O.merge_models(np.stack([res[r]["own"] for r in range(world)]))
    for r in range(world):
        np.testing.assert_allclose(res[r]["avg"], expected, rtol=1e-15, atol=0)


@pytest.mark.parametrize("n,world", [(10, 3), (64700, 8), (3, 5), (581012, 8)])
def test_shard_rows_partition(n, world):
    spans = [SD.shard_rows(n, r, world) for r in range(world)]
    assert sum(c for _, c in spans) == n
    pos = 0
    for b, c in spans:
        if c:
            assert b == pos
            pos += c
