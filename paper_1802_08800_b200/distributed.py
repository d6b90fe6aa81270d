"""Multi-GPU plumbing: one process per GPU, torch.distributed (NCCL) as the
collective provider behind the engine's allreduce hook (include/sgdb.h,
sgdb_allreduce_fn).

The reference has no multi-device path; its closest analogs are
the worker-count-invariant reduction of the sync path
(proj/include/sgdbench/linalg.hpp:14-18) and numa_dual_train's replica
averaging (proj/src/async_engine.cpp:462-520). Here:

* sync SGD: rows are sharded in contiguous chunks
  (``shard_rows``, the chunk rule of assign(), dataset.cpp:484-490); every
  rank walks the same global mini-batch schedule, computes the partial
  gradient of its members, the engine SUM-all-reduces g (fp64) and applies
  the identical update on every rank.
* Hogwild: each rank runs the Hogwild kernels on its replica (its row shard,
  or the full data for the numa_dual_train-style mode) and the replicas are
  averaged ``segments`` times per epoch (``hogwild_epoch_ranks``): every
  worker's assign() list is cut into ``segments`` equal position ranges and
  the ranks all-reduce the model after each ("every k batches").
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import _lib as L
from .api import Device, DeviceDataset, DeviceModel, ExecutionPlan, Task, hogwild_epoch


def shard_rows(n: int, rank: int, world: int) -> tuple[int, int]:
    """(row_base, n_local) of rank's contiguous chunk: ceil(n/world) rows each."""
    chunk = (n + world - 1) // world
    base = min(n, rank * chunk)
    return base, min(n, base + chunk) - base


class _CudaArray:
    """Zero-copy view of a device buffer for torch.as_tensor."""

    def __init__(self, ptr: int, count: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None,
                                         "stream": None}


def device_view(ptr: int, count: int, dtype: int) -> torch.Tensor:
    """torch tensor aliasing an engine buffer (dtype 0 = float32, 1 = float64)."""
    return torch.as_tensor(_CudaArray(ptr, count, "<f4" if dtype == 0 else "<f8"), device="cuda")


def sum_in_place(t: torch.Tensor, group=None) -> torch.Tensor:
    """The collective the engine asks for: SUM all-reduce, in place."""
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def attach(dev: Device, group=None) -> None:
    """Installs torch.distributed as the engine's allreduce hook on dev.

    The engine calls the hook on its own stream; torch's current stream must be
    that stream (create the Device with stream=torch.cuda.current_stream().cuda_stream).
    """
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        dev.set_allreduce(None)
        return

    def hook(ptr, count, dtype, stream):
        # The collective runs on the engine's stream, whatever torch's current
        # stream is, so it is ordered with the engine's kernels (handles 0 / 1 /
        # 2 are the legacy / per-thread default streams).
        s = (torch.cuda.default_stream() if stream in (0, 1, 2)
             else torch.cuda.ExternalStream(stream))
        with torch.cuda.stream(s):
            sum_in_place(device_view(ptr, count, dtype), group)

    dev.set_allreduce(hook)


def attach_nccl(dev: Device, group=None) -> None:
    """Gives the engine its own NCCL communicator over the ranks of the
    initialised process group: rank 0 creates the id (sgdb_nccl_get_unique_id),
    the process group broadcasts it, every rank calls sgdb_ctx_init_nccl. The
    engine then issues ncclAllReduce on its stream itself (no Python hop per
    step; multi-rank mini-batch epochs stay CUDA-graph-replayed)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [Device.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    dev.init_nccl(world, rank, obj[0])


def average_ranks(dev: Device, model: DeviceModel, world: int) -> None:
    """Replica averaging across ranks: SUM all-reduce of the fp64 model, / world."""
    L.check(L.load().sgdb_model_average_ranks(dev.handle, model.handle, world))


def hogwild_epoch_ranks(dev: Device, dds: DeviceDataset, model: DeviceModel, task: Task,
                        alpha: float, plan: ExecutionPlan, world: int, segments: int = 1) -> int:
    """One multi-GPU Hogwild epoch: ``segments`` segments of this rank's replica
    epoch (sgdb_hogwild_segment), each followed by the cross-rank average of
    the replicas. segments=1 is a per-epoch merge (numa_dual_train with
    merge_period 1, async_engine.cpp:478-501). Returns this rank's evaluations."""
    if segments < 1:
        raise ValueError("segments must be >= 1")
    evals = 0
    for s in range(segments):
        evals += hogwild_epoch(dds, model, task, alpha, plan, s, segments)
        average_ranks(dev, model, world)
    return evals
