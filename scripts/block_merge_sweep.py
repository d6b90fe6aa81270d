"""rcv1-shaped LR Hogwild, block scope: replicas merged k times per epoch.

The reference's block replication (async_engine.cpp:293-331) prepares the
replicas at the start of an epoch and merges them at its end. Here an epoch
runs as k segments (sgdb_hogwild_segment): every segment starts from the merged
model and merges at its end, i.e. the replicas are averaged k times per epoch.
Per (R, k, alpha): mean segmented-epoch time (L2 flushed before each epoch)
and the loss after each of 15 epochs from w = 0, against L* (the bench's GPU
batch-GD probe value). Kernel scope beside it.
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_08800_b200 as S  # noqa: E402

L_STAR = 270641.50501465274
EPOCHS = 15


def run(dev, dds, host, plan, alpha, k, flush, stream):
    model = S.DeviceModel(dev, host.n_features)
    losses, times = [], []
    for _ in range(EPOCHS):
        flush.zero_(); flush.view(torch.float32).sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for seg in range(k):
            S.hogwild_epoch(dds, model, S.Task.LR, alpha, plan, seg, k)
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
        losses.append(S.device_loss(dds, model, S.Task.LR))
    hit = next((i + 1 for i, l in enumerate(losses) if l <= 1.01 * L_STAR), None)
    return {"epoch_ms": float(np.mean(times[1:])), "losses": [round(x) for x in losses],
            "epochs_to_1pct": hit,
            "time_to_1pct_ms": float(np.mean(times[1:])) * hit if hit else None}


def main():
    torch.cuda.init()
    stream = torch.cuda.current_stream()
    dev = S.Device(0, stream=stream.cuda_stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    host = S.fixtures.sparse_classification(677399, 47236, 73.16, 20250813)
    dds = S.DeviceDataset(dev, host)
    workers = dev.resident_workers(dds)
    cases = [("kernel", None, 1, 0.01)]
    for R in (148, 16):
        for k in (1, 4, 16, 64):
            for alpha in ((0.1, 0.03) if R == 148 else (0.08,)):
                cases.append(("block", R, k, alpha))
    only = sys.argv[1:]
    for scope, R, k, alpha in cases:
        if only and f"{R}:{k}" not in only and scope != "kernel":
            continue
        plan = S.parse_plan(f"row-ch:{scope}:0")
        plan.workers = workers
        if R:
            plan.group_size = workers // R
        t0 = time.time()
        r = run(dev, dds, host, plan, alpha, k, flush, stream)
        r.update({"scope": scope, "R": R, "merges_per_epoch": k, "alpha": alpha, "wall_s": round(time.time() - t0, 1)})
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
