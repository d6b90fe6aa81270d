"""Kernel-scope Hogwild: lanes per worker x worker count (epoch time and loss).

    python scripts/hogwild_lanes.py [w8a|rcv1|realsim ...]

CUDA-event epoch time (L2 flushed before each epoch: written, then read),
median over epochs 3..12, and the loss after 12 epochs.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_08800_b200 as S  # noqa: E402

CFG = {
    "w8a": (lambda: S.fixtures.sparse_classification(64700, 300, 11.65, 20250811), S.Task.SVM, 0.01),
    "rcv1": (lambda: S.fixtures.sparse_classification(677399, 47236, 73.16, 20250813), S.Task.LR, 0.01),
    "realsim": (lambda: S.fixtures.sparse_classification(72309, 20958, 51.3, 20250812), S.Task.SVM, 0.03),
}


def run(dev, dds, task, plan, alpha, epochs, flush, stream):
    model = S.DeviceModel(dev, dds.n_features)
    times = []
    for _ in range(epochs):
        flush.zero_()
        flush.view(torch.float32).sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        S.hogwild_epoch(dds, model, task, alpha, plan)
        b.record(stream)
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    return times, S.device_loss(dds, model, task)


def main():
    torch.cuda.init()
    stream = torch.cuda.current_stream()
    dev = S.Device(0, stream=stream.cuda_stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for name in sys.argv[1:] or ["w8a"]:
        make, task, alpha = CFG[name]
        host = make()
        dds = S.DeviceDataset(dev, host)
        for lanes in (4, 8, 16, 32):
            res = dev.resident_workers(dds, lanes)
            for frac in (1, 2):
                plan = S.parse_plan("row-ch:kernel:0")
                plan.workers = res // frac
                plan.lanes_per_worker = lanes
                times, loss = run(dev, dds, task, plan, alpha, 12, flush, stream)
                print(json.dumps({"data": name, "lanes": lanes, "workers": plan.workers,
                                  "epoch_us": 1e3 * float(np.median(times[2:])),
                                  "loss": round(loss, 1)}), flush=True)


if __name__ == "__main__":
    main()
