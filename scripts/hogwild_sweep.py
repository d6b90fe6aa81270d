"""Hogwild kernel-variant sweep (device timing + statistical progress).

Runs on one GPU: for each dataset / plan / model-access mode / worker count,
times epochs with CUDA events (L2 flushed before each) and reports the loss
after a fixed number of epochs, so speed and statistical efficiency are read
side by side. Output: one JSON line per configuration.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_08800_b200 as S  # noqa: E402


def run(dev, dds, task, plan, alpha, epochs, flush, stream):
    model = S.DeviceModel(dev, dds.n_features)
    times, losses = [], []
    for _ in range(epochs):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        S.hogwild_epoch(dds, model, task, alpha, plan)
        b.record(stream)
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
        losses.append(S.device_loss(dds, model, task))
    return times, losses


def main():
    torch.cuda.init()
    stream = torch.cuda.current_stream()
    dev = S.Device(0, stream=stream.cuda_stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    which = sys.argv[1] if len(sys.argv) > 1 else "w8a"
    if which == "w8a":
        host = S.fixtures.sparse_classification(64700, 300, 11.65, 20250811)
        task, alpha = S.Task.SVM, 0.01
    elif which == "covtype":
        host = S.fixtures.dense_classification(581012, 54, 20250810)
        task, alpha = S.Task.LR, 1e-4
    elif which == "rcv1":
        host = S.fixtures.sparse_classification(677399, 47236, 73.16, 20250813)
        task, alpha = S.Task.LR, 0.01
    elif which == "realsim":
        host = S.fixtures.sparse_classification(72309, 20958, 51.3, 20250812)
        task, alpha = S.Task.SVM, 0.01
    else:
        host = S.fixtures.sparse_classification(19996, 1355191, 455.0, 20250814)
        task, alpha = S.Task.SVM, 0.01
    dds = S.DeviceDataset(dev, host)
    resident = dev.resident_workers(dds)
    configs = []
    spreads = [int(x) for x in os.environ.get("SWEEP_SPREAD", "0,1").split(",")]
    for plan_text in ("row-ch:kernel:0",):
        for spread in spreads:
            for mode, refresh in ((1, 1), (2, 1), (2, 4), (2, 16)):
                for workers in (resident // 8, resident):
                    configs.append((plan_text, mode, refresh, workers, 0, spread))
    for workers, gs in ((resident, 32), (resident, 256)):
        configs.append(("row-ch:block:0", 0, 1, workers, gs, 0))
    for plan_text, mode, refresh, workers, gs, spread in configs:
        os.environ["SGDB_HOGWILD_MODE"] = str(mode)
        os.environ["SGDB_HOGWILD_REFRESH"] = str(refresh)
        os.environ["SGDB_HOGWILD_SPREAD"] = str(spread)
        plan = S.parse_plan(plan_text)
        plan.workers = workers
        if gs:
            plan.group_size = gs
        times, losses = run(dev, dds, task, plan, alpha, 12, flush, stream)
        print(json.dumps({"data": which, "plan": plan_text, "mode": mode, "refresh": refresh,
                          "spread": spread,
                          "workers": workers, "group_size": gs,
                          "epoch_ms_median": float(np.median(times[2:])),
                          "ex_per_s": host.n_examples / (float(np.median(times[2:])) / 1e3),
                          "loss": [round(x, 2) for x in losses[::3]] + [round(losses[-1], 2)]}),
              flush=True)


if __name__ == "__main__":
    main()
