"""Hogwild epochs on every BASELINE shape with the paper's plans.

One GPU, L2 flushed before each epoch (outside the event window), epochs
enqueued back to back. Reports epoch time, examples/s, the algorithmic sweep
rate (one read of the stored matrix) and its fraction of the
measured HBM copy bandwidth, and the loss after the timed epochs.

    python scripts/async_sweep.py [w8a rcv1 news20 realsim covtype]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_08800_b200 as S  # noqa: E402

CFG = {
    # name: (generator, task, alpha, plans)
    "w8a": (lambda: S.fixtures.sparse_classification(64700, 300, 11.65, 20250811), S.Task.SVM, 1e-2,
            ["row-ch:kernel:0", "row-ch:kernel:10", "row-rr:kernel:0"]),
    "rcv1": (lambda: S.fixtures.sparse_classification(677399, 47236, 73.16, 20250813), S.Task.LR, 1e-2,
             ["row-ch:kernel:0", "row-ch:block:0"]),
    "news20": (lambda: S.fixtures.sparse_classification(19996, 1355191, 455.0, 20250814), S.Task.SVM, 1e-4,
               ["row-rr:kernel:10", "row-ch:kernel:0"]),
    "realsim": (lambda: S.fixtures.sparse_classification(72309, 20958, 51.3, 20250812), S.Task.SVM, 1e-3,
                ["row-rr:kernel:10", "row-ch:kernel:0"]),
    "covtype": (lambda: S.fixtures.dense_classification(581012, 54, 20250810), S.Task.LR, 1e-4,
                ["row-ch:kernel:0", "row-rr:kernel:0", "row-ch:block:0"]),
}


def peak():
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                               "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6544.3


def main():
    torch.cuda.init()
    stream = torch.cuda.current_stream()
    dev = S.Device(0, stream=stream.cuda_stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    pk = peak()
    for name in sys.argv[1:] or list(CFG):
        make, task, alpha, plans = CFG[name]
        host = make()
        dds = S.DeviceDataset(dev, host)
        sweep = dds.sweep_bytes()
        for pt in plans:
            plan = S.parse_plan(pt)
            plan.workers = dev.resident_workers(dds)
            model = S.DeviceModel(dev, host.n_features)
            for _ in range(2):
                S.hogwild_epoch(dds, model, task, alpha, plan)
            evs = []
            for _ in range(10):
                flush.zero_(); flush.view(torch.float32).sum()  # clean L2: written, then read
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                S.hogwild_epoch(dds, model, task, alpha, plan)
                b.record(stream)
                evs.append((a, b))
            torch.cuda.synchronize()
            ms = float(np.median([x.elapsed_time(y) for x, y in evs]))
            dev.set_profiling(True)
            flush.zero_(); flush.view(torch.float32).sum()  # clean L2: written, then read
            S.hogwild_epoch(dds, model, task, alpha, plan)
            stats = dev.kernel_stats()
            dev.set_profiling(False)
            print(json.dumps({
                "data": name, "plan": pt, "workers": plan.workers, "epoch_us": round(ms * 1e3, 2),
                "ex_per_s": host.n_examples / (ms / 1e3), "alg_GBps": sweep / (ms / 1e3) / 1e9,
                "frac": sweep / (ms / 1e3) / 1e9 / pk,
                "kernels_us": {k: round(v[1] * 1e3, 2) for k, v in stats.items()},
                "loss_after_13": S.device_loss(dds, model, task)}), flush=True)
        del dds


if __name__ == "__main__":
    main()
