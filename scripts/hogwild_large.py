"""Kernel-scope Hogwild on the large sparse shapes (rcv1, news20, real-sim):
model layout (slice-spread vs flat), lanes per worker and update mode, with
device-timed epochs (L2 flushed) and the loss after the timed epochs.

    python scripts/hogwild_large.py [rcv1 news20 realsim]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_08800_b200 as S  # noqa: E402

CFG = {
    "rcv1": (lambda: S.fixtures.sparse_classification(677399, 47236, 73.16, 20250813), S.Task.LR, 1e-2, "row-ch:kernel:0"),
    "news20": (lambda: S.fixtures.sparse_classification(19996, 1355191, 455.0, 20250814), S.Task.SVM, 1e-4, "row-ch:kernel:0"),
    "realsim": (lambda: S.fixtures.sparse_classification(72309, 20958, 51.3, 20250812), S.Task.SVM, 1e-3, "row-ch:kernel:0"),
    "w8a": (lambda: S.fixtures.sparse_classification(64700, 300, 11.65, 20250811), S.Task.SVM, 1e-2, "row-ch:kernel:0"),
}


def main():
    torch.cuda.init()
    stream = torch.cuda.current_stream()
    dev = S.Device(0, stream=stream.cuda_stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for name in sys.argv[1:] or ["rcv1", "news20", "realsim"]:
        make, task, alpha, pt = CFG[name]
        host = make()
        dds = S.DeviceDataset(dev, host)
        for spread in (1, 0):
            for lanes in (32, 16, 8):
                for mode in (2, 0):
                    os.environ["SGDB_HOGWILD_SPREAD"] = str(spread)
                    os.environ["SGDB_HOGWILD_MODE"] = str(mode)
                    plan = S.parse_plan(pt)
                    plan.lanes_per_worker = lanes
                    plan.workers = dev.resident_workers(dds, lanes)
                    model = S.DeviceModel(dev, host.n_features)
                    S.hogwild_epoch(dds, model, task, alpha, plan)
                    evs = []
                    for _ in range(6):
                        flush.zero_()
                        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        a.record(stream)
                        S.hogwild_epoch(dds, model, task, alpha, plan)
                        b.record(stream)
                        evs.append((a, b))
                    torch.cuda.synchronize()
                    ms = float(np.median([x.elapsed_time(y) for x, y in evs]))
                    print(json.dumps({"data": name, "spread": spread, "lanes": lanes, "mode": mode,
                                      "workers": plan.workers, "epoch_us": round(ms * 1e3, 1),
                                      "loss_after_7": round(S.device_loss(dds, model, task), 1)}),
                          flush=True)
        del dds


if __name__ == "__main__":
    main()
