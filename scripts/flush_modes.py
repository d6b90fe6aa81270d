"""How the between-step L2 treatment changes the measured full-batch epoch.

    python scripts/flush_modes.py [rcv1|realsim|news20|w8a ...]

Modes: "memset" (write 256 MiB: L2 left full of DIRTY lines the next step's
first kernel must write back), "read" (read 256 MiB after the memset: L2 left
full of clean lines), "none" (no flush; valid only when a step streams more
than L2 holds). CUDA-event epoch time, median of 15 after 3 warm-up epochs.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_08800_b200 as S  # noqa: E402

CFG = {
    "w8a": lambda: (S.fixtures.sparse_classification(64700, 300, 11.65, 20250811), S.Task.SVM, 1e-5),
    "realsim": lambda: (S.fixtures.sparse_classification(72309, 20958, 51.3, 20250812), S.Task.SVM, 1e-5),
    "rcv1": lambda: (S.fixtures.sparse_classification(677399, 47236, 73.16, 20250813), S.Task.LR, 1e-2),
    "news20": lambda: (S.fixtures.sparse_classification(19996, 1355191, 455.0, 20250814), S.Task.SVM, 1e-5),
}


def main():
    torch.cuda.init()
    stream = torch.cuda.current_stream()
    dev = S.Device(0, stream=stream.cuda_stream)
    buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    sink = torch.empty(1, dtype=torch.float32, device="cuda")

    def memset():
        buf.zero_()

    def read():
        buf.zero_()
        sink.copy_(buf.view(torch.float32).sum())

    modes = {"memset": memset, "read": read, "none": lambda: None}
    for name in sys.argv[1:] or ["rcv1", "realsim"]:
        host, task, alpha = CFG[name]()
        dds = S.DeviceDataset(dev, host.rounded_f32())
        n = host.n_examples
        for mode, fl in modes.items():
            model = S.DeviceModel(dev, host.n_features)
            evs = []
            for i in range(18):
                fl()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                S.sync_epoch(dds, model, task, alpha, None, n, check_finite=False)
                e1.record(stream)
                evs.append((e0, e1))
            torch.cuda.synchronize()
            t = [a.elapsed_time(b) * 1e3 for a, b in evs[3:]]
            print(json.dumps({"data": name, "mode": mode, "epoch_us": round(float(np.median(t)), 1),
                              "min_us": round(min(t), 1)}), flush=True)


if __name__ == "__main__":
    main()
