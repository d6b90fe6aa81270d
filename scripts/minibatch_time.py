"""Mini-batch sync epoch timing on the BASELINE shapes (B given), L2 flushed."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_08800_b200 as S  # noqa: E402

SHAPES = {
    "covtype": (lambda: S.fixtures.dense_classification(581012, 54, 20250810), S.Task.LR),
    "dense1000": (lambda: S.fixtures.dense_classification(200000, 1000, 7), S.Task.LR),
    "dense256": (lambda: S.fixtures.dense_classification(300000, 256, 9), S.Task.SVM),
    "rcv1": (lambda: S.fixtures.sparse_classification(677399, 47236, 73.16, 20250813), S.Task.LR),
    "realsim": (lambda: S.fixtures.sparse_classification(72309, 20958, 51.3, 20250812), S.Task.SVM),
    "w8a": (lambda: S.fixtures.sparse_classification(64700, 300, 11.65, 20250811), S.Task.SVM),
    "news20": (lambda: S.fixtures.sparse_classification(19996, 1355191, 455.0, 20250814), S.Task.SVM),
}


def main():
    names = sys.argv[1].split(",")
    bs = [int(b) for b in (sys.argv[2] if len(sys.argv) > 2 else "4096").split(",")]
    torch.cuda.init()
    stream = torch.cuda.current_stream()
    dev = S.Device(0, stream=stream.cuda_stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for name in names:
        make, task = SHAPES[name]
        host = make()
        dds = S.DeviceDataset(dev, host)
        order = np.random.default_rng(0).permutation(host.n_examples).astype(np.uint32)
        for B in bs:
            model = S.DeviceModel(dev, host.n_features)
            times = []
            for i in range(8):
                flush.zero_(); flush.view(torch.float32).sum()  # clean L2: written, then read
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                S.sync_epoch(dds, model, task, 1e-7, order, B)
                b.record(stream)
                torch.cuda.synchronize()
                times.append(a.elapsed_time(b))
            steps = (host.n_examples + B - 1) // B
            ms = float(np.median(times[2:]))
            print(json.dumps({"data": name, "B": B, "steps": steps, "epoch_ms": ms,
                              "us_per_step": ms * 1e3 / steps,
                              "loss": S.device_loss(dds, model, task)}), flush=True)


if __name__ == "__main__":
    main()
