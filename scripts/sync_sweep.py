"""Synchronous-engine throughput sweep on one GPU (device timing, L2 flushed).

For each config: one epoch = sgdb_sync_epoch; reports epoch time, examples/s,
algorithmic GB/s (one sweep of the stored matrix) and the
per-kernel CUDA-event breakdown from the library's profiler.
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_08800_b200 as S  # noqa: E402

CFG = {
    "covtype": lambda: (S.fixtures.dense_classification(581012, 54, 20250810), S.Task.LR, 1e-6),
    "w8a": lambda: (S.fixtures.sparse_classification(64700, 300, 11.65, 20250811), S.Task.SVM, 1e-5),
    "realsim": lambda: (S.fixtures.sparse_classification(72309, 20958, 51.3, 20250812), S.Task.SVM, 1e-5),
    "rcv1": lambda: (S.fixtures.sparse_classification(677399, 47236, 73.16, 20250813), S.Task.LR, 1e-6),
    "news20": lambda: (S.fixtures.sparse_classification(19996, 1355191, 455.0, 20250814), S.Task.SVM, 1e-5),
    "dense1000": lambda: (S.fixtures.dense_classification(200000, 1000, 7), S.Task.LR, 1e-7),
    "dense256": lambda: (S.fixtures.dense_classification(300000, 256, 9), S.Task.SVM, 1e-6),
}


def main():
    torch.cuda.init()
    stream = torch.cuda.current_stream()
    dev = S.Device(0, stream=stream.cuda_stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    names = sys.argv[1:] or list(CFG)
    peak = 6544.3
    for name in names:
        t0 = time.time()
        host, task, alpha = CFG[name]()
        gen_s = time.time() - t0
        dds = S.DeviceDataset(dev, host)
        sweep = dds.sweep_bytes()
        n = host.n_examples
        for b in (n, 4096):
            model = S.DeviceModel(dev, host.n_features)
            sched = S.Schedule(1, n)
            order = sched.next()
            evs = []
            for i in range(8):
                flush.zero_(); flush.view(torch.float32).sum()  # clean L2: written, then read
                ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ev0.record(stream)
                S.sync_epoch(dds, model, task, alpha, order if b < n else None, b, check_finite=False)
                ev1.record(stream)
                evs.append((ev0, ev1))
            torch.cuda.synchronize()
            times = [e0.elapsed_time(e1) for e0, e1 in evs]
            dev.set_profiling(True)
            for i in range(3):
                flush.zero_(); flush.view(torch.float32).sum()  # clean L2: written, then read
                S.sync_epoch(dds, model, task, alpha, order if b < n else None, b)
            stats = dev.kernel_stats()
            dev.set_profiling(False)
            ms = float(np.median(times[3:]))
            print(json.dumps({
                "data": name, "B": b, "epoch_ms": ms, "ex_per_s": n / (ms / 1e3),
                "alg_GBps": sweep / (ms / 1e3) / 1e9, "frac": sweep / (ms / 1e3) / 1e9 / peak,
                "kernels": {k: [v[0] // 3, round(v[1] / 3, 4)] for k, v in stats.items()},
                "loss": S.device_loss(dds, model, task), "gen_s": round(gen_s, 1)}), flush=True)


if __name__ == "__main__":
    main()
