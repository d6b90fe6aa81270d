"""e2e leg diagnostics: per-step time of (a) H2D only, (b) serial H2D+epoch+get,
(c) double-buffered H2D on a copy stream, for the bench workload."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_08800_b200 as S  # noqa: E402

K = 50


def main():
    torch.cuda.init()
    stream = torch.cuda.current_stream()
    dev = S.Device(0, stream=stream.cuda_stream)
    host = S.fixtures.sparse_classification(64700, 300, 11.65, 20250811)
    bufs = [S.DeviceDataset(dev, host), S.DeviceDataset(dev, host)]
    model = S.DeviceModel(dev, 300)
    plan = S.parse_plan("row-ch:kernel:0")
    plan.workers = dev.resident_workers(bufs[0])
    vals = torch.from_numpy(host.values.astype(np.float32)).pin_memory()
    labs = torch.from_numpy(host.labels.astype(np.float32)).pin_memory()
    idx = torch.from_numpy(host.indices.astype(np.int32)).pin_memory()
    rp = torch.from_numpy(host.row_offsets.astype(np.int32)).pin_memory()
    cs = torch.cuda.Stream()
    print("copy stream", cs, "query flags n/a")
    cdev = S.Device(0, stream=cs.cuda_stream)
    global K
    K = 50

    def timed(fn):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / K * 1e6

    def h2d_only():
        for _ in range(K):
            bufs[0].refresh_f32(vals, labs, idx, rp)
    print("h2d only (ctx stream) us", timed(h2d_only))

    def h2d_copy_stream():
        for _ in range(K):
            bufs[0].refresh_f32(vals, labs, idx, rp, device=cdev)
    print("h2d only (copy stream) us", timed(h2d_copy_stream))

    def epoch_only():
        for _ in range(K):
            S.hogwild_epoch(bufs[0], model, S.Task.SVM, 0.01, plan)
    print("epoch only us", timed(epoch_only))

    def epoch_get():
        for _ in range(K):
            S.hogwild_epoch(bufs[0], model, S.Task.SVM, 0.01, plan)
            model.get()
    print("epoch+get us", timed(epoch_get))

    def serial():
        for _ in range(K):
            bufs[0].refresh_f32(vals, labs, idx, rp)
            S.hogwild_epoch(bufs[0], model, S.Task.SVM, 0.01, plan)
            model.get()
    print("serial us", timed(serial))

    def double():
        ready = [torch.cuda.Event(), torch.cuda.Event()]
        free = [torch.cuda.Event(), torch.cuda.Event()]
        used = [False, False]
        bufs[0].refresh_f32(vals, labs, idx, rp, device=cdev)
        ready[0].record(cs)
        for k in range(K):
            b = k % 2
            if k + 1 < K:
                nb = 1 - b
                if used[nb]:
                    cs.wait_event(free[nb])
                bufs[nb].refresh_f32(vals, labs, idx, rp, device=cdev)
                ready[nb].record(cs)
            stream.wait_event(ready[b])
            S.hogwild_epoch(bufs[b], model, S.Task.SVM, 0.01, plan)
            free[b].record(stream)
            used[b] = True
            model.get()
    print("double-buffered us", timed(double))

    # The bench's sequence: flushed epochs, a profiling on/off cycle, then K=20 runs.
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(5):
        flush.zero_()
        S.hogwild_epoch(bufs[0], model, S.Task.SVM, 0.01, plan)
    dev.set_profiling(True)
    for _ in range(20):
        flush.zero_()
        S.hogwild_epoch(bufs[0], model, S.Task.SVM, 0.01, plan)
    dev.kernel_stats()
    dev.set_profiling(False)
    print("after profiling: double-buffered us", timed(double))
    print("after profiling: serial us", timed(serial))
    print("after profiling: epoch+get us", timed(epoch_get))


if __name__ == "__main__":
    main()
