"""Kernel-scope Hogwild: additive model shards x feature dimension (contention test)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_08800_b200 as S  # noqa: E402
from hogwild_sweep import run  # noqa: E402


def main():
    torch.cuda.init()
    stream = torch.cuda.current_stream()
    dev = S.Device(0, stream=stream.cuda_stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for d in (300, 3000, 30000):
        host = S.fixtures.sparse_classification(64700, d, 11.65, 20250811)
        dds = S.DeviceDataset(dev, host)
        for shards in (1, 2, 4, 8, 16):
            os.environ["SGDB_HOGWILD_SHARDS"] = str(shards)
            plan = S.parse_plan("row-ch:kernel:0")
            plan.workers = dev.resident_workers(dds)
            times, losses = run(dev, dds, S.Task.SVM, plan, 0.01, 12, flush, stream)
            dev.set_profiling(True)
            model = S.DeviceModel(dev, d)
            for _ in range(4):
                flush.zero_()
                S.hogwild_epoch(dds, model, S.Task.SVM, 0.01, plan)
            st = dev.kernel_stats()
            dev.set_profiling(False)
            print(json.dumps({"d": d, "shards": shards, "epoch_us": 1e3 * float(np.median(times[2:])),
                              "kernel_us": {k: round(1e3 * v[1] / v[0], 1) for k, v in st.items()},
                              "loss": [round(x, 1) for x in losses[::4]] + [round(losses[-1], 1)]}),
                  flush=True)


if __name__ == "__main__":
    main()
