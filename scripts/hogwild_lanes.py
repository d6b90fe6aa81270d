"""w8a kernel-scope Hogwild: lanes per worker x worker count (time and loss)."""
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
    host = S.fixtures.sparse_classification(64700, 300, 11.65, 20250811)
    dds = S.DeviceDataset(dev, host)
    for plan_text in ("row-ch:kernel:0", "row-rr:kernel:0"):
        for lanes in (4, 8, 16, 32):
            res = dev.resident_workers(dds, lanes)
            for frac in (1, 2, 4):
                plan = S.parse_plan(plan_text)
                plan.workers = res // frac
                plan.lanes_per_worker = lanes
                times, losses = run(dev, dds, S.Task.SVM, plan, 0.01, 12, flush, stream)
                print(json.dumps({"plan": plan_text, "lanes": lanes, "workers": plan.workers,
                                  "epoch_us": 1e3 * float(np.median(times[2:])),
                                  "loss": round(losses[-1], 1)}), flush=True)


if __name__ == "__main__":
    main()
