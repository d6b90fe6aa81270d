"""Hogwild kernel A/B timing: median epoch time (CUDA events, L2 flushed before
every epoch) and the loss after the timed epochs, for lanes x workers on the
BASELINE shapes. One JSON line per configuration.

    python scripts/hogwild_ab.py [w8a,realsim,rcv1,covtype] [tag]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_08800_b200 as S  # noqa: E402

DATA = {
    "w8a": (lambda: S.fixtures.sparse_classification(64700, 300, 11.65, 20250811), S.Task.SVM, 0.01),
    "realsim": (lambda: S.fixtures.sparse_classification(72309, 20958, 51.3, 20250812), S.Task.SVM, 0.01),
    "rcv1": (lambda: S.fixtures.sparse_classification(677399, 47236, 73.16, 20250813), S.Task.LR, 0.01),
    "covtype": (lambda: S.fixtures.dense_classification(581012, 54, 20250810), S.Task.LR, 1e-4),
}


def main():
    which = (sys.argv[1] if len(sys.argv) > 1 else "w8a,realsim").split(",")
    tag = sys.argv[2] if len(sys.argv) > 2 else ""
    torch.cuda.init()
    stream = torch.cuda.current_stream()
    dev = S.Device(0, stream=stream.cuda_stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    occs = os.environ.get("SGDB_AB_OCC", "0").split(",")
    lanes_list = [int(x) for x in os.environ.get("SGDB_AB_LANES", "8,16,32").split(",")]
    for name in which:
        make, task, alpha = DATA[name]
        host = make()
        dds = S.DeviceDataset(dev, host)
        for occ, lanes in [(o, g) for o in occs for g in lanes_list]:
            os.environ["SGDB_HOGWILD_OCC"] = occ
            resident = dev.resident_workers(dds, lanes)
            for workers in (resident // 2, resident):
                plan = S.parse_plan("row-ch:kernel:0")
                plan.workers, plan.lanes_per_worker = workers, lanes
                model = S.DeviceModel(dev, host.n_features)
                times = []
                for _ in range(12):
                    flush.zero_()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    S.hogwild_epoch(dds, model, task, alpha, plan)
                    b.record(stream)
                    torch.cuda.synchronize()
                    times.append(a.elapsed_time(b) * 1e3)
                print(json.dumps({"tag": tag, "occ": occ, "data": name, "lanes": lanes,
                                  "workers": workers,
                                  "epoch_us": float(np.median(times[2:])),
                                  "loss12": round(S.device_loss(dds, model, task), 3)}), flush=True)


if __name__ == "__main__":
    main()
