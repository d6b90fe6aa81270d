import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_08800_b200 as S
from hogwild_sweep import run
torch.cuda.init(); stream = torch.cuda.current_stream()
dev = S.Device(0, stream=stream.cuda_stream)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name, host, task in (("w8a", S.fixtures.sparse_classification(64700, 300, 11.65, 20250811), S.Task.SVM),
                         ("realsim", S.fixtures.sparse_classification(72309, 20958, 51.3, 20250812), S.Task.SVM),
                         ("rcv1", S.fixtures.sparse_classification(677399, 47236, 73.16, 20250813), S.Task.LR)):
    dds = S.DeviceDataset(dev, host)
    for staged in (0, 1):
        os.environ["SGDB_HOGWILD_STAGED"] = str(staged)
        for lanes in (8, 16, 32):
            res = dev.resident_workers(dds, lanes)
            for frac in (1, 2):
                plan = S.parse_plan("row-ch:kernel:0"); plan.workers = res // frac; plan.lanes_per_worker = lanes
                times, losses = run(dev, dds, task, plan, 0.01, 10, flush, stream)
                print(json.dumps({"data": name, "staged": staged, "lanes": lanes, "workers": plan.workers,
                                  "epoch_us": 1e3 * float(np.median(times[2:])), "loss": round(losses[-1], 1)}), flush=True)
