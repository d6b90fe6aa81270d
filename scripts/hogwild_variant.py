import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_08800_b200 as S
from hogwild_sweep import run
torch.cuda.init(); stream = torch.cuda.current_stream()
dev = S.Device(0, stream=stream.cuda_stream)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
noflush = torch.empty(1, dtype=torch.uint8, device="cuda")
host = S.fixtures.sparse_classification(64700, 300, 11.65, 20250811)
dds = S.DeviceDataset(dev, host)
for variant in (0, 1, 2):
    for fl in (flush, noflush):
        for lanes, workers in ((32, 4736), (8, 18944), (32, 64700)):
            os.environ["SGDB_HOGWILD_VARIANT"] = str(variant)
            plan = S.parse_plan("row-ch:kernel:0"); plan.workers = workers; plan.lanes_per_worker = lanes
            times, losses = run(dev, dds, S.Task.SVM, plan, 0.01, 12, fl, stream)
            print(json.dumps({"variant": variant, "flush": fl.numel() > 1, "lanes": lanes, "workers": workers,
                              "epoch_us": 1e3 * float(np.median(times[2:])), "loss": round(losses[-1], 1)}), flush=True)
