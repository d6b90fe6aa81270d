import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1802_08800_b200 as S
torch.cuda.init(); stream = torch.cuda.current_stream()
dev = S.Device(0, stream=stream.cuda_stream)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
host = S.fixtures.sparse_classification(64700, 300, 11.65, 20250811); dds = S.DeviceDataset(dev, host)
for mode, workers in (("1", 4736), ("3", 4144), ("3", 2072)):
    os.environ["SGDB_HOGWILD_MODE"] = mode
    plan = S.parse_plan("row-ch:kernel:0"); plan.workers = workers
    model = S.DeviceModel(dev, host.n_features)
    evs = []; losses = []
    for ep in range(12):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream); S.hogwild_epoch(dds, model, S.Task.SVM, 0.01, plan); b.record(stream); evs.append((a, b))
        losses.append(S.device_loss(dds, model, S.Task.SVM))
    torch.cuda.synchronize()
    print(json.dumps({"mode": mode, "workers": workers, "epoch_us": round(1e3 * float(np.median([x.elapsed_time(y) for x, y in evs[2:]])), 2), "loss": [round(v, 1) for v in losses[:4]] + [round(losses[-1], 1)]}), flush=True)
