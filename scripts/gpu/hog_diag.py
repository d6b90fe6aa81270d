import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1802_08800_b200 as S
torch.cuda.init(); stream = torch.cuda.current_stream()
dev = S.Device(0, stream=stream.cuda_stream)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name, make, task in [("rcv1", lambda: S.fixtures.sparse_classification(677399, 47236, 73.16, 20250813), S.Task.LR),
                         ("w8a", lambda: S.fixtures.sparse_classification(64700, 300, 11.65, 20250811), S.Task.SVM)]:
    host = make(); dds = S.DeviceDataset(dev, host)
    for diag in (0, 1, 2, 3):
        os.environ["SGDB_HOGWILD_DIAG"] = str(diag)
        plan = S.parse_plan("row-ch:kernel:0"); plan.workers = dev.resident_workers(dds)
        model = S.DeviceModel(dev, host.n_features)
        S.hogwild_epoch(dds, model, task, 0.01, plan)
        evs = []
        for _ in range(6):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream); S.hogwild_epoch(dds, model, task, 0.01, plan); b.record(stream); evs.append((a, b))
        torch.cuda.synchronize()
        print(json.dumps({"data": name, "diag": diag, "epoch_us": round(1e3 * float(np.median([x.elapsed_time(y) for x, y in evs])), 1)}), flush=True)
    del dds
