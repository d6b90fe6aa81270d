import os, sys
import torch
sys.path.insert(0, os.getcwd())
import paper_1802_08800_b200 as S
torch.cuda.init(); stream = torch.cuda.current_stream()
dev = S.Device(0, stream=stream.cuda_stream)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
host = S.fixtures.sparse_classification(64700, 300, 11.65, 20250811); dds = S.DeviceDataset(dev, host)
os.environ["SGDB_HOGWILD_TL"] = "1"
for workers in (4736, 2368, 1184):
    plan = S.parse_plan("row-ch:kernel:0"); plan.workers = workers
    model = S.DeviceModel(dev, host.n_features)
    for _ in range(3):
        flush.zero_(); torch.cuda.synchronize()
        print("workers", workers, file=sys.stderr, flush=True)
        S.hogwild_epoch(dds, model, S.Task.SVM, 0.01, plan)
