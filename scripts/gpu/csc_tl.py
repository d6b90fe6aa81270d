import os, sys
import torch
sys.path.insert(0, os.getcwd())
import paper_1802_08800_b200 as S
torch.cuda.init(); stream = torch.cuda.current_stream()
dev = S.Device(0, stream=stream.cuda_stream)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
host = S.fixtures.sparse_classification(677399, 47236, 73.16, 20250813); dds = S.DeviceDataset(dev, host)
model = S.DeviceModel(dev, host.n_features)
os.environ["SGDB_CSC_TL"] = "1"
for _ in range(3):
    flush.zero_(); torch.cuda.synchronize()
    S.sync_epoch(dds, model, S.Task.LR, 1e-6, None, host.n_examples)
