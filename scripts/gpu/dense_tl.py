import os, sys
import torch
sys.path.insert(0, os.getcwd())
import paper_1802_08800_b200 as S
torch.cuda.init(); stream = torch.cuda.current_stream()
dev = S.Device(0, stream=stream.cuda_stream)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
host = S.fixtures.dense_classification(581012, 54, 20250810); dds = S.DeviceDataset(dev, host)
model = S.DeviceModel(dev, 54)
os.environ["SGDB_DENSE_TL"] = "1"
for _ in range(4):
    flush.zero_(); torch.cuda.synchronize()
    S.sync_epoch(dds, model, S.Task.LR, 1e-6, None, host.n_examples)
