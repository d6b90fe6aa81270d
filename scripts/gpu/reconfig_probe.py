"""Does the L2 flush (torch memset between epochs) cost our SMEM-heavy kernels
an SM carveout reconfiguration at their start? covtype / rcv1 full-batch
epochs timed after: a memset flush; no flush; a memset flush followed by an
untimed epoch of a tiny dataset (same kernels, restores the SMEM config, does
not touch the big data)."""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1802_08800_b200 as S
torch.cuda.init(); stream = torch.cuda.current_stream()
dev = S.Device(0, stream=stream.cuda_stream)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name, make, task in [("covtype", lambda: S.fixtures.dense_classification(581012, 54, 20250810), S.Task.LR),
                         ("rcv1", lambda: S.fixtures.sparse_classification(677399, 47236, 73.16, 20250813), S.Task.LR)]:
    host = make(); dds = S.DeviceDataset(dev, host); model = S.DeviceModel(dev, host.n_features)
    tiny_host = (S.fixtures.dense_classification(4096, 54, 1) if name == "covtype" else
                 S.fixtures.sparse_classification(4096, 47236, 73.16, 1))
    tiny = S.DeviceDataset(dev, tiny_host); tm = S.DeviceModel(dev, tiny_host.n_features)
    for method in ("memset", "none", "memset+tiny"):
        evs = []
        for _ in range(8):
            if method != "none": flush.zero_()
            if method == "memset+tiny": S.sync_epoch(tiny, tm, task, 1e-6, None, 4096, check_finite=False)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream); S.sync_epoch(dds, model, task, 1e-6, None, host.n_examples, check_finite=False); b.record(stream)
            evs.append((a, b))
        torch.cuda.synchronize()
        print(json.dumps({"data": name, "flush": method, "epoch_us": round(1e3 * float(np.median([x.elapsed_time(y) for x, y in evs[2:]])), 1)}), flush=True)
    del dds, tiny
