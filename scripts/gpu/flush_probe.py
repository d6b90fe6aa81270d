"""How the L2 flush method affects a short kernel: memset (leaves L2 full of
dirty lines the next kernel must write back) vs memset + read (clean L2)."""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1802_08800_b200 as S
torch.cuda.init(); stream = torch.cuda.current_stream()
dev = S.Device(0, stream=stream.cuda_stream)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush2 = torch.empty(256 << 20, dtype=torch.uint8, device="cuda").fill_(1)
host = S.fixtures.sparse_classification(64700, 300, 11.65, 20250811); dds = S.DeviceDataset(dev, host)
def run(method, chunk):
    os.environ["SGDB_HOGWILD_CHUNK"] = chunk
    plan = S.parse_plan("row-ch:kernel:0"); plan.workers = dev.resident_workers(dds)
    model = S.DeviceModel(dev, host.n_features)
    S.hogwild_epoch(dds, model, S.Task.SVM, 0.01, plan)
    evs = []
    for _ in range(10):
        if method == "memset": flush.zero_()
        elif method == "memset+read": flush.zero_(); flush2.sum(dtype=torch.int32)
        elif method == "read": flush2.sum(dtype=torch.int32)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream); S.hogwild_epoch(dds, model, S.Task.SVM, 0.01, plan); b.record(stream); evs.append((a, b))
    torch.cuda.synchronize()
    return round(1e3 * float(np.median([x.elapsed_time(y) for x, y in evs])), 2)
for method in ("memset", "memset+read", "read", "none"):
    print(json.dumps({"flush": method, "K5_us": run(method, "0"), "K5c_us": run(method, "1")}), flush=True)
