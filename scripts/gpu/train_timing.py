import os, sys, time
import numpy as np
sys.path.insert(0, os.getcwd())
import paper_1802_08800_b200 as S
dev = S.Device(0)
host = S.fixtures.sparse_classification(677399, 47236, 73.16, 20250813)
dds = S.DeviceDataset(dev, host)
plan = S.parse_plan("row-ch:kernel:0"); plan.workers = dev.resident_workers(dds)
hp = S.Hyperparams(alpha=0.01, batch_b=1, epochs=6, task=S.Task.LR)
r = S.hogwild.train(S.Task.LR, dds, hp, plan, 0)
print("hogwild.train epoch s:", [round(e.seconds * 1e3, 3) for e in r.trace.epochs])
m = S.DeviceModel(dev, host.n_features)
for i in range(4):
    dev.synchronize(); t0 = time.perf_counter()
    S.hogwild_epoch(dds, m, S.Task.LR, 0.01, plan)
    dev.synchronize(); t1 = time.perf_counter()
    l = S.device_loss(dds, m, S.Task.LR)
    print("epoch+sync ms", round((t1 - t0) * 1e3, 3))
hp2 = S.Hyperparams(alpha=1e-6, batch_b=host.n_examples, epochs=4, task=S.Task.LR)
r2 = S.sync.train(S.Task.LR, dds, hp2, 0)
print("sync.train epoch s:", [round(e.seconds * 1e3, 3) for e in r2.trace.epochs])
