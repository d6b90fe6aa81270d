"""Small driver for ncu captures: runs a few epochs of one target op.

    python scripts/prof_targets.py {hogwild_w8a|hogwild_rcv1|hogwild_rcv1_block|hogwild_rcv1_block8|hogwild_w8a_example|
                                    sync_covtype|sync_rcv1|sync_realsim|sync_news20|sync_dense1000|sync_c5|
                                    minibatch_covtype|minibatch_rcv1|minibatch_w8a} [epochs]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_08800_b200 as S  # noqa: E402


def main():
    target = sys.argv[1]
    epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    torch.cuda.init()
    dev = S.Device(0, stream=torch.cuda.current_stream().cuda_stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    if target == "hogwild_w8a":
        host = S.fixtures.sparse_classification(64700, 300, 11.65, 20250811)
        dds = S.DeviceDataset(dev, host)
        plan = S.parse_plan("row-ch:kernel:0")
        plan.workers = dev.resident_workers(dds)
        model = S.DeviceModel(dev, host.n_features)
        for _ in range(epochs):
            flush.zero_()
            S.hogwild_epoch(dds, model, S.Task.SVM, 0.01, plan)
    elif target == "hogwild_rcv1":
        host = S.fixtures.sparse_classification(677399, 47236, 73.16, 20250813)
        dds = S.DeviceDataset(dev, host)
        plan = S.parse_plan("row-ch:kernel:0")
        plan.workers = dev.resident_workers(dds)
        model = S.DeviceModel(dev, host.n_features)
        for _ in range(epochs):
            flush.zero_()
            S.hogwild_epoch(dds, model, S.Task.LR, 0.01, plan)
    elif target in ("hogwild_rcv1_block", "hogwild_rcv1_block8"):
        host = S.fixtures.sparse_classification(677399, 47236, 73.16, 20250813)
        dds = S.DeviceDataset(dev, host)
        plan = S.parse_plan("row-ch:block:0")
        plan.workers = dev.resident_workers(dds)
        if target.endswith("8"):
            plan.group_size = plan.workers // 8  # 8 replicas in L2 (K6g)
        model = S.DeviceModel(dev, host.n_features)
        for _ in range(epochs):
            flush.zero_()
            S.hogwild_epoch(dds, model, S.Task.LR, 0.01, plan)
    elif target == "hogwild_w8a_example":
        host = S.fixtures.sparse_classification(64700, 300, 11.65, 20250811)
        dds = S.DeviceDataset(dev, host)
        plan = S.parse_plan("row-ch:example:0")
        plan.workers = dev.resident_workers(dds)
        model = S.DeviceModel(dev, host.n_features)
        for _ in range(epochs):
            flush.zero_()
            S.hogwild_epoch(dds, model, S.Task.SVM, 0.01, plan)
    elif target in ("minibatch_covtype", "minibatch_rcv1", "minibatch_w8a"):
        if target.endswith("covtype"):
            host, task, alpha = S.fixtures.dense_classification(581012, 54, 20250810), S.Task.LR, 1e-3
        elif target.endswith("w8a"):
            host, task, alpha = S.fixtures.sparse_classification(64700, 300, 11.65, 20250811), S.Task.SVM, 1e-3
        else:
            host, task, alpha = S.fixtures.sparse_classification(677399, 47236, 73.16, 20250813), S.Task.LR, 1e-2
        dds = S.DeviceDataset(dev, host)
        model = S.DeviceModel(dev, host.n_features)
        order = S.Schedule(1, host.n_examples).next()
        for _ in range(epochs):
            flush.zero_()
            S.sync_epoch(dds, model, task, alpha, order, 4096)
    elif target == "sync_c5":
        # C5 shape (d = 1000), device Philox generator; 2M rows = 8 GB > L2.
        dds = S.DeviceDataset.generate_dense(dev, 2_000_000, 1000, 20250814)
        model = S.DeviceModel(dev, 1000)
        for _ in range(epochs):
            S.sync_epoch(dds, model, S.Task.LR, 1e-7, None, 2_000_000)
    else:
        name = target.split("_")[1]
        if name == "covtype":
            host, task = S.fixtures.dense_classification(581012, 54, 20250810), S.Task.LR
        elif name == "news20":
            host, task = S.fixtures.sparse_classification(19996, 1355191, 455.0, 20250814), S.Task.SVM
        elif name == "realsim":
            host, task = S.fixtures.sparse_classification(72309, 20958, 51.3, 20250812), S.Task.SVM
        elif name == "dense1000":
            host, task = S.fixtures.dense_classification(200000, 1000, 7), S.Task.LR
        else:
            host, task = S.fixtures.sparse_classification(677399, 47236, 73.16, 20250813), S.Task.LR
        dds = S.DeviceDataset(dev, host)
        model = S.DeviceModel(dev, host.n_features)
        for _ in range(epochs):
            flush.zero_()
            S.sync_epoch(dds, model, task, 1e-6, None, host.n_examples)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
