"""B = N epoch timer used for the late round-2 A/B runs of the full-batch step.

The variant under test is chosen outside this script (the library is swapped
between runs, or a since-removed switch selected it); SGDB_FUSED_AB only labels
the run. Per shape: median device-timed epoch at B = N (L2 flushed, written then
read, before each), the kernel breakdown, and the fp64 model after 5 epochs
saved to gpurun_out/fused_ab_<label>_<shape>.npy; `--compare` reports the
model difference between labels 0 and 1. Results: profiles/round2_*_ab.jsonl,
profiles/round2_fused_step_experiment.jsonl, round2_dense_tile_sweep.jsonl.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")


def compare(names):
    for name in names:
        a = np.load(os.path.join(OUT, f"fused_ab_0_{name}.npy"))
        b = np.load(os.path.join(OUT, f"fused_ab_1_{name}.npy"))
        print(json.dumps({"data": name, "model_rel_l2": float(np.linalg.norm(a - b) / np.linalg.norm(a))}))


def main():
    import torch
    import paper_1802_08800_b200 as S
    from sync_sweep import CFG

    mode = os.environ.get("SGDB_FUSED_AB", "rule")
    torch.cuda.init()
    stream = torch.cuda.current_stream()
    dev = S.Device(0, stream=stream.cuda_stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for name in sys.argv[1:]:
        host, task, alpha = CFG[name]()
        dds = S.DeviceDataset(dev, host)
        n = host.n_examples
        sweep = dds.sweep_bytes()
        model = S.DeviceModel(dev, host.n_features)
        for _ in range(5):
            S.sync_epoch(dds, model, task, alpha, None, n, check_finite=False)
        torch.cuda.synchronize()
        os.makedirs(OUT, exist_ok=True)
        np.save(os.path.join(OUT, f"fused_ab_{mode}_{name}.npy"), model.get())
        evs = []
        for _ in range(20):
            flush.zero_(); flush.view(torch.float32).sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            S.sync_epoch(dds, model, task, alpha, None, n, check_finite=False)
            e1.record(stream)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        t = sorted(a.elapsed_time(b) for a, b in evs[3:])
        dev.set_profiling(True)
        for _ in range(3):
            flush.zero_(); flush.view(torch.float32).sum()
            S.sync_epoch(dds, model, task, alpha, None, n)
        stats = dev.kernel_stats()
        dev.set_profiling(False)
        ms = t[len(t) // 2]
        print(json.dumps({"mode": mode, "data": name, "epoch_us": round(ms * 1e3, 2),
                          "min_us": round(t[0] * 1e3, 2), "frac_one_sweep": sweep / (ms / 1e3) / 1e9 / 6538.3,
                          "kernels_us": {k: round(v[1] / 3 * 1e3, 2) for k, v in stats.items()},
                          "loss": S.device_loss(dds, model, task)}), flush=True)


if __name__ == "__main__":
    if sys.argv[1:2] == ["--compare"]:
        compare(sys.argv[2:])
    else:
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        main()
