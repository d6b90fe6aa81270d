"""warpsim cross-check: the reference's warp lockstep
simulator (proj/src/simd_sim.cpp, warpsim::simulate_epoch /
count_transactions) against the sectors a real sm_100a warp moves.

The simulator's "thread per example" warp — 32 lanes, each lane a Hogwild
worker walking its assign() list, one coordinate access per lane per
micro-step — is exactly the device's Hogwild kernel with one lane per worker
(lanes_per_worker = 1) and 32 workers on one model in global memory (here:
block scope with one replica of 32 workers, a flat fp32 layout with red.add
updates, kernels_hogwild.cu). The simulator counts the distinct
segment_size-coordinate segments touched per lockstep access; with fp32 data
and model and segment_size = 8, a segment is one 32-byte L1/L2 sector.

    python scripts/warpsim_crosscheck.py gpu          # one epoch per case (run under ncu)
    python scripts/warpsim_crosscheck.py report CSV   # join the ncu sectors with the simulator

Per case the report gives the simulator's total memory_transactions and its
split by access kind (recomputed with the reference's own count_transactions
on the lanes' address streams), the device's global-load and reduction
sectors (ncu l1tex__t_sectors_pipe_lsu_mem_global_op_{ld,red}.sum), and the
prediction device_ld = data + model + data again (the device kernel re-reads
each x value in its update loop, where the simulator keeps it), device_red =
writes.
"""
import csv
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

N, D, SEED = 2048, 64, 31
CASES = [("row-major", "row-rr"), ("row-major", "row-ch"), ("col-major", "col-rr"),
         ("col-major", "col-ch")]
W = 32  # lanes = workers
SEG = 8


def _data(S):
    ds = S.fixtures.dense_classification(N, D, SEED).rounded_f32()
    return {"row-major": ds, "col-major": S.convert_layout(ds, S.Layout.DenseColMajor)}


def gpu():
    import torch
    import paper_1802_08800_b200 as S
    dev = S.Device(0, stream=torch.cuda.current_stream().cuda_stream)
    data = _data(S)
    for layout, access in CASES:
        ds = data[layout]
        dds = S.DeviceDataset(dev, ds)
        m = S.DeviceModel(dev, D)
        plan = S.parse_plan(f"{access}:block:0")
        plan.workers, plan.group_size, plan.lanes_per_worker = W, W, 1
        S.hogwild_epoch(dds, m, S.Task.LR, 0.01, plan)
        torch.cuda.synchronize()
        print(json.dumps({"case": f"{layout} {access}"}), flush=True)


def _streams(ds_rows, access, assign):
    """Per-lane address streams by kind for a dense dataset in lockstep (every
    row has D slots): data (value addresses in the plan's storage order),
    model (coordinates), writes (coordinates, rotated by the circular offset
    lane % D as warpsim and process_examples do)."""
    col = access.startswith("col")
    data, model, write, reread = [], [], [], []
    for lane, lst in enumerate(assign):
        dl, ml, wl, rl = [], [], [], []
        for e in lst:
            for s in range(D):
                dl.append(s * N + e if col else e * D + s)
                ml.append(s)
            start = lane % D
            for i in range(D):
                s = (start + i) % D
                wl.append(s)
                rl.append(s * N + e if col else e * D + s)
        data.append(dl), model.append(ml), write.append(wl), reread.append(rl)
    return data, model, write, reread


def report(csv_path, out_path=None):
    import oracle
    ref = oracle.reference()
    # ncu csv: one row per (launch, metric)
    rows = list(csv.reader(open(csv_path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Name" in r)
    h = rows[hi]
    launches = {}
    for r in rows[hi + 1:]:
        d = dict(zip(h, r))
        if "hogwild_kernel" not in d.get("Kernel Name", ""):
            continue
        key = int(d["ID"])
        launches.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    measured = [launches[k] for k in sorted(launches)]
    strategy = {"row-rr": True, "col-rr": True, "row-ch": False, "col-ch": False}
    out = []
    for (layout, access), meas in zip(CASES, measured):
        host = ref.fixture_dense(N, D, SEED)
        ds = ref.convert_layout(host, 1) if layout == "col-major" else host
        _, st = ref.warpsim_epoch(ds, 0, 0.01, f"{access}:kernel:0", W, SEG, True)
        assign = ref.assign(N, W, strategy[access], 0)
        data, model, write, reread = _streams(None, access, assign)
        kinds = {k: ref.count_transactions(v, SEG) for k, v in
                 (("data", data), ("model", model), ("write", write), ("data_reread", reread))}
        ld = meas.get("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", float("nan"))
        red = meas.get("l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum", 0.0) + \
            meas.get("l1tex__t_sectors_pipe_lsu_mem_global_op_atom.sum", 0.0)
        pred_ld = kinds["data"] + kinds["model"] + kinds["data_reread"]
        rec = {"case": f"{layout} {access}", "warp_width": W, "segment_size": SEG,
               "sim_memory_transactions": st["memory_transactions"],
               "sim_split": {k: kinds[k] for k in ("data", "model", "write")},
               "sim_split_sum": kinds["data"] + kinds["model"] + kinds["write"],
               "device_ld_sectors": ld, "device_red_sectors": red,
               "predicted_device_ld": pred_ld, "predicted_device_red": kinds["write"],
               "ld_ratio": ld / pred_ld if pred_ld else None,
               "red_ratio": red / kinds["write"] if kinds["write"] else None}
        out.append(rec)
        print(json.dumps(rec))
    if out_path:
        with open(out_path, "w") as f:
            for r in out:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    if sys.argv[1] == "gpu":
        gpu()
    else:
        report(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
