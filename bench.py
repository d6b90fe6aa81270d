#!/usr/bin/env python
"""bench.py — headline benchmark of the B200 GLM SGD engine.

Workload (BASELINE.json configs[1]): SVM Hogwild async SGD, warp-group-per-
example kernel, on sparse synthetic w8a-shaped data — 64,700 x 300 CSR,
fixtures::sparse_classification(64700, 300, 11.65, 20250811),
plan row-ch + kernel + no-rep with every resident lane group a worker.

A step is one Hogwild epoch over the dataset. metric = examples/sec per epoch
(N / t_epoch); the whole-job value at N GPUs is N*n / t_epoch
(weak scaling: every rank trains its own w8a-shaped partition, seed + rank,
and the replicas are averaged over NCCL after every epoch). The dataset
(6.5 MB) is L2-resident, so L2 is flushed (256 MiB memset) before every timed
epoch, outside the per-epoch CUDA-event window.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_EX, D, AVG, SEED = 64700, 300, 11.65, 20250811
PLAN = "row-ch:kernel:0"
TASK_SVM = 1
METRIC = "examples/sec per epoch (SVM Hogwild, w8a-shaped 64,700x300 CSR)"
UNIT = "examples/s"
WORKLOAD = "C2 w8a-shaped SVM Hogwild (BASELINE.json configs[1])"


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def _ncu_traffic(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from
    the committed `ncu --set full` summary (profiles/round1_ncu_*_current.txt,
    written by scripts/ncu_summary.py from scripts/round1_profile.sh)."""
    import glob
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "round1_ncu_*_current.txt"))):
        cur, got = None, {}
        for line in open(path):
            if line.startswith("== "):
                cur = line
                continue
            parts = line.split()
            if cur and kernel in cur and parts and parts[0] in ("dram__bytes_read.sum",
                                                                 "dram__bytes_write.sum"):
                got[parts[0]] = float(parts[1]) * scale.get(parts[2], 1)
        if len(got) == 2:
            return int(sum(got.values())), os.path.relpath(path, ROOT)
    return None, None


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    smax.append(float(parts[2]))
                except ValueError:
                    continue
                for nm, v in zip(names, parts[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        finally:
            if self.path and os.path.exists(self.path):
                os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax),
                "reasons": sorted(reasons), "samples": len(sm)}


def _reference_time_epochs(ref, ds, plan, workers, epochs, alpha, handle=None):
    _, losses, secs, _ = ref.hogwild_train(ds, TASK_SVM, alpha, epochs, plan, workers=workers,
                                           handle=handle)
    return losses, secs


def _epochs_to(losses, l_star, tol=0.01):
    for i, v in enumerate(losses):
        if v <= (1 + tol) * l_star:
            return i + 1
    return None


# --------------------------------------------------------------------------------------
def run_reference(args):
    """--impl reference: the reference's own CPU Hogwild (oracle/_ref, built from
    /root/reference/proj/src) with every host thread, same workload/metric."""
    rank = _env_int("RANK", 0)
    if rank != 0:
        return 0
    import oracle
    if not oracle.reference_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return 0
    ref = oracle.reference()
    ds = ref.fixture_sparse(N_EX, D, AVG, SEED)
    threads = ref.hardware_threads()
    h = ref.to_handle(ds)
    try:
        epochs = args.warmup + args.steps
        _, secs = _reference_time_epochs(ref, ds, PLAN, threads, epochs, 0.01, handle=h)
    finally:
        ref.lib.ref_ds_free(h)
    timed = list(secs[args.warmup:]) or list(secs)
    mean = float(np.mean(timed))
    value = N_EX / mean
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": len(timed), "warmup": args.warmup,
        "ms_per_step": mean * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference fixtures)",
        "config": {"workload": WORKLOAD, "plan": PLAN, "workers": threads,
                   "n": N_EX, "d": D},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{len(timed)} timed epochs of hogwild::train (+{args.warmup} "
                                   f"warm-up), EpochRecord.seconds mean"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))
    return 0


# --------------------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1802_08800_b200 as S
    from paper_1802_08800_b200 import distributed as SD

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(local)
    torch.cuda.init()
    stream = torch.cuda.current_stream()
    dev = S.Device(local, stream=stream.cuda_stream)
    SD.attach(dev)

    host = S.fixtures.sparse_classification(N_EX, D, AVG, SEED + rank)
    dds = S.DeviceDataset(dev, host)
    model = S.DeviceModel(dev, D)
    plan = S.parse_plan(PLAN)
    plan.workers = dev.resident_workers(dds) if args.workers <= 0 else args.workers
    alpha = args.alpha
    task = S.Task.SVM
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def step():
        # N > 1: rank replicas averaged args.segments times per epoch (§8(e)).
        SD.hogwild_epoch_ranks(dev, dds, model, task, alpha, plan, world, args.segments)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        flush.zero_()
        step()
    barrier()
    launches0 = dev.launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    with ClockSampler(local) as clocks:
        barrier()
        t_wall0 = time.perf_counter()
        for i in range(args.steps):
            flush.zero_()  # L2 flush, outside the event window
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        barrier()
        t_wall1 = time.perf_counter()
    launches = dev.launch_count() - launches0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = float(np.mean(step_ms))
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * N_EX / (ms / 1e3)

    # Dominant-kernel roofline: per-launch CUDA-event time of hogwild_kernel.
    dev.set_profiling(True)
    for _ in range(args.steps):
        flush.zero_()
        step()
    stats = dev.kernel_stats()
    dev.set_profiling(False)
    name = "hogwild_kernel"
    launches_k, total_ms = stats.get(name, (0, 0.0))
    kern_ms = total_ms / max(1, launches_k)
    sweep = dds.sweep_bytes()
    peak, peak_src = _peaks()
    traffic, traffic_src = _ncu_traffic("hogwild_kernel")
    achieved = sweep / (kern_ms / 1e3) / 1e9 if kern_ms > 0 else 0.0
    share = total_ms / max(1e-9, sum(v[1] for v in stats.values()))

    # End to end through the public API with host buffers: per step, pinned-host
    # fp32 CSR arrays -> device (sgdb_dataset_refresh_f32), the epoch, and the
    # trained model back to the host (sgdb_model_get).
    vals = torch.from_numpy(host.values.astype(np.float32)).pin_memory()
    labs = torch.from_numpy(host.labels.astype(np.float32)).pin_memory()
    # Column ids travel as 16 bits (d <= 65536) and are widened on the device
    # (sgdb_dataset_refresh_idx16); values, labels and row offsets as fp32 / u32.
    idx = torch.from_numpy(host.indices.astype(np.uint16).view(np.int16)).pin_memory()
    rp = torch.from_numpy(host.row_offsets.astype(np.int32)).pin_memory()
    h2d = vals.numel() * 4 + labs.numel() * 4 + idx.numel() * 2 + rp.numel() * 4
    d2h = D * 8
    e2e_steps = max(3, args.steps)
    # Double-buffered: step k+1's inputs are copied into the other device buffer
    # on a copy stream while step k's epoch runs; every step still copies its
    # whole input from pinned host memory and reads its result back.
    # Two copy streams: the values on one, ids / labels / offsets on the other
    # (B200 has several copy engines; SGDB_E2E_STREAMS=1 uses one).
    n_copy = 1 if os.environ.get("SGDB_E2E_STREAMS") == "1" else 2
    copy_streams = [torch.cuda.Stream() for _ in range(n_copy)]
    copy_devs = [S.Device(local, stream=cs.cuda_stream) for cs in copy_streams]
    cA, cB = copy_devs[0], copy_devs[-1]
    bufs = [S.DeviceDataset(dev, host), S.DeviceDataset(dev, host)]  # dds keeps its CSC copy
    ready = [[torch.cuda.Event() for _ in range(n_copy)] for _ in range(2)]
    free = [torch.cuda.Event(), torch.cuda.Event()]
    used = [False, False]

    def refresh(b):
        bufs[b].refresh_f32(vals, None, None, None, device=cA)
        bufs[b].refresh_f32(None, labs, None, rp, device=cB)
        bufs[b].refresh_idx16(idx, device=cB)
        for ev, cs in zip(ready[b], copy_streams):
            ev.record(cs)

    def e2e_step(k):
        b = k % 2
        if k + 1 < e2e_steps:
            nb = 1 - b
            if used[nb]:
                for cs in copy_streams:
                    cs.wait_event(free[nb])
            refresh(nb)
        for ev in ready[b]:
            stream.wait_event(ev)
        SD.hogwild_epoch_ranks(dev, bufs[b], model, task, alpha, plan, world, args.segments)
        free[b].record(stream)
        used[b] = True
        model.get()

    def e2e_run():
        used[0] = used[1] = False
        refresh(0)  # step 0's inputs
        for k in range(e2e_steps):
            e2e_step(k)

    # Untimed warm-up: the host->device path takes a few dozen transfers to
    # reach steady state (freshly pinned buffers, link power state).
    for _ in range(max(3, args.warmup)):
        e2e_run()
    barrier()
    t0 = time.perf_counter()
    e2e_run()
    barrier()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = world * N_EX / e2e_s

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference fixtures, seed+rank)",
        "config": {"workload": WORKLOAD, "plan": PLAN, "workers": plan.workers,
                   "replica_averages_per_epoch": args.segments if world > 1 else 0,
                   "lanes_per_worker": "auto", "alpha": alpha, "n_per_gpu": N_EX, "d": D,
                   "nnz_per_gpu": dds.nnz, "l2": "flushed before every step (256 MiB memset, "
                                                  "outside the event window)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "kernel": name,
                     "kernel_ms": kern_ms, "kernel_share_of_step": share,
                     "algorithmic_bytes_per_launch": sweep, "peak_source": peak_src},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3,
                "copy_streams": n_copy,
                "pipeline": "double-buffered: step k+1's H2D (copy streams) overlaps step k's "
                            "epoch; every step copies its inputs (column ids as 16 bits, widened "
                            "on the device) and reads the model back"},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "wall_s_timed_region": t_wall1 - t_wall0,
        "step_ms_median": float(np.median(step_ms)),
    }
    if not args.no_extra:
        extra = {}
        extra["c5_sync_lr_dense1000"] = extra_c5(S, dev, world, rank, args.c5_rows, barrier)
        if world == 1:
            extra["sync_full_batch"] = extra_sync_shapes(S, dev)
        out["extra"] = extra
    if rank == 0 and world == 1 and not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(host)
    if rank == 0 and not args.no_convergence:
        out["convergence"] = convergence(S, dev, dds, plan, alpha, ms, out.get("cpu_baseline"))
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def _time_epochs(S, dds, model, task, alpha, epochs, warmup, flush=None):
    import torch
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        S.sync_epoch(dds, model, task, alpha, None, dds.n_global)
    # Epochs are enqueued asynchronously (no per-epoch flag read-back), so the
    # host's launch latency hides behind the L2 flush that precedes each one;
    # the events bracket the epoch's kernels on the stream. Divergence is
    # checked once afterwards.
    evs = []
    for _ in range(epochs):
        if flush is not None:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        S.sync_epoch(dds, model, task, alpha, None, dds.n_global, check_finite=False)
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    times = [a.elapsed_time(b) for a, b in evs]
    assert S.sync_epoch(dds, model, task, alpha, None, dds.n_global), "diverged"
    return float(np.mean(times))


def extra_c5(S, dev, world, rank, rows_per_gpu, barrier):
    """BASELINE.json configs[4]: row-sharded synchronous LR on
    dense 1,000-d data, rows_per_gpu rows per GPU generated on the device (K9),
    full-batch epochs, fp64 gradient all-reduced over NCCL when N > 1."""
    import torch
    import torch.distributed as dist
    d = 1000
    n_global = rows_per_gpu * world
    dds = S.DeviceDataset.generate_dense(dev, rows_per_gpu, d, 20250815, row_base=rank * rows_per_gpu,
                                         n_global=n_global)
    model = S.DeviceModel(dev, d)
    barrier()
    dev.set_profiling(True)
    ms = _time_epochs(S, dds, model, S.Task.LR, 1e-9, 5, 2)
    stats = dev.kernel_stats()
    dev.set_profiling(False)
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    k = stats.get("dense_full_kernel", (1, 0.0))
    kern_ms = k[1] / max(1, k[0])
    sweep = dds.sweep_bytes()
    peak, _ = _peaks()
    loss = S.device_loss(dds, model, S.Task.LR)
    out = {"rows_per_gpu": rows_per_gpu, "n_global": n_global, "d": d, "batch": "N",
           "epoch_ms": ms, "value": n_global / (ms / 1e3), "unit": UNIT,
           "kernel": "dense_full_kernel", "kernel_ms": kern_ms,
           "hbm_GBps": sweep / (kern_ms / 1e3) / 1e9 if kern_ms else None,
           "frac": sweep / (kern_ms / 1e3) / 1e9 / peak if kern_ms else None,
           "loss_after": loss, "scaling": "weak",
           "note": "epoch = dense_full_kernel + NCCL all-reduce of g (d fp64) + apply when N > 1"}
    del dds
    torch.cuda.empty_cache()
    return out


def _time_hogwild(S, dds, model, task, alpha, plan, epochs, warmup, flush):
    import torch
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        S.hogwild_epoch(dds, model, task, alpha, plan)
    evs = []
    for _ in range(epochs):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        S.hogwild_epoch(dds, model, task, alpha, plan)
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    return float(np.mean([x.elapsed_time(y) for x, y in evs]))


def extra_sync_shapes(S, dev):
    """Full-batch synchronous epochs on the other BASELINE shapes,
    and Hogwild epochs with the paper's plan for the shapes BASELINE.json runs
    asynchronously (C3, C4a, C4b; kernel scope, every resident warp a worker)."""
    import torch
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    shapes = {
        "C1_covtype_lr": (lambda: S.fixtures.dense_classification(581012, 54, 20250810), S.Task.LR, 1e-6,
                          None, None),
        "C3_rcv1_lr": (lambda: S.fixtures.sparse_classification(677399, 47236, 73.16, 20250813), S.Task.LR, 1e-6,
                       "row-ch:kernel:0", 1e-2),
        "C4a_news20_svm": (lambda: S.fixtures.sparse_classification(19996, 1355191, 455.0, 20250814), S.Task.SVM, 1e-5,
                           "row-ch:kernel:0", 1e-4),
        "C4b_realsim_svm": (lambda: S.fixtures.sparse_classification(72309, 20958, 51.3, 20250812), S.Task.SVM, 1e-5,
                            "row-ch:kernel:0", 1e-3),
    }
    peak, _ = _peaks()
    out = {}
    for name, (make, task, alpha, plan_text, async_alpha) in shapes.items():
        host = make()
        dds = S.DeviceDataset(dev, host)
        model = S.DeviceModel(dev, host.n_features)
        ms = _time_epochs(S, dds, model, task, alpha, 5, 2, flush)
        sweep = dds.sweep_bytes()
        out[name] = {"n": host.n_examples, "d": host.n_features, "epoch_ms": ms,
                     "value": host.n_examples / (ms / 1e3), "unit": UNIT,
                     "alg_GBps": sweep / (ms / 1e3) / 1e9, "frac": sweep / (ms / 1e3) / 1e9 / peak}
        if plan_text:
            plan = S.parse_plan(plan_text)
            plan.workers = dev.resident_workers(dds)
            hm = S.DeviceModel(dev, host.n_features)
            ams = _time_hogwild(S, dds, hm, task, async_alpha, plan, 5, 2, flush)
            out[name]["hogwild"] = {
                "plan": plan_text, "workers": plan.workers, "epoch_ms": ams,
                "value": host.n_examples / (ams / 1e3), "unit": UNIT,
                "alg_GBps": sweep / (ams / 1e3) / 1e9, "frac": sweep / (ams / 1e3) / 1e9 / peak,
                "note": "bound by L2 transactions (one model gather + one red.add per nonzero) and "
                        "the per-example gather chain, not HBM (DESIGN.md §4)"}
            del hm
        del dds, model, host
    return out


def cpu_baseline(host):
    """The unmodified reference (oracle/_ref) timed on this box's host cores:
    hogwild::train, same data and plan, 1 worker (sequential Alg. 3)."""
    import oracle
    if not oracle.reference_available():
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                "sample": "unavailable: oracle/_ref not built"}
    ref = oracle.reference()
    h = ref.to_handle(host)
    try:
        epochs = 400
        t0 = time.perf_counter()
        _, secs = _reference_time_epochs(ref, host, PLAN, 1, epochs, 0.01, handle=h)
        wall = time.perf_counter() - t0
        threads = ref.hardware_threads()
        _, secs_mt = _reference_time_epochs(ref, host, PLAN, threads, 100, 0.01, handle=h)
    finally:
        ref.lib.ref_ds_free(h)
    v1 = N_EX / float(np.mean(secs))
    vmt = N_EX / float(np.mean(secs_mt))
    return {"value": v1, "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"{epochs} epochs of the reference hogwild::train, 1 worker, full w8a-shaped "
                      f"data ({wall:.1f} s wall incl. loss)",
            "multithread": {"value": vmt, "cores": threads, "sample": "100 epochs"}}


def convergence(S, dev, dds, plan, alpha, ms_epoch, cpu):
    """Time to 1% of L* (harness.cpp:44-50): L* = min loss over GPU batch-GD probes
    (alpha grid, harness.cpp:275-289) and the runs below."""
    task = S.Task.SVM
    l_star = float("inf")
    for a in (1e-5, 1e-4, 1e-3, 1e-2):
        r = S.sync.train(task, dds, S.Hyperparams(alpha=a, batch_b=dds.n_global, epochs=300,
                                                  task=task), 0)
        l_star = min([l_star] + [v for v in r.trace.losses() if np.isfinite(v)])
    hp = S.Hyperparams(alpha=alpha, batch_b=1, epochs=100, task=task)
    gpu = S.hogwild.train(task, dds, hp, plan, 0)
    l_star = min([l_star] + gpu.trace.losses())
    out = {"l_star": l_star, "gpu_epochs_to_1pct": _epochs_to(gpu.trace.losses(), l_star)}
    if out["gpu_epochs_to_1pct"]:
        out["gpu_time_to_1pct_s"] = out["gpu_epochs_to_1pct"] * ms_epoch / 1e3
    try:
        import oracle
        if oracle.reference_available():
            ref = oracle.reference()
            host = dds.host
            _, losses, secs, _ = ref.hogwild_train(host, 1, alpha, 100, PLAN, workers=1)
            e = _epochs_to(list(losses), l_star)
            out["cpu_epochs_to_1pct"] = e
            if e:
                out["cpu_time_to_1pct_s"] = float(np.sum(secs[:e]))
    except Exception as exc:  # reported, not fatal
        out["cpu_error"] = str(exc)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workers", type=int, default=0, help="0 = every resident lane group")
    ap.add_argument("--alpha", type=float, default=0.01)
    ap.add_argument("--segments", type=int, default=1,
                    help="N > 1: cross-rank replica averages per Hogwild epoch")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-convergence", action="store_true")
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--c5-rows", type=int, default=25_000_000,
                    help="rows per GPU of the 200M x 1000 configuration (25M = 8 GPUs x 25M)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
