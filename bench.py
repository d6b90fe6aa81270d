#!/usr/bin/env python
"""bench.py — headline benchmark of the B200 GLM SGD engine.

Workload (BASELINE.json configs[2], the largest configuration that fits one
GPU): logistic regression, synchronous SGD at B = N (the
paper's batch-GD sync benchmark) on sparse synthetic
rcv1-shaped data — fixtures::sparse_classification(677399, 47236, 73.16,
20250813), 48.9M nonzeros, values rounded to fp32 — step size 0.01.

A step is one epoch: margin pass, coefficients, gradient pass, update
(sync::train's epoch at B = N, proj/src/sync_engine.cpp:86-100). metric =
examples/sec per epoch (N / t_epoch); at N GPUs every rank owns
its own rcv1-shaped shard (seed + rank; weak scaling) and the fp64 gradient is
SUM-all-reduced every epoch by the engine's own NCCL communicator, so the
whole-job value is N * 677,399 / t_epoch. The stored data (397 MB CSR + 300 MB
blocked CSC) exceeds L2; L2 is flushed before every timed epoch anyway,
outside the event window: 256 MiB written, then read back, so the epoch starts
from a cold and CLEAN L2 (a write-only flush leaves 126 MB of dirty lines whose
write-back the next epoch's first kernel would pay: +14 us on rcv1,
profiles/round2_flush_modes.jsonl).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

--gpus N without a torchrun environment re-launches itself under
torch.distributed.run with N ranks. --impl reference times the unmodified
reference (oracle/_ref, built from /root/reference/proj/src) on the host: its
sync::train on the same configuration with every host thread.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_EX, D, AVG, SEED = 677399, 47236, 73.16, 20250813
ALPHA = 0.01
TASK_LR = 0
METRIC = "examples/sec per epoch (LR sync SGD, B = N, rcv1-shaped 677,399 x 47,236 CSR)"
UNIT = "examples/s"
WORKLOAD = "C3 rcv1-shaped LR, synchronous SGD at B = N (BASELINE.json configs[2])"


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def _ncu_traffic(kernel, summary="round2_ncu_rcv1_full_batch.txt"):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from
    the committed `ncu --set full` summary of the headline configuration
    (profiles/round2_ncu_rcv1_full_batch.txt, written by scripts/ncu_summary.py
    from scripts/round2_profile.sh)."""
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    # The library's profiler names -> the CUDA function ncu reports.
    kernel = {"k3s_grad_kernel": "blocked_pass_kernel<0,",
              "k2w_margin_kernel": "blocked_pass_kernel<1,",
              "k23g_step_kernel": "glued_step_kernel<"}.get(kernel, kernel)
    path = os.path.join(ROOT, "profiles", summary)
    if not os.path.exists(path):
        return None, None
    cur, got = None, {}
    for line in open(path):
        if line.startswith("== "):
            if cur and kernel in cur and len(got) == 2:
                break
            cur, got = line, {}
            continue
        parts = line.split()
        if cur and kernel in cur and parts and parts[0] in ("dram__bytes_read.sum",
                                                             "dram__bytes_write.sum"):
            got[parts[0]] = float(parts[1]) * scale.get(parts[2], 1)
    if cur and kernel in cur and len(got) == 2:
        return int(sum(got.values())), os.path.relpath(path, ROOT)
    return None, None


class L2Flush:
    """Between-step L2 flush: write 256 MiB (2x L2), then read it back so the
    next step starts cold AND clean (no dirty lines left for its first kernel
    to write back). Runs on torch's current stream, outside the event window."""

    def __init__(self):
        import torch
        self.buf = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
        self.sink = torch.empty((), dtype=torch.float32, device="cuda")

    def __call__(self):
        self.buf.zero_()
        self.sink.copy_(self.buf.sum())


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
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
                 "--format=csv,noheader,nounits", "-lms", "50"],
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


def _epochs_to(losses, l_star, tol=0.01):
    for i, v in enumerate(losses):
        if v <= (1 + tol) * l_star:
            return i + 1
    return None


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_under_torchrun(args) -> int:
    """--gpus N > 1 outside torchrun: start N ranks (one per GPU) on this node."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# --------------------------------------------------------------------------------------
def run_reference(args):
    """--impl reference: the reference's own CPU sync::train (oracle/_ref, built
    from /root/reference/proj/src), every host thread, same configuration."""
    if _env_int("RANK", 0) != 0:
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
        _, losses, secs, _ = ref.sync_train(ds, TASK_LR, ALPHA, N_EX, epochs, 7, workers=threads,
                                            handle=h)
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
        "config": {"workload": WORKLOAD, "task": "LR", "batch": "N", "alpha": ALPHA,
                   "workers": threads, "n": N_EX, "d": D},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{len(timed)} timed epochs of sync::train at B = N (+{args.warmup} "
                                   f"warm-up), EpochRecord.seconds mean, {threads} workers"},
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
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.init()
    stream = torch.cuda.current_stream()
    dev = S.Device(local, stream=stream.cuda_stream)
    SD.attach_nccl(dev)  # the engine's own communicator (no-op at N = 1)

    host = S.fixtures.sparse_classification(N_EX, D, AVG, SEED + rank).rounded_f32()
    n_global = world * N_EX
    dds = S.DeviceDataset(dev, host, row_base=rank * N_EX, n_global=n_global)
    model = S.DeviceModel(dev, D)
    task = S.Task.LR
    flush = L2Flush()

    def step(ds=dds):
        S.sync_epoch(ds, model, task, ALPHA, None, n_global, check_finite=False)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        flush()
        step()
    barrier()
    launches0 = dev.launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    with ClockSampler(local) as clocks:
        barrier()
        t_wall0 = time.perf_counter()
        for i in range(args.steps):
            flush()  # L2 flush, outside the event window
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
    value = n_global / (ms / 1e3)
    assert np.isfinite(S.device_loss(dds, model, task)), "diverged"

    # Per-kernel CUDA-event times on the launching stream (the library's profiler).
    dev.set_profiling(True)
    for _ in range(args.steps):
        flush()
        step()
    stats = dev.kernel_stats()
    dev.set_profiling(False)
    peak, peak_src = _peaks()
    nnz = dds.nnz
    # Algorithmic bytes per launch: each pass streams its copy of
    # the nonzeros (fp32 value + 16-bit id) and the head bitmap (1 bit per slot);
    # the margin pass writes n coefficients and reads n labels, the gradient
    # pass reads the n coefficients.
    idx_bytes = 2 if D <= 65536 else 4
    alg = {"k2s_margin_kernel": nnz * (4 + idx_bytes) + nnz // 8 + 2 * N_EX * 4,
           "k3s_grad_kernel": nnz * 6 + nnz // 8 + N_EX * 4}
    # K23g (the default): both passes in one launch.
    alg["k23g_step_kernel"] = alg["k2s_margin_kernel"] + alg["k3s_grad_kernel"]
    per = {k: (v[1] / max(1, v[0])) for k, v in stats.items() if k in alg}
    name = max(per, key=per.get)
    kern_ms = per[name]
    achieved = alg[name] / (kern_ms / 1e3) / 1e9
    traffic, traffic_src = _ncu_traffic(name)
    share = stats[name][1] / max(1e-9, sum(v[1] for v in stats.values()))
    sweep = dds.sweep_bytes()

    e2e = e2e_leg(S, dev, host, model, task, stream, n_global, world, args, barrier)

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference fixtures rounded to fp32; rank r uses seed + r)",
        "config": {"workload": WORKLOAD, "task": "LR", "batch": "N (all rows of all ranks)",
                   "alpha": ALPHA, "n_per_gpu": N_EX, "d": D, "nnz_per_gpu": nnz,
                   "parallelism": f"dp{world}: row shards, fp64 gradient all-reduced in-engine (NCCL)",
                   "l2": "inputs (697 MB) larger than L2, and L2 flushed before every step "
                         "(256 MiB written then read back: cold, clean L2; outside the event window)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "frac_of_nominal_8TBps": achieved / 8000.0,
                     "traffic": traffic, "traffic_source": traffic_src,
                     "kernel": name, "kernel_ms": kern_ms, "kernel_share_of_step": share,
                     "algorithmic_bytes_per_launch": alg[name], "peak_source": peak_src,
                     "kernels_ms": {k: round(v, 5) for k, v in per.items()},
                     "epoch_one_sweep_bytes": sweep,
                     "epoch_frac_of_one_sweep": sweep / (ms / 1e3) / 1e9 / peak},
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "wall_s_timed_region": t_wall1 - t_wall0,
        "step_ms_median": float(np.median(step_ms)),
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(args)
    if rank == 0 and world == 1 and not args.no_convergence:
        out["convergence"] = convergence(S, dev, dds, task, ms, out.get("cpu_baseline"))
    if not args.no_extra:
        extra = {}
        extra["c5_sync_lr_dense1000"] = extra_c5(S, dev, world, rank, args.c5_rows, barrier)
        if world == 1:
            extra["other_shapes"] = extra_shapes(S, dev)
            extra["dropin_exact_fp64_c3"] = extra_exact(S, dev, host)
        out["extra"] = extra
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def e2e_leg(S, dev, host, model, task, stream, n_global, world, args, barrier):
    """End to end through the public API with host buffers: every step copies
    the whole rcv1-shaped CSR from pinned host memory (values fp32, column ids
    as 16 bits, row offsets, labels) into a device dataset
    (sgdb_dataset_refresh_f32 / _idx16), the engine rebuilds its full-batch
    structures on the device (head bitmaps, blocked CSC by radix sort), runs
    the epoch, and the model is read back (sgdb_model_get). Double-buffered:
    step k+1's copies (two copy streams) overlap step k's rebuild + epoch."""
    import torch
    vals = torch.from_numpy(host.values.astype(np.float32)).pin_memory()
    labs = torch.from_numpy(host.labels.astype(np.float32)).pin_memory()
    idx = torch.from_numpy(host.indices.astype(np.uint16).view(np.int16)).pin_memory()
    rp = torch.from_numpy(host.row_offsets.astype(np.int32)).pin_memory()
    h2d = vals.numel() * 4 + labs.numel() * 4 + idx.numel() * 2 + rp.numel() * 4
    d2h = D * 8
    rank = _env_int("RANK", 0)
    copy_streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    copy_devs = [S.Device(dev.ordinal, stream=cs.cuda_stream) for cs in copy_streams]
    bufs = [S.DeviceDataset(dev, host, row_base=rank * N_EX, n_global=n_global) for _ in range(2)]
    ready = [[torch.cuda.Event() for _ in copy_streams] for _ in range(2)]
    free = [torch.cuda.Event(), torch.cuda.Event()]
    used = [False, False]
    steps = max(3, args.steps)

    def refresh(b):
        bufs[b].refresh_f32(vals, None, None, None, device=copy_devs[0])
        bufs[b].refresh_f32(None, labs, None, rp, device=copy_devs[1])
        bufs[b].refresh_idx16(idx, device=copy_devs[1])
        for ev, cs in zip(ready[b], copy_streams):
            ev.record(cs)

    def run():
        used[0] = used[1] = False
        refresh(0)
        for k in range(steps):
            b = k % 2
            if k + 1 < steps:
                nb = 1 - b
                if used[nb]:
                    for cs in copy_streams:
                        cs.wait_event(free[nb])
                refresh(nb)
            for e in ready[b]:
                stream.wait_event(e)
            S.sync_epoch(bufs[b], model, task, ALPHA, None, n_global, check_finite=False)
            free[b].record(stream)
            used[b] = True
            model.get()

    run()  # warm-up (pinned buffers, link state, rebuild scratch)
    barrier()
    t0 = time.perf_counter()
    run()
    barrier()
    e2e_s = (time.perf_counter() - t0) / steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    del bufs
    # The link's own rate for the same bytes, moved the way the steps move
    # them (pinned host -> device, split over two copy streams): the floor of
    # a step that must move them.
    half = (h2d // 4 + 1) // 2 + 1
    srcs = [torch.empty(half, dtype=torch.float32).pin_memory() for _ in range(2)]
    dsts = [torch.empty(half, dtype=torch.float32, device="cuda") for _ in range(2)]
    cps = [torch.cuda.Stream() for _ in range(2)]

    def copy_all():
        for src, dst, cs in zip(srcs, dsts, cps):
            with torch.cuda.stream(cs):
                dst.copy_(src, non_blocking=True)

    copy_all()
    torch.cuda.synchronize()
    link_gbps = 0.0
    for _ in range(5):  # the best of five (the link's rate, not its noise)
        t0 = time.perf_counter()
        copy_all()
        torch.cuda.synchronize()
        link_gbps = max(link_gbps, 2 * half * 4 / (time.perf_counter() - t0) / 1e9)
    del srcs, dsts
    return {"value": n_global / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3, "steps": steps,
            "h2d_link_GBps_probe": link_gbps,
            "step_vs_link_floor": (h2d / (link_gbps * 1e9)) / e2e_s,
            "pipeline": "double-buffered: step k+1's H2D (two copy streams) overlaps step k's "
                        "device rebuild of the full-batch structures + epoch; the model is read "
                        "back every step"}


def _time_sync(S, dds, model, task, alpha, batch, epochs, warmup, flush, order=None):
    import torch
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        S.sync_epoch(dds, model, task, alpha, order, batch)
    evs = []
    for _ in range(epochs):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        S.sync_epoch(dds, model, task, alpha, order, batch, check_finite=False)
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    return float(np.mean([x.elapsed_time(y) for x, y in evs]))


def _time_hogwild(S, dds, model, task, alpha, plan, epochs, warmup, flush):
    import torch
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        S.hogwild_epoch(dds, model, task, alpha, plan)
    evs = []
    for _ in range(epochs):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        S.hogwild_epoch(dds, model, task, alpha, plan)
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    return float(np.mean([x.elapsed_time(y) for x, y in evs]))


def extra_c5(S, dev, world, rank, rows_per_gpu, barrier):
    """BASELINE.json configs[4]: row-sharded synchronous LR on
    dense 1,000-d data, rows_per_gpu rows per GPU generated on the device (K9),
    full-batch epochs, fp64 gradient all-reduced by the engine's NCCL
    communicator when N > 1."""
    import torch
    import torch.distributed as dist
    d = 1000
    n_global = rows_per_gpu * world
    dds = S.DeviceDataset.generate_dense(dev, rows_per_gpu, d, 20250815, row_base=rank * rows_per_gpu,
                                         n_global=n_global)
    model = S.DeviceModel(dev, d)
    barrier()
    flush = L2Flush()
    dev.set_profiling(True)
    ms = _time_sync(S, dds, model, S.Task.LR, 1e-9, n_global, 5, 2, flush)
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
           "note": "epoch = dense_full_kernel + in-engine ncclAllReduce of g (d fp64) + apply when N > 1"}
    del dds
    torch.cuda.empty_cache()
    return out


def extra_shapes(S, dev):
    """Other BASELINE shapes on one GPU: full-batch and B = 4096 sync epochs,
    and Hogwild epochs with the paper's plans (every resident lane group a
    worker). Context for the headline, not headline numbers."""
    import torch
    flush = L2Flush()
    peak, _ = _peaks()
    shapes = {
        # name: (make, task, sync alpha (B = N), hogwild plan, hogwild alpha)
        "C1_covtype_lr": (lambda: S.fixtures.dense_classification(581012, 54, 20250810), S.Task.LR,
                          1e-5, None, None),
        "C2_w8a_svm": (lambda: S.fixtures.sparse_classification(64700, 300, 11.65, 20250811),
                       S.Task.SVM, 1e-2, "row-ch:kernel:10", 1e-2),
        "C3_rcv1_lr": (lambda: S.fixtures.sparse_classification(677399, 47236, 73.16, 20250813),
                       S.Task.LR, 1e-2, "row-ch:kernel:0", 1e-2),
        "C4a_news20_svm": (lambda: S.fixtures.sparse_classification(19996, 1355191, 455.0, 20250814),
                           S.Task.SVM, 1e-4, "row-rr:kernel:10", 1e-4),
        "C4b_realsim_svm": (lambda: S.fixtures.sparse_classification(72309, 20958, 51.3, 20250812),
                            S.Task.SVM, 1e-3, "row-rr:kernel:10", 1e-3),
    }
    out = {}
    for name, (make, task, alpha, plan_text, async_alpha) in shapes.items():
        host = make().rounded_f32()
        dds = S.DeviceDataset(dev, host)
        n = host.n_examples
        sweep = dds.sweep_bytes()
        rec = {"n": n, "d": host.n_features}
        if name != "C3_rcv1_lr":
            model = S.DeviceModel(dev, host.n_features)
            ms = _time_sync(S, dds, model, task, alpha, n, 5, 2, flush)
            rec["sync_B_N"] = {"epoch_ms": ms, "value": n / (ms / 1e3), "unit": UNIT,
                               "frac_one_sweep": sweep / (ms / 1e3) / 1e9 / peak}
        order = S.Schedule(1, n).next()
        model = S.DeviceModel(dev, host.n_features)
        ms = _time_sync(S, dds, model, task, alpha / 16, 4096, 5, 2, flush, order=order)
        rec["sync_B_4096"] = {"epoch_ms": ms, "value": n / (ms / 1e3), "unit": UNIT,
                              "us_per_step": ms * 1e3 / ((n + 4095) // 4096),
                              "frac_one_sweep": sweep / (ms / 1e3) / 1e9 / peak}
        if plan_text:
            plan = S.parse_plan(plan_text)
            plan.workers = dev.resident_workers(dds)
            hm = S.DeviceModel(dev, host.n_features)
            ams = _time_hogwild(S, dds, hm, task, async_alpha, plan, 5, 2, flush)
            rec["hogwild"] = {"plan": plan_text, "workers": plan.workers, "epoch_ms": ams,
                              "value": n / (ams / 1e3), "unit": UNIT,
                              "frac_one_sweep": sweep / (ams / 1e3) / 1e9 / peak}
        if name == "C3_rcv1_lr":  # block scope, 8 replicas in L2 (C3: "per-block model replication")
            plan = S.parse_plan("row-ch:block:0")
            plan.workers = dev.resident_workers(dds)
            plan.group_size = plan.workers // 8
            hm = S.DeviceModel(dev, host.n_features)
            ams = _time_hogwild(S, dds, hm, task, 0.03, plan, 5, 2, flush)
            rec["hogwild_block_R8"] = {"plan": "row-ch:block:0", "workers": plan.workers,
                                       "group_size": plan.group_size, "epoch_ms": ams,
                                       "value": n / (ams / 1e3), "unit": UNIT}
        out[name] = rec
        del dds, host
    return out


def extra_exact(S, dev, host):
    """The drop-in adapter's default precision (exact fp64 mode: the reference's
    operation order, bit-identical results; kernels_linalg.cu) on the headline
    configuration — what a C++ maintainer gets from INTEGRATION.md unless
    SGDB_PRECISION=fp32."""
    import torch
    dds = S.DeviceDataset(dev, host, exact=True)
    model = S.DeviceModel(dev, D)
    flush = L2Flush()
    ms = _time_sync(S, dds, model, S.Task.LR, ALPHA, N_EX, 3, 1, flush)
    out = {"epoch_ms": ms, "value": N_EX / (ms / 1e3), "unit": UNIT,
           "note": "sgdb_dataset_upload_ex(SGDB_UPLOAD_EXACT_FP64): matvec / coefficient / "
                   "matvec_transposed (256-row partials + pairwise tree) in fp64, reference order"}
    del dds
    torch.cuda.empty_cache()
    return out


def cpu_baseline(args):
    """The unmodified reference (oracle/_ref) timed on this box's host cores:
    sync::train at B = N, 1 worker (sequential) and every hardware thread, on
    the headline configuration and the other sync configurations of
    BASELINE.json (C1, C4a, C4b; C5 as a 200,000-row slice of the 1,000-d data,
    regenerated by the oracle's Philox restatement — the full 200M x 1000 is
    1.6 TB in fp64). A bounded number of epochs each."""
    import oracle
    if not oracle.reference_available():
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                "sample": "unavailable: oracle/_ref not built"}
    ref = oracle.reference()
    threads = ref.hardware_threads()
    cfgs = [
        ("C3_rcv1_lr", lambda: ref.fixture_sparse(N_EX, D, AVG, SEED), 0, 0.01, 2),
        ("C1_covtype_lr", lambda: ref.fixture_dense(581012, 54, 20250810), 0, 1e-5, 3),
        ("C4a_news20_svm", lambda: ref.fixture_sparse(19996, 1355191, 455.0, 20250814), 1, 1e-4, 2),
        ("C4b_realsim_svm", lambda: ref.fixture_sparse(72309, 20958, 51.3, 20250812), 1, 1e-3, 3),
        ("C5_slice_200k_x_1000_lr", lambda: oracle.oracle().philox_dense(200000, 1000, 20250815), 0, 1e-9, 2),
    ]
    table = {}
    t_start = time.perf_counter()
    for name, make, task, alpha, epochs in cfgs:
        ds = make()
        h = ref.to_handle(ds)
        try:
            rec = {"n": ds.n_examples, "d": ds.n_features}
            for label, workers in (("sequential", 1), ("all_threads", threads)):
                _, _, secs, _ = ref.sync_train(ds, task, alpha, ds.n_examples, epochs, 7,
                                               workers=workers, handle=h)
                mean = float(np.mean(secs))
                rec[label] = {"epoch_s": mean, "value": ds.n_examples / mean, "cores": workers,
                              "epochs": len(secs)}
            table[name] = rec
        finally:
            ref.lib.ref_ds_free(h)
        del ds
    head = table["C3_rcv1_lr"]["all_threads"]
    return {"value": head["value"], "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"sync::train at B = N on the headline data, {head['epochs']} epochs, "
                      f"{threads} workers (EpochRecord.seconds mean)",
            "sequential": table["C3_rcv1_lr"]["sequential"], "configs": table,
            "wall_s": time.perf_counter() - t_start}


def convergence(S, dev, dds, task, ms_epoch, cpu):
    """Time to 1 % of L* (harness.cpp:44-50) for the headline run: L* = min loss
    over GPU batch-GD probes (a step-size grid, harness.cpp:275-289) and the
    runs below; the reference's epochs are the same algorithm in fp64."""
    l_star = float("inf")
    runs = {}
    for a in (3e-3, 1e-2, 3e-2):
        r = S.sync.train(task, dds, S.Hyperparams(alpha=a, batch_b=dds.n_global, epochs=150,
                                                  task=task), 7)
        runs[a] = [v for v in r.trace.losses() if np.isfinite(v)]
        l_star = min([l_star] + runs[a])
    gpu_losses = runs[ALPHA]
    out = {"l_star": l_star, "alpha": ALPHA, "gpu_epochs_to_1pct": _epochs_to(gpu_losses, l_star)}
    if out["gpu_epochs_to_1pct"]:
        out["gpu_time_to_1pct_s"] = out["gpu_epochs_to_1pct"] * ms_epoch / 1e3
    try:
        import oracle
        if oracle.reference_available():
            ref = oracle.reference()
            ds = ref.fixture_sparse(N_EX, D, AVG, SEED)
            e = out["gpu_epochs_to_1pct"] or 12
            _, losses, secs, _ = ref.sync_train(ds, 0, ALPHA, N_EX, e + 1, 7,
                                                workers=ref.hardware_threads())
            ec = _epochs_to(list(losses), l_star)
            out["cpu_epochs_to_1pct"] = ec
            out["cpu_workers"] = ref.hardware_threads()
            if ec:
                out["cpu_time_to_1pct_s"] = float(np.sum(secs[:ec]))
    except Exception as exc:  # reported, not fatal
        out["cpu_error"] = str(exc)
    return out


def selftest_launch(args):
    """Launcher check without a GPU (tests/test_bench_launcher.py): every rank
    joins a gloo group and rank 0 prints the world size it saw."""
    import torch
    import torch.distributed as dist
    world = _env_int("WORLD_SIZE", 1)
    if world > 1:
        dist.init_process_group("gloo")
        t = torch.ones(1)
        dist.all_reduce(t)
        seen = int(t.item())
        dist.destroy_process_group()
    else:
        seen = 1
    if _env_int("RANK", 0) == 0:
        print(json.dumps({"n_gpus": world, "ranks_seen": seen, "selftest": True}))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-convergence", action="store_true")
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--c5-rows", type=int, default=25_000_000,
                    help="rows per GPU of the 200M x 1000 configuration (25M = 8 GPUs x 25M)")
    ap.add_argument("--selftest-launch", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args)
    if args.selftest_launch:
        return selftest_launch(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
