"""Methodology harness over the device engines: sgdbench::harness
(proj/include/sgdbench/harness.hpp, proj/src/harness.cpp) with the GPU sync,
Hogwild and dual-instance engines behind `run`.

Turns epoch throughput into the paper's third axis, time to convergence
(§6.1): `run` repeats a configuration, averages epoch times across
repetitions and reports epochs / seconds to within {10, 5, 2, 1} % of the
optimal loss; `estimate_optimal_loss` probes synchronous batch GD over the
step-size grid; `grid_search_alpha` picks the step size with the fastest time
to 1 %. The warp simulator engine (Engine::WarpSim) is out of scope: real
sm_100a kernels plus ncu replace it.
"""
from __future__ import annotations

import enum
import hashlib
import math
from dataclasses import dataclass, field, replace
from typing import Optional, Sequence

import numpy as np

from .api import (Device, DeviceDataset, ExecutionPlan, Hyperparams, LossTrace, Options, Task,
                  TrainOptions, _as_device_dataset, hogwild, plan_to_string, sync)

TOLERANCES_PERCENT = (10, 5, 2, 1)  # harness.hpp kTolerancesPercent
CSV_HEADER = ("engine,task,data,layout,plan,workers,alpha,batch,epochs,seed,repetitions,"
              "tolerance_pct,epochs_to,time_to_s,time_per_epoch_ms,final_loss,optimal_loss,diverged")


class Engine(enum.Enum):  # harness.hpp Engine (WarpSim not provided)
    Sync = "sync"
    Async = "async"
    NumaDual = "numa"


def engine_from_name(name: str) -> Optional[Engine]:
    try:
        return Engine(name)
    except ValueError:
        return None


@dataclass
class RunConfig:  # harness.hpp RunConfig
    engine: Engine = Engine.Sync
    task: Task = Task.LR
    data_path: str = ""
    hyper: Hyperparams = field(default_factory=Hyperparams)
    workers: int = 1
    plan: Optional[ExecutionPlan] = None
    repetitions: int = 3
    max_epochs: int = 1000
    wall_clock_budget_seconds: float = 60.0
    seed: int = 0
    optimal_loss: Optional[float] = None
    skip_warmup: int = 0

    def validate(self) -> None:  # harness.cpp RunConfig::validate
        if self.repetitions < 1:
            raise ValueError("repetitions must be >= 1")
        if not self.wall_clock_budget_seconds > 0.0:
            raise ValueError("budget must be > 0")
        if self.max_epochs == 0:
            raise ValueError("max_epochs must be >= 1")


@dataclass
class RunReport:  # harness.hpp RunReport
    config: RunConfig
    trace: LossTrace
    cumulative_seconds: list
    time_per_epoch_ms: float
    epochs_to: dict
    time_to_convergence_s: dict
    optimal_loss_used: float
    final_loss: float
    diverged: bool
    divergence_note: str = ""
    gradient_evals_per_epoch: list = field(default_factory=list)


def convergence_epochs(losses: Sequence[float], l_star: float, tol: float) -> Optional[int]:
    """First 1-based epoch with loss <= (1 + tol) * l_star (harness.cpp:44-50)."""
    threshold = (1.0 + tol) * l_star
    for i, loss in enumerate(losses):
        if loss <= threshold:
            return i + 1
    return None


def _fill_convergence(r: RunReport) -> None:  # harness.cpp fill_convergence
    losses = r.trace.losses()
    for tol in TOLERANCES_PERCENT:
        e = convergence_epochs(losses, r.optimal_loss_used, tol / 100.0)
        r.epochs_to[tol] = e
        r.time_to_convergence_s[tol] = (r.cumulative_seconds[e - 1]
                                        if e is not None and e <= len(r.cumulative_seconds) else None)


def _run_engine_once(config: RunConfig, ds, device: Optional[Device]):
    hyper = replace(config.hyper, epochs=min(config.hyper.epochs, config.max_epochs))
    if config.engine == Engine.Sync:
        o = TrainOptions(workers=config.workers, max_seconds=config.wall_clock_budget_seconds)
        r = sync.train(config.task, ds, hyper, config.seed, o, device=device)
        return r.trace, []
    plan = config.plan
    if plan is None:
        plan = ExecutionPlan()
        plan.workers = config.workers
    o = Options(max_seconds=config.wall_clock_budget_seconds)
    fn = hogwild.train if config.engine == Engine.Async else hogwild.numa_dual_train
    r = fn(config.task, ds, hyper, plan, config.seed, o, device=device)
    return r.trace, list(r.evals_per_epoch)


def run(config: RunConfig, ds, device: Optional[Device] = None) -> RunReport:
    """harness.cpp run(): repetitions share the seed, so deterministic engines
    stay on one trajectory; losses come from the first repetition, epoch times
    are averaged across repetitions."""
    config.validate()
    ds = _as_device_dataset(ds, device)
    traces, evals = [], []
    for rep in range(config.repetitions):
        t, ev = _run_engine_once(config, ds, device)
        if rep == 0:
            evals = ev
        traces.append(t)
    first = traces[0]
    epochs = []
    for i, rec in enumerate(first.epochs):
        secs = [t.epochs[i].seconds for t in traces if i < len(t.epochs)]
        epochs.append(replace(rec, seconds=float(np.mean(secs)) if secs else 0.0))
    trace = LossTrace(epochs, first.diverged, first.divergence_note)
    cumulative = list(np.cumsum([e.seconds for e in epochs])) if epochs else []
    timed = [e.seconds for e in epochs[config.skip_warmup:]]
    diverged = any(t.diverged for t in traces)
    note = next((t.divergence_note for t in traces if t.diverged), "")
    report = RunReport(config=config, trace=trace, cumulative_seconds=[float(c) for c in cumulative],
                       time_per_epoch_ms=float(np.mean(timed)) * 1e3 if timed else 0.0,
                       epochs_to={}, time_to_convergence_s={},
                       optimal_loss_used=(config.optimal_loss if config.optimal_loss is not None
                                          else trace.min_loss()),
                       final_loss=trace.final_loss(), diverged=diverged, divergence_note=note,
                       gradient_evals_per_epoch=evals)
    _fill_convergence(report)
    return report


def default_alpha_grid() -> list[float]:  # {1e-6, ..., 1e2} by decades
    return [10.0 ** p for p in range(-6, 3)]


_OPTIMAL_LOSS_CACHE: dict = {}


def _fingerprint(ds) -> str:
    if isinstance(ds, DeviceDataset):
        if ds.host is None:
            raise ValueError("estimate_optimal_loss: device dataset without its host copy")
        ds = ds.host
    h = hashlib.sha1()
    h.update(np.asarray([ds.n_examples, ds.n_features, ds.values.size], np.int64).tobytes())
    step = max(1, ds.values.size // 512)
    h.update(np.ascontiguousarray(ds.values[::step]).tobytes())
    h.update(np.ascontiguousarray(ds.labels[::max(1, ds.labels.size // 128)]).tobytes())
    return h.hexdigest()


def _n_examples(ds) -> int:
    return ds.n_global if isinstance(ds, DeviceDataset) else ds.n_examples


def clear_optimal_loss_cache() -> None:
    _OPTIMAL_LOSS_CACHE.clear()


def estimate_optimal_loss(task: Task, ds, probes: Optional[Sequence[RunConfig]] = None,
                          budget_seconds_per_config: float = 60.0, max_epochs: int = 100000,
                          device: Optional[Device] = None) -> float:
    """Lowest finite loss across the probes (default: synchronous batch GD over
    the step-size grid), cached per (task, dataset content) — harness.cpp:250-289."""
    key = (int(task), _fingerprint(ds))
    if key in _OPTIMAL_LOSS_CACHE:
        return _OPTIMAL_LOSS_CACHE[key]
    if probes is None:
        probes = [RunConfig(engine=Engine.Sync, task=task,
                            hyper=Hyperparams(alpha=a, batch_b=_n_examples(ds), epochs=max_epochs,
                                              task=task),
                            max_epochs=max_epochs) for a in default_alpha_grid()]
    if not probes:
        raise ValueError("estimate_optimal_loss: no probes")
    ds = _as_device_dataset(ds, device)  # upload once for every probe
    best = math.inf
    for p in probes:
        p = replace(p, task=task, hyper=replace(p.hyper, task=task), repetitions=1,
                    wall_clock_budget_seconds=budget_seconds_per_config)
        r = run(p, ds, device)
        finite = [x for x in r.trace.losses() if math.isfinite(x)]
        if finite:
            best = min(best, min(finite))
    _OPTIMAL_LOSS_CACHE[key] = best
    return best


@dataclass
class AlphaRun:
    alpha: float
    losses: list
    cumulative_seconds: list
    diverged: bool = False


def select_best_alpha(runs: Sequence[AlphaRun], l_star: Optional[float], tol: float) -> tuple[int, bool]:
    """harness.cpp select_best_alpha: fastest time to the threshold (ties to
    the smaller step); if nothing converges, the lowest finite final loss."""
    if not runs:
        raise ValueError("select_best_alpha: no runs")
    target = l_star if l_star is not None else min(
        (x for r in runs for x in r.losses if math.isfinite(x)), default=math.inf)
    best, best_time = None, math.inf
    for i, r in enumerate(runs):
        e = convergence_epochs(r.losses, target, tol)
        if e is None or e > len(r.cumulative_seconds):
            continue
        t = r.cumulative_seconds[e - 1]
        if t < best_time:
            best, best_time = i, t
    if best is not None:
        return best, True
    best, best_loss = 0, math.inf
    for i, r in enumerate(runs):
        fl = r.losses[-1] if r.losses else math.inf
        if math.isfinite(fl) and fl < best_loss:
            best, best_loss = i, fl
    return best, False


@dataclass
class GridSearchResult:
    best_alpha: float
    converged: bool
    optimal_loss_used: float
    reports: list


def grid_search_alpha(config: RunConfig, ds, grid: Optional[Sequence[float]] = None,
                      device: Optional[Device] = None) -> GridSearchResult:
    """harness.cpp grid_search_alpha: one run per step size (ascending), the
    thresholds recomputed against the shared optimum."""
    grid = sorted(grid if grid is not None else default_alpha_grid())
    if not grid:
        raise ValueError("grid_search_alpha: empty grid")
    ds = _as_device_dataset(ds, device)
    reports, runs = [], []
    for a in grid:
        r = run(replace(config, hyper=replace(config.hyper, alpha=a)), ds, device)
        reports.append(r)
        runs.append(AlphaRun(a, r.trace.losses(), r.cumulative_seconds, r.diverged))
    l_star = config.optimal_loss
    if l_star is None:
        l_star = min((x for r in runs for x in r.losses if math.isfinite(x)), default=math.inf)
    for r in reports:
        r.optimal_loss_used = l_star
        _fill_convergence(r)
    best, converged = select_best_alpha(runs, l_star, 0.01)
    return GridSearchResult(runs[best].alpha, converged, l_star, reports)


def _fmt(v: float) -> str:
    if v is None:
        return "dnc"
    if math.isnan(v):
        return "nan"
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    return "%.17g" % v


def export_csv(reports: Sequence[RunReport]) -> str:
    """harness.cpp export_csv: one row per (report, tolerance)."""
    lines = [CSV_HEADER]
    for r in reports:
        c = r.config
        plan = plan_to_string(c.plan) if c.plan is not None else ""
        for tol in TOLERANCES_PERCENT:
            e = r.epochs_to.get(tol)
            t = r.time_to_convergence_s.get(tol)
            lines.append(",".join([
                c.engine.value, "lr" if c.task == Task.LR else "svm", c.data_path, "", plan,
                str(c.workers), _fmt(c.hyper.alpha), str(c.hyper.batch_b), str(len(r.trace.epochs)),
                str(c.seed), str(c.repetitions), str(tol), str(e) if e is not None else "dnc",
                _fmt(t) if t is not None else "dnc", _fmt(r.time_per_epoch_ms), _fmt(r.final_loss),
                _fmt(r.optimal_loss_used), "1" if r.diverged else "0"]))
    return "\n".join(lines) + "\n"
