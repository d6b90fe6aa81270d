"""Time to within {10, 5, 2, 1} % of the optimal loss on the BASELINE shapes
(§6.1 methodology), through the harness mirror over the
device engines: L* from GPU batch-GD probes over the step-size grid, then each
engine / plan at its step size with epoch times averaged over repetitions.
Synchronous step sizes are searched below the 2/L stability bound of the
data (L = lambda_max(X^T X) / 4 for LR, lambda_max(X^T X) for the SVM's
subgradient, scaled by B/N for mini-batches), so the harness's
fastest-to-threshold rule cannot pick a step that touches the threshold and
then diverges.
For the small shapes the unmodified reference (oracle/_ref) is timed the same
way on the host cores, 1 worker and all hardware threads.

    python scripts/time_to_1pct.py [w8a realsim rcv1 news20 covtype]  > profiles/...csv
"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_08800_b200 as S  # noqa: E402
from paper_1802_08800_b200 import harness as H  # noqa: E402

SHAPES = {
    # name: (generator, task, [(engine, plan, alpha, batch, epochs)], cpu_reference)
    "w8a": (lambda: S.fixtures.sparse_classification(64700, 300, 11.65, 20250811), S.Task.SVM,
            [(H.Engine.Async, "row-ch:kernel:0", None, 1, 30)], True),
    "realsim": (lambda: S.fixtures.sparse_classification(72309, 20958, 51.3, 20250812), S.Task.SVM,
                [(H.Engine.Sync, None, None, "N", 300), (H.Engine.Async, "row-ch:kernel:0", None, 1, 30)],
                True),
    "rcv1": (lambda: S.fixtures.sparse_classification(677399, 47236, 73.16, 20250813), S.Task.LR,
             [(H.Engine.Sync, None, None, "N", 100), (H.Engine.Sync, None, None, 4096, 20),
              (H.Engine.Async, "row-ch:kernel:0", None, 1, 30),
              (H.Engine.Async, "row-ch:block:0@8", None, 1, 30)], False),
    "news20": (lambda: S.fixtures.sparse_classification(19996, 1355191, 455.0, 20250814), S.Task.SVM,
               [(H.Engine.Sync, None, None, "N", 100), (H.Engine.Async, "row-ch:kernel:0", None, 1, 30)],
               False),
    "covtype": (lambda: S.fixtures.dense_classification(581012, 54, 20250810), S.Task.LR,
                [(H.Engine.Sync, None, None, "N", 100), (H.Engine.Sync, None, None, 4096, 20)], False),
}


def lambda_max(ds, iters=30):
    """Largest eigenvalue of X^T X by power iteration on the host."""
    import numpy as np
    import scipy.sparse as sp
    if ds.layout == S.Layout.Csr:
        x = sp.csr_matrix((ds.values, ds.indices.astype(np.int64), ds.row_offsets.astype(np.int64)),
                          shape=(ds.n_examples, ds.n_features))
    else:
        x = np.asarray(ds.values).reshape(ds.n_examples, ds.n_features)
    v = np.random.default_rng(0).normal(size=ds.n_features)
    lam = 0.0
    for _ in range(iters):
        u = x.T @ (x @ v)
        lam = float(np.linalg.norm(u))
        v = u / lam
    return lam


def alpha_cap(ds, task, b):
    lam = lambda_max(ds) * (b / ds.n_examples)
    curv = lam / 4.0 if task == S.Task.LR else lam
    return 2.0 / curv


def main():
    dev = S.Device(0)
    reports, summary = [], []
    for name in sys.argv[1:] or list(SHAPES):
        make, task, runs, cpu = SHAPES[name]
        ds = make()
        dds = S.DeviceDataset(dev, ds)
        H.clear_optimal_loss_cache()
        l_star = H.estimate_optimal_loss(task, ds, budget_seconds_per_config=3.0, max_epochs=300,
                                         device=dev)
        for engine, plan_text, alpha, batch, epochs in runs:
            b = ds.n_examples if batch == "N" else batch
            cfg = H.RunConfig(engine=engine, task=task, data_path=name, repetitions=3,
                              hyper=S.Hyperparams(alpha=alpha or 1.0, batch_b=b, epochs=epochs, task=task),
                              optimal_loss=l_star)
            if plan_text:
                text, _, reps = plan_text.partition("@")
                cfg.plan = S.parse_plan(text)
                cfg.plan.workers = dev.resident_workers(dds)
                if reps:  # block scope with R replicas (K6g)
                    cfg.plan.group_size = max(1, cfg.plan.workers // int(reps))
            if alpha is None:  # the fastest step size of the grid (harness grid search)
                if engine == H.Engine.Sync:
                    cap = alpha_cap(ds, task, b)
                    grid = [a for a in (c * 10.0 ** p for p in range(-8, 1) for c in (1.0, 3.0))
                            if a < cap]
                else:
                    grid = [c * 10.0 ** p for p in range(-5, 0) for c in (1.0, 3.0)]
                res = H.grid_search_alpha(cfg, dds, grid, device=dev)
                cfg.hyper.alpha = res.best_alpha
            r = H.run(cfg, dds, dev)
            reports.append(r)
            summary.append({"data": name, "engine": engine.value, "plan": plan_text, "batch": b,
                            "alpha_cap_2_over_L": alpha_cap(ds, task, b) if engine == H.Engine.Sync else None,
                            "alpha": cfg.hyper.alpha, "l_star": l_star,
                            "epoch_ms": r.time_per_epoch_ms,
                            "epochs_to": {str(k): v for k, v in r.epochs_to.items()},
                            "time_to_s": {str(k): v for k, v in r.time_to_convergence_s.items()},
                            "impl": "b200"})
        if cpu:
            import oracle
            if oracle.reference_available():
                ref = oracle.reference()
                for engine, plan_text, alpha, batch, epochs in runs:
                    if engine != H.Engine.Async:
                        continue
                    for workers in (1, ref.hardware_threads()):
                        alpha = next(x["alpha"] for x in summary
                                     if x["data"] == name and x["plan"] == plan_text)
                        _, losses, secs, _ = ref.hogwild_train(ds, int(task), alpha, epochs, plan_text.split("@")[0],
                                                               workers=workers)
                        cum = list(__import__("itertools").accumulate(secs))
                        e1 = H.convergence_epochs(list(losses), l_star, 0.01)
                        summary.append({"data": name, "engine": "async", "plan": plan_text,
                                        "alpha": alpha, "l_star": l_star, "impl": "reference",
                                        "workers": workers, "epoch_ms": 1e3 * sum(secs) / len(secs),
                                        "epochs_to_1pct": e1,
                                        "time_to_1pct_s": cum[e1 - 1] if e1 else None})
        del dds
    with open(os.environ.get("TTC_OUT", "profiles/round2_time_to_1pct.jsonl"), "w") as f:
        for s in summary:
            f.write(json.dumps(s) + "\n")
    sys.stdout.write(H.export_csv(reports))


if __name__ == "__main__":
    main()
