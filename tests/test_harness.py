"""The methodology harness mirror (paper_1802_08800_b200/harness.py) against
sgdbench::harness semantics (proj/src/harness.cpp): convergence epochs, the
step-size selection rule, CSV export, config validation — host logic, no GPU —
and, on a GPU, run / estimate_optimal_loss / grid_search_alpha over the
device engines."""
import math

import numpy as np
import pytest


def test_convergence_epochs(sgdb):
    H = sgdb.harness
    assert H.convergence_epochs([5.0, 3.0, 2.02, 2.0], 2.0, 0.01) == 3
    assert H.convergence_epochs([5.0, 3.0], 2.0, 0.01) is None
    assert H.convergence_epochs([], 1.0, 0.1) is None


def test_select_best_alpha_rule(sgdb):
    H = sgdb.harness
    runs = [H.AlphaRun(0.1, [3.0, 1.5, 1.01], [1.0, 2.0, 3.0]),
            H.AlphaRun(1.0, [2.0, 1.0], [1.5, 3.0]),
            H.AlphaRun(10.0, [math.inf], [0.1], True)]
    # l* = 1.0: run 0 reaches 1.01 at t=3.0, run 1 reaches 1.0 at t=3.0 -> tie keeps the smaller alpha
    assert H.select_best_alpha(runs, None, 0.01) == (0, True)
    # nothing within 0.1 %: lowest finite final loss wins, flagged non-converged
    runs2 = [H.AlphaRun(0.1, [3.0, 2.0], [1.0, 2.0]), H.AlphaRun(1.0, [2.5, 1.8], [1.0, 2.0])]
    assert H.select_best_alpha(runs2, 1.0, 0.001) == (1, False)
    with pytest.raises(ValueError):
        H.select_best_alpha([], None, 0.01)


def test_default_grid_and_validation(sgdb):
    H = sgdb.harness
    g = H.default_alpha_grid()
    assert len(g) == 9 and g[0] == pytest.approx(1e-6) and g[-1] == pytest.approx(100.0)
    with pytest.raises(ValueError):
        H.RunConfig(repetitions=0).validate()
    with pytest.raises(ValueError):
        H.RunConfig(max_epochs=0).validate()
    assert H.engine_from_name("numa") == H.Engine.NumaDual and H.engine_from_name("warpsim") is None


def test_export_csv_header_and_rows(sgdb):
    S, H = sgdb, sgdb.harness
    trace = S.LossTrace([S.EpochRecord(1, 2.0, 0.5), S.EpochRecord(2, 1.0, 0.5)])
    r = H.RunReport(config=H.RunConfig(), trace=trace, cumulative_seconds=[0.5, 1.0],
                    time_per_epoch_ms=500.0, epochs_to={}, time_to_convergence_s={},
                    optimal_loss_used=1.0, final_loss=1.0, diverged=False)
    H._fill_convergence(r)
    lines = H.export_csv([r]).splitlines()
    assert lines[0] == H.CSV_HEADER
    assert len(lines) == 1 + len(H.TOLERANCES_PERCENT)
    assert lines[-1].split(",")[11:14] == ["1", "2", "1"]


@pytest.mark.gpu
def test_run_and_grid_search_on_device(sgdb, dev):
    S, H = sgdb, sgdb.harness
    ds = S.fixtures.sparse_classification(4000, 300, 12.0, 5).rounded_f32()
    H.clear_optimal_loss_cache()
    l_star = H.estimate_optimal_loss(S.Task.SVM, ds, budget_seconds_per_config=5.0, max_epochs=200,
                                     device=dev)
    assert math.isfinite(l_star)
    plan = S.parse_plan("row-ch:kernel:0")
    plan.workers = 64
    cfg = H.RunConfig(engine=H.Engine.Async, task=S.Task.SVM, plan=plan, repetitions=2,
                      hyper=S.Hyperparams(alpha=0.05, batch_b=1, epochs=20, task=S.Task.SVM),
                      optimal_loss=l_star)
    r = H.run(cfg, ds, dev)
    assert len(r.trace.epochs) == 20 and len(r.cumulative_seconds) == 20
    assert all(b >= a for a, b in zip(r.cumulative_seconds, r.cumulative_seconds[1:]))
    assert r.gradient_evals_per_epoch[0] == ds.n_examples
    if r.epochs_to[10] is not None:
        assert r.time_to_convergence_s[10] == pytest.approx(r.cumulative_seconds[r.epochs_to[10] - 1])
    res = H.grid_search_alpha(H.RunConfig(engine=H.Engine.Sync, task=S.Task.SVM, repetitions=1,
                                          hyper=S.Hyperparams(alpha=1.0, batch_b=ds.n_examples,
                                                              epochs=30, task=S.Task.SVM)),
                              ds, [1e-3, 1e-2, 1e-1], device=dev)
    assert res.best_alpha in (1e-3, 1e-2, 1e-1) and len(res.reports) == 3
    assert all(rep.optimal_loss_used == res.optimal_loss_used for rep in res.reports)
