"""paper_1802_08800_b200.harness (the mirror of sgdbench::harness over the
device engines) against the reference harness itself (proj/src/harness.cpp,
run through oracle/_ref) on the same data: run() (per-epoch losses and the
epochs to 10/5/2/1 % of the loss used), estimate_optimal_loss() over the
default probes' step-size grid, and grid_search_alpha()'s selection
(harness.cpp:75-124, :250-289, :343-384).

The device engines compute in fp32 against the reference's fp64 on the same
fp32-rounded data, so losses agree to the sync tolerance (rel 1e-6, DESIGN.md
§Numerics) and the convergence epochs and the selected step size are equal.
"""
import math

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu

SYNC, ASYNC = 0, 1


@pytest.fixture(scope="module")
def data(sgdb):
    S = sgdb
    return {"sparse": S.fixtures.sparse_classification(3000, 300, 15.0, 5).rounded_f32(),
            "dense": S.fixtures.dense_classification(2000, 24, 6).rounded_f32()}


@pytest.mark.parametrize("name,task,alpha,batch,epochs", [
    ("sparse", 0, 0.01, "N", 25), ("sparse", 1, 0.002, 64, 8), ("dense", 0, 1e-3, 128, 10),
    ("dense", 1, 2e-4, "N", 30)])
def test_run_matches_reference_harness(sgdb, dev, ref, data, name, task, alpha, batch, epochs):
    S = sgdb
    from paper_1802_08800_b200 import harness as H
    ds = data[name]
    b = ds.n_examples if batch == "N" else batch
    l_star = min(ref.harness_run(ds, SYNC, task, alpha, b, 3 * epochs)[0])  # shared L*
    ol, oet, olu = ref.harness_run(ds, SYNC, task, alpha, b, epochs, seed=3, optimal_loss=l_star)
    cfg = H.RunConfig(engine=H.Engine.Sync, task=S.Task(task),
                      hyper=S.Hyperparams(alpha=alpha, batch_b=b, epochs=epochs, task=S.Task(task)),
                      repetitions=1, seed=3, optimal_loss=l_star)
    r = H.run(cfg, ds, dev)
    gl = r.trace.losses()
    assert len(gl) == len(ol) == epochs
    assert max(rel(g, o) for g, o in zip(gl, ol)) <= 1e-6
    assert r.optimal_loss_used == olu
    assert {t: r.epochs_to[t] for t in (10, 5, 2, 1)} == oet


def test_estimate_optimal_loss_matches_reference_harness(sgdb, dev, ref, data):
    S = sgdb
    from paper_1802_08800_b200 import harness as H
    ds = data["sparse"]
    H.clear_optimal_loss_cache()
    g = H.estimate_optimal_loss(S.Task.LR, ds, max_epochs=200, device=dev)
    o = ref.estimate_optimal_loss(ds, 0, 200)
    assert math.isfinite(g) and rel(g, o) <= 1e-6


@pytest.mark.parametrize("name,task", [("sparse", 0), ("dense", 1)])
def test_grid_search_selects_the_reference_step(sgdb, dev, ref, data, name, task):
    """Per grid point the epochs to 1 % equal the reference's; the selection
    (fastest wall-clock time to 1 %, so among the fewest-epoch step sizes) is
    one of the reference's fewest-epoch step sizes, and both agree on
    convergence."""
    S = sgdb
    from paper_1802_08800_b200 import harness as H
    ds = data[name]
    grid = [1e-5, 1e-4, 1e-3, 1e-2]
    b = ds.n_examples
    l_star = min(min(ref.harness_run(ds, SYNC, task, a, b, 120)[0]) for a in grid[:3])
    ref_epochs = {a: ref.harness_run(ds, SYNC, task, a, b, 40, optimal_loss=l_star)[1][1] for a in grid}
    o_best, o_conv, _ = ref.grid_search_alpha(ds, SYNC, task, b, 40, grid, optimal_loss=l_star)
    cfg = H.RunConfig(engine=H.Engine.Sync, task=S.Task(task),
                      hyper=S.Hyperparams(alpha=grid[0], batch_b=b, epochs=40, task=S.Task(task)),
                      repetitions=1, optimal_loss=l_star)
    res = H.grid_search_alpha(cfg, ds, grid, device=dev)
    ours = {r.config.hyper.alpha: r.epochs_to[1] for r in res.reports}
    assert ours == ref_epochs
    reached = [e for e in ref_epochs.values() if e is not None]
    fastest = {a for a, e in ref_epochs.items() if reached and e == min(reached)}
    assert res.converged == o_conv == bool(reached)
    if reached:
        assert res.best_alpha in fastest and o_best in fastest
    else:
        assert res.best_alpha == o_best
