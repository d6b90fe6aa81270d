"""Device results against the committed golden vectors of the unmodified
reference (tests/golden/reference_golden.npz) — runs on the GPU box where
/root/reference does not exist. Tolerances as in test_gpu_sync.py /
test_gpu_hogwild.py."""
import os

import numpy as np
import pytest

from conftest import rel, rel_l2

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz"))


def ds_from_gold(S, prefix):
    n, d, layout, pw = (int(x) for x in GOLD[f"{prefix}_shape"])
    return S.Dataset(n, d, S.Layout(layout), GOLD[f"{prefix}_labels"], GOLD[f"{prefix}_values"],
                     GOLD[f"{prefix}_indices"], GOLD[f"{prefix}_row_offsets"], pw).rounded_f32()


@pytest.mark.parametrize("key", [str(k) for k in GOLD["sync_runs"]])
def test_sync_against_golden(sgdb, dev, key):
    S = sgdb
    _, name, t, b = key.split("_")
    ds = ds_from_gold(S, name)
    task, b = S.Task(int(t[1:])), int(b[1:])
    dds = S.DeviceDataset(dev, ds)
    model = S.DeviceModel(dev, ds.n_features)
    sched = S.Schedule(17, ds.n_examples)
    for e in range(5):
        order = sched.next()
        assert S.sync_epoch(dds, model, task, 1.0 / b, order if b < ds.n_examples else None, b)
        assert rel_l2(model.get(), GOLD[key + "_models"][e]) <= 1e-5
        assert rel(S.device_loss(dds, model, task), GOLD[key + "_losses"][e]) <= 1e-6


@pytest.mark.parametrize("entry", [str(k) for k in GOLD["hog_runs"]])
def test_one_worker_hogwild_against_golden(sgdb, dev, entry):
    S = sgdb
    key, name, plan_text, task = entry.split("|")
    ds = ds_from_gold(S, name)
    plan = S.parse_plan(plan_text)
    plan.workers = 1
    hp = S.Hyperparams(alpha=0.05, batch_b=1, epochs=3, task=S.Task(int(task)))
    r = S.hogwild.train(S.Task(int(task)), ds, hp, plan, 0, device=dev)
    assert rel_l2(r.model, GOLD[key + "_model"]) <= 1e-4
    for e in range(3):
        assert rel(r.trace.epochs[e].loss, GOLD[key + "_losses"][e]) <= 1e-5
    assert r.evals_per_epoch == [int(x) for x in GOLD[key + "_evals"]]


def test_primitives_against_golden(sgdb, dev):
    S = sgdb
    ds = ds_from_gold(S, "sparse")
    w = GOLD["prim_w"]
    for task in (0, 1):
        assert rel(S.dataset_loss(S.Task(task), ds, w, device=dev), GOLD[f"prim_loss_t{task}"][0]) <= 1e-12
        g = S.sync.batch_gradient(S.Task(task), ds, None, w, device=dev)
        assert rel_l2(g, GOLD[f"prim_grad_t{task}"]) <= 1e-6
        g = S.sync.batch_gradient(S.Task(task), ds, np.arange(0, 400, 3), w, device=dev)
        assert rel_l2(g, GOLD[f"prim_grad_rows_t{task}"]) <= 1e-6
