"""Pins the CPU oracle (oracle/glm_oracle.cpp) to the reference.

* against the committed golden vectors (tests/golden/reference_golden.npz,
  generated from the unmodified reference by tests/golden/make_golden.py):
  bit-exact;
* against the live reference (oracle/_ref, when built here): bit-exact on
  fresh seeds, including the reference tests' known answers.
"""
import os

import numpy as np
import pytest

import oracle

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz"))


def ds_from_gold(prefix):
    n, d, layout, pw = (int(x) for x in GOLD[f"{prefix}_shape"])
    return oracle.HostData(n, d, layout, GOLD[f"{prefix}_labels"], GOLD[f"{prefix}_values"],
                           GOLD[f"{prefix}_indices"], GOLD[f"{prefix}_row_offsets"], pw)


@pytest.fixture(scope="module")
def O():
    return oracle.oracle()


def test_fixtures_bit_exact(O):
    a = O.fixture_dense(300, 12, 20250810)
    assert np.array_equal(a.values, GOLD["dense_values"]) and np.array_equal(a.labels, GOLD["dense_labels"])
    b = O.fixture_sparse(400, 60, 6.0, 20250811)
    for f in ("values", "indices", "row_offsets", "labels"):
        assert np.array_equal(getattr(b, f), GOLD[f"sparse_{f}"]), f


@pytest.mark.parametrize("target,name", [(oracle.PADDED, "padded"), (oracle.DENSE_COL, "dcol")])
def test_layout_conversion_bit_exact(O, target, name):
    src = ds_from_gold("sparse" if name == "padded" else "dense")
    out = O.convert_layout(src, target)
    for f in ("values", "indices", "labels"):
        assert np.array_equal(getattr(out, f), GOLD[f"{name}_{f}"]), f
    assert out.padded_width == int(GOLD[f"{name}_shape"][3])


@pytest.mark.parametrize("key", [str(k) for k in GOLD["sync_runs"]])
def test_sync_train_bit_exact(O, key):
    _, name, t, b = key.split("_")
    ds = O.round_f32(ds_from_gold(name))
    task, b = int(t[1:]), int(b[1:])
    models, losses, div = O.sync_train(ds, task, 1.0 / b, b, 5, 17)
    assert not div
    assert np.array_equal(models, GOLD[key + "_models"])
    assert np.array_equal(losses, GOLD[key + "_losses"])


RR = {"rowrr": 1, "rowch": 0, "colrr": 1, "colch": 0}
REPL = {"kernel": 0, "block": 1, "thread": 2}


@pytest.mark.parametrize("entry", [str(k) for k in GOLD["hog_runs"]])
def test_one_worker_hogwild_bit_exact(O, entry):
    key, name, plan, task = entry.split("|")
    access, repl, k = plan.split(":")
    ds = O.round_f32(ds_from_gold(name))
    models, losses, evals = O.hogwild_serial(ds, int(task), 0.05, 3, RR[access.replace("-", "")],
                                             REPL[repl], int(k), 1)
    assert np.array_equal(models[-1], GOLD[key + "_model"])
    assert np.array_equal(losses, GOLD[key + "_losses"])
    assert np.array_equal(evals, GOLD[key + "_evals"])


def test_primitives_bit_exact(O):
    ds = O.round_f32(ds_from_gold("sparse"))
    w = GOLD["prim_w"]
    for task in (0, 1):
        assert O.dataset_loss(ds, task, w) == GOLD[f"prim_loss_t{task}"][0]
        assert np.array_equal(O.batch_gradient(ds, task, None, w), GOLD[f"prim_grad_t{task}"])
        assert np.array_equal(O.batch_gradient(ds, task, np.arange(0, 400, 3), w),
                              GOLD[f"prim_grad_rows_t{task}"])


def test_scalar_cores_bit_exact(O):
    for task in (0, 1):
        for y in (1, -1):
            c = [O.fn("point_coefficient")(task, z, float(y)) for z in GOLD["core_z"]]
            l = [O.fn("point_loss_from_margin")(task, z, float(y)) for z in GOLD["core_z"]]
            assert np.array_equal(c, GOLD[f"core_coef_t{task}_y{y}"])
            assert np.array_equal(l, GOLD[f"core_loss_t{task}_y{y}"])


def test_scalar_core_known_answers(O):
    """test_glm.cpp:34-88: log 2 and 1 at w=0, log1p(e^-100) at margin 100, the SVM kink."""
    f = O.fn("point_loss_from_margin")
    g = O.fn("point_coefficient")
    assert f(0, 0.0, 1.0) == np.log(2.0)
    assert f(1, 0.0, 1.0) == 1.0
    assert f(0, 100.0, 1.0) == np.log1p(np.exp(-100.0))
    assert f(0, -1e4, 1.0) == 1e4
    assert g(1, 1.0, 1.0) == 0.0  # zero subgradient at the margin itself
    assert g(0, 0.0, 1.0) == -0.5


@pytest.mark.parametrize("i", range(9))
def test_parser_matches_golden(O, i):
    text = str(GOLD["parse_cases"][i])
    ds, err = O.parse_libsvm(text)
    if f"parse_{i}_error_line" in GOLD:
        assert err is not None and err[1] == int(GOLD[f"parse_{i}_error_line"][0])
    else:
        assert err is None
        for f in ("values", "indices", "row_offsets", "labels"):
            assert np.array_equal(getattr(ds, f), GOLD[f"parse_{i}_{f}"]), f
        assert ds.n_features == int(GOLD[f"parse_{i}_shape"][1])


def test_assign_matches_golden(O):
    for case in GOLD["assign_cases"]:
        n, wk, rr, k = (int(x) for x in str(case).split(","))
        lists = O.assign(n, wk, rr, k)
        flat = np.array([x for l in lists for x in l], np.uint32)
        assert np.array_equal(flat, GOLD[f"assign_{n}_{wk}_{rr}_{k}_ids"])


def test_schedule_matches_golden(O):
    assert np.array_equal(O.schedule(7, 50, 3), GOLD["schedule_7_50"])


def test_merge_models_matches_golden(O):
    reps = GOLD["merge_reps"]
    assert np.array_equal(O.merge_models(reps), GOLD["merge_mean"])
    assert np.array_equal(O.merge_models(reps, np.array([3.0, 1.0, 0.5, 2.0, 0.25])),
                          GOLD["merge_weighted"])


# ---- live reference (built in this container; travels as oracle/_ref) ----------------

@pytest.mark.parametrize("seed", [1, 2, 3])
def test_live_reference_sync_and_hogwild(O, ref, seed):
    rng = np.random.default_rng(seed)
    ds = O.fixture_sparse(int(rng.integers(50, 500)), int(rng.integers(5, 200)), 5.0, seed)
    dense = O.fixture_dense(int(rng.integers(50, 300)), int(rng.integers(1, 40)), seed)
    for d in (ds, dense):
        for task in (0, 1):
            b = int(rng.integers(1, d.n_examples + 1))
            m, l, _ = O.sync_train(d, task, 0.05, b, 3, seed)
            rm, rl, _, _ = ref.sync_train(d, task, 0.05, b, 3, seed)
            assert np.array_equal(m[-1], rm) and np.array_equal(l, rl)
            hm, hl, he = O.hogwild_serial(d, task, 0.05, 2, 1, 1, 3, 1)
            rhm, rhl, _, rhe = ref.hogwild_train(d, task, 0.05, 2, "row-rr:block:3", workers=1)
            assert np.array_equal(hm[-1], rhm) and np.array_equal(hl, rhl)
            assert np.array_equal(he, rhe)


def test_live_reference_dual_and_thread(O, ref):
    """thread scope with 3 workers and the dual-instance merge are deterministic
    in the reference (replicas never interact within an epoch)."""
    ds = O.fixture_sparse(51, 14, 3.0, 8)
    m, l, _ = O.hogwild_serial(ds, 0, 0.07, 3, 0, 2, 0, 3)
    rm, rl, _, _ = ref.hogwild_train(ds, 0, 0.07, 3, "row-ch:thread:0", workers=3)
    assert np.array_equal(m[-1], rm) and np.array_equal(l, rl)
    dm, dl, _, de = ref.hogwild_train(ds, 0, 0.08, 4, "row-ch:kernel:0", workers=1, dual=True)
    sm, sl, _ = O.hogwild_serial(ds, 0, 0.08, 4, 0, 0, 0, 1)
    assert np.array_equal(dm, sm[-1]) and np.array_equal(dl, sl)
    assert int(de[0]) == 2 * ds.n_examples


def test_live_reference_linalg(O, ref):
    """The linalg:: wrappers the operator-API GPU tests compare against: the
    reference is bit-identical for any worker count and agrees with numpy."""
    ds = O.fixture_sparse(256 * 5 + 9, 300, 10.0, 77)
    dense = np.zeros((ds.n_examples, ds.n_features))
    for i in range(ds.n_examples):
        lo, hi = int(ds.row_offsets[i]), int(ds.row_offsets[i + 1])
        dense[i, ds.indices[lo:hi]] = ds.values[lo:hi]
    rng = np.random.default_rng(0)
    a = rng.standard_normal(ds.n_examples)
    v = rng.standard_normal(ds.n_features)
    t1 = ref.matvec_transposed(ds, a, workers=1)
    assert np.array_equal(t1, ref.matvec_transposed(ds, a, workers=3))
    assert np.allclose(t1, dense.T @ a, rtol=1e-12, atol=1e-12)
    assert np.allclose(ref.matvec(ds, v), dense @ v, rtol=1e-12, atol=1e-12)
    assert np.array_equal(ref.elementwise(3, a), -a)
    assert np.array_equal(ref.axpy(v, 0.5, v), v - 0.5 * v)
