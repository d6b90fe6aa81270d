"""Generates tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref,
compiled from /root/reference/proj/src by oracle/Makefile).

Run here (the reference exists only in this container):
    make -C oracle && python tests/golden/make_golden.py

The fixtures are small on purpose (committed, a few hundred KB). Every array
is exactly what the reference computes in fp64; the CPU tests pin the oracle
restatement to them bit for bit and the GPU tests compare the device against
them within the stated fp32 tolerance.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402


def pack_ds(prefix, ds, out):
    out[f"{prefix}_shape"] = np.array([ds.n_examples, ds.n_features, ds.layout, ds.padded_width],
                                      np.uint64)
    out[f"{prefix}_labels"] = ds.labels
    out[f"{prefix}_values"] = ds.values
    out[f"{prefix}_indices"] = ds.indices
    out[f"{prefix}_row_offsets"] = ds.row_offsets


def main():
    R = oracle.reference()
    out = {}
    # Fixtures (fixtures.cpp:30-100) — the acceptance defaults, scaled down.
    dense = R.fixture_dense(300, 12, 20250810)
    sparse = R.fixture_sparse(400, 60, 6.0, 20250811)
    pack_ds("dense", dense, out)
    pack_ds("sparse", sparse, out)
    padded = R.convert_layout(sparse, oracle.PADDED)
    dcol = R.convert_layout(dense, oracle.DENSE_COL)
    pack_ds("padded", padded, out)
    pack_ds("dcol", dcol, out)

    # Synchronous training, per-epoch models and losses (sync_engine.cpp:56-121),
    # on fp32-rounded inputs (what the device stores).
    runs = []
    for name, ds in (("dense", dense), ("sparse", sparse)):
        ds32 = oracle.oracle().round_f32(ds)
        for task in (0, 1):
            for b in (ds.n_examples, 32, 1):
                alpha = 1.0 / b
                models, losses = R.sync_train_dump(ds32, task, alpha, b, 5, 17)
                model, tl, _, _ = R.sync_train(ds32, task, alpha, b, 5, 17)
                assert np.array_equal(model, models[-1]) and np.array_equal(tl, losses)
                key = f"sync_{name}_t{task}_b{b}"
                out[key + "_models"] = models
                out[key + "_losses"] = losses
                runs.append(key)
    out["sync_runs"] = np.array(runs)

    # One-worker Hogwild == sequential Alg. 3 (async_engine.cpp:178-195).
    hw = []
    for name, ds, plan in (("sparse", sparse, "row-ch:kernel:0"), ("sparse", sparse, "row-rr:block:2"),
                           ("dense", dense, "row-rr:thread:0"), ("padded", padded, "col-ch:kernel:0"),
                           ("dcol", dcol, "col-rr:block:0")):
        ds32 = oracle.oracle().round_f32(ds)
        for task in (0, 1):
            model, losses, _, evals = R.hogwild_train(ds32, task, 0.05, 3, plan, workers=1)
            key = f"hog_{name}_{plan.replace(':', '_').replace('-', '')}_t{task}"
            out[key + "_model"] = model
            out[key + "_losses"] = losses
            out[key + "_evals"] = evals
            hw.append(f"{key}|{name}|{plan}|{task}")
    out["hog_runs"] = np.array(hw)

    # Primitives at a random model.
    w = np.random.default_rng(5).normal(0, 0.5, 60)
    sp32 = oracle.oracle().round_f32(sparse)
    out["prim_w"] = w
    for task in (0, 1):
        out[f"prim_loss_t{task}"] = np.array([R.dataset_loss(sp32, task, w)])
        out[f"prim_grad_t{task}"] = R.batch_gradient(sp32, task, None, w)
        out[f"prim_grad_rows_t{task}"] = R.batch_gradient(sp32, task, np.arange(0, 400, 3), w)

    # Scalar cores (glm.cpp:24-34): margins incl. the extremes of test_glm.cpp.
    zs = np.array([-1e4, -745.0, -100.0, -1.0, -1e-9, 0.0, 1e-9, 0.5, 1.0, 1.0 + 1e-12, 100.0,
                   745.0, 1e4])
    out["core_z"] = zs
    for task in (0, 1):
        for y in (1.0, -1.0):
            out[f"core_coef_t{task}_y{int(y)}"] = np.array(
                [R.fn("point_coefficient")(task, z, y) for z in zs])
            out[f"core_loss_t{task}_y{int(y)}"] = np.array(
                [R.fn("point_loss_from_margin")(task, z, y) for z in zs])

    # Parser (dataset.cpp:167-230) cases from test_dataset.cpp:42-93.
    parse_cases = ["+1 1:0.5 3:2.0\n-1 2:1.0\n", "0 1:1\n1 1:1\n2 1:1\n-1 1:1\n+1 1:1\n3 1:1\n",
                   "", "+1\n-1 1:2.0\n", "+1 1:1.0 # comment\r\n\n  -1 4:0 5:-2.5e-3\n",
                   "+1 1:0.5\n-1 oops\n", "+1 3:1.0 2:1.0\n", "maybe 1:1\n", "+1 0:1\n"]
    out["parse_cases"] = np.array(parse_cases)
    for i, text in enumerate(parse_cases):
        ds, err = R.parse_libsvm(text)
        if err:
            out[f"parse_{i}_error_line"] = np.array([err[1]])
        else:
            pack_ds(f"parse_{i}", ds, out)
    ds, err = R.parse_libsvm("+1 5:1.0\n", 4)
    out["parse_declared_error_line"] = np.array([err[1]])

    # assign (dataset.cpp:470-503) known answers + a sweep.
    akat = []
    for n, wk, rr, k in ((5, 2, 1, 0), (6, 2, 0, 2), (10, 3, 0, 0), (3, 5, 0, 0), (7, 3, 1, 4),
                         (64700, 37, 0, 10)):
        lists = R.assign(n, wk, rr, k)
        flat = np.array([x for l in lists for x in l], np.uint32)
        offs = np.cumsum([0] + [len(l) for l in lists]).astype(np.uint64)
        out[f"assign_{n}_{wk}_{rr}_{k}_ids"] = flat
        out[f"assign_{n}_{wk}_{rr}_{k}_offs"] = offs
        akat.append(f"{n},{wk},{rr},{k}")
    out["assign_cases"] = np.array(akat)

    # Schedule (sync_engine.cpp:75-84): 3 epochs of mt19937_64(7) + std::shuffle.
    out["schedule_7_50"] = oracle.oracle().schedule(7, 50, 3)

    # merge_models (async_engine.cpp:133-156).
    reps = np.random.default_rng(9).normal(0, 1, (5, 17))
    out["merge_reps"] = reps
    out["merge_mean"] = R.merge_models(reps)
    out["merge_weighted"] = R.merge_models(reps, np.array([3.0, 1.0, 0.5, 2.0, 0.25]))

    path = os.path.join(HERE, "reference_golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(out)} arrays)")


if __name__ == "__main__":
    main()
