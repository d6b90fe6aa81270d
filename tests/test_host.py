"""The product's host layer (libsgdb_b200.so, host C++) against the golden
vectors and the reference: fixtures, LIBSVM parsing, layouts, binary cache,
assignment, plan grammar, the mini-batch schedule. Bit-exact (north star:
"the parsers and CSR indexing must be bit-exact"). Mirrors
proj/tests/test_dataset.cpp and the plan cases of test_async_engine.cpp.
No GPU needed.
"""
import os

import numpy as np
import pytest

import paper_1802_08800_b200 as S

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz"))


def same_ds(a, prefix):
    for f in ("values", "indices", "row_offsets", "labels"):
        assert np.array_equal(getattr(a, f), GOLD[f"{prefix}_{f}"]), f
    n, d, layout, pw = (int(x) for x in GOLD[f"{prefix}_shape"])
    assert (a.n_examples, a.n_features, int(a.layout), a.padded_width) == (n, d, layout, pw)


def test_fixtures_bit_exact():
    same_ds(S.fixtures.dense_classification(300, 12, 20250810), "dense")
    same_ds(S.fixtures.sparse_classification(400, 60, 6.0, 20250811), "sparse")


@pytest.mark.parametrize("seed", [20250811, 20250813])
def test_fixtures_match_live_reference(ref, seed):
    a = S.fixtures.sparse_classification(5000, 47236, 73.16, seed)
    b = ref.fixture_sparse(5000, 47236, 73.16, seed)
    for f in ("values", "indices", "row_offsets", "labels"):
        assert np.array_equal(getattr(a, f), getattr(b, f))
    a = S.fixtures.dense_classification(1000, 54, seed)
    b = ref.fixture_dense(1000, 54, seed)
    assert np.array_equal(a.values, b.values) and np.array_equal(a.labels, b.labels)


def test_layout_conversions_bit_exact():
    sparse = S.fixtures.sparse_classification(400, 60, 6.0, 20250811)
    same_ds(S.convert_layout(sparse, S.Layout.PaddedDense), "padded")
    dense = S.fixtures.dense_classification(300, 12, 20250810)
    same_ds(S.convert_layout(dense, S.Layout.DenseColMajor), "dcol")


def test_conversion_matrix_preserves_content():
    """test_dataset.cpp:282-299: every layout pair round-trips the canonical content."""
    rng = np.random.default_rng(1234)
    for _ in range(10):
        ds = S.fixtures.sparse_classification(int(rng.integers(1, 20)), int(rng.integers(1, 15)),
                                              3.0, int(rng.integers(1 << 30)))
        for a in S.Layout:
            x = S.convert_layout(ds, a)
            x.validate()
            back = S.convert_layout(x, S.Layout.Csr)
            assert np.array_equal(back.values, ds.values)
            assert np.array_equal(back.indices, ds.indices)
            assert np.array_equal(back.row_offsets, ds.row_offsets)


def test_densify_refuses_above_cap():
    ds = S.fixtures.sparse_classification(1000, 100000, 5.0, 1)
    with pytest.raises(S.CapacityError):
        S.convert_layout(ds, S.Layout.DenseRowMajor, max_dense_bytes=1 << 20)


@pytest.mark.parametrize("i", range(9))
def test_parser_bit_exact(i):
    text = str(GOLD["parse_cases"][i])
    if f"parse_{i}_error_line" in GOLD:
        with pytest.raises(S.ParseError) as e:
            S.parse_libsvm(text)
        assert e.value.line_number == int(GOLD[f"parse_{i}_error_line"][0])
        assert f"line {e.value.line_number}" in str(e.value)
    else:
        same_ds(S.parse_libsvm(text), f"parse_{i}")


def test_parser_declared_dimension():
    """test_dataset.cpp:95-99 and the out-of-range case."""
    assert S.parse_libsvm("+1 1:1.0\n", 54).n_features == 54
    with pytest.raises(S.ParseError) as e:
        S.parse_libsvm("+1 5:1.0\n", 4)
    assert e.value.line_number == int(GOLD["parse_declared_error_line"][0])


def test_parser_label_codings():
    ds = S.parse_libsvm("0 1:1\n1 1:1\n2 1:1\n-1 1:1\n+1 1:1\n3 1:1\n")
    assert ds.labels.tolist() == [-1, 1, -1, -1, 1, 1]


def test_libsvm_round_trip_matches_reference(ref):
    ds = S.fixtures.sparse_classification(40, 30, 6.0, 7)
    text = S.write_libsvm(ds)
    assert text == ref.write_libsvm(ds)
    back = S.parse_libsvm(text, ds.n_features)
    assert np.array_equal(back.values, ds.values) and np.array_equal(back.indices, ds.indices)


def test_binary_cache_round_trip(tmp_path):
    """test_dataset.cpp:106-122: bit-exact."""
    ds = S.fixtures.sparse_classification(25, 40, 6.0, 11)
    p = str(tmp_path / "c.bin")
    S.save_binary(ds, p)
    back = S.load_binary(p)
    for f in ("values", "indices", "row_offsets", "labels"):
        assert getattr(back, f).tobytes() == getattr(ds, f).tobytes()
    with open(p, "r+b") as f:
        f.write(b"XXXXXXXX")
    with pytest.raises(Exception):
        S.load_binary(p)


def test_assign_bit_exact():
    for case in GOLD["assign_cases"]:
        n, wk, rr, k = (int(x) for x in str(case).split(","))
        lists = S.assign(n, wk, S.Strategy.RoundRobin if rr else S.Strategy.Chunk, k)
        flat = np.array([x for l in lists for x in l], np.uint32)
        assert np.array_equal(flat, GOLD[f"assign_{n}_{wk}_{rr}_{k}_ids"])


def test_assign_property():
    """test_dataset.cpp:242-280: k=0 partitions [0,n); k>0 appends k wrapped ids."""
    rng = np.random.default_rng(99)
    for _ in range(60):
        n, workers = int(rng.integers(1, 81)), int(rng.integers(1, 9))
        strat = S.Strategy(int(rng.integers(0, 2)))
        k = int(rng.integers(0, 5))
        base = S.assign(n, workers, strat, 0)
        assert sorted(x for l in base for x in l) == list(range(n))
        rep = S.assign(n, workers, strat, k)
        for b, r in zip(base, rep):
            if not b:
                assert not r
                continue
            assert r[:len(b)] == b
            assert r[len(b):] == [(b[-1] + 1 + i) % n for i in range(k)]


def test_schedule_bit_exact():
    s = S.Schedule(7, 50)
    for e in range(3):
        assert np.array_equal(s.next(), GOLD["schedule_7_50"][e])


def test_plan_grammar():
    """test_async_engine.cpp:50-75."""
    p1 = S.parse_plan("col-rr + block + no-rep")
    assert (p1.access_path, p1.model_replication, p1.data_replication_k) == (
        S.AccessPath.ColRR, S.ModelReplication.Block, 0)
    p2 = S.parse_plan("row-rr + kernel + rep-10")
    assert (p2.access_path, p2.data_replication_k) == (S.AccessPath.RowRR, 10)
    assert S.plan_to_string(p2) == "row-rr:kernel:10"
    p3 = S.parse_plan("row-ch:example:5")
    assert p3.model_replication == S.ModelReplication.Example and p3.data_replication_k == 5
    for bad in ("diagonal + kernel + no-rep", "row-rr + socket + no-rep", "row-rr + kernel + rep-x",
                "row-rr + kernel"):
        with pytest.raises(ValueError):
            S.parse_plan(bad)
    assert (p2.workers, p2.group_size, p2.circular_offsets, p2.merge_period_epochs) == (1, 32, True, 1)


def test_plan_validation():
    """test_async_engine.cpp:77-97."""
    csr = S.fixtures.sparse_classification(20, 30, 3.0, 1)
    padded = S.convert_layout(csr, S.Layout.PaddedDense)
    drow = S.fixtures.dense_classification(20, 6, 2)
    dcol = S.convert_layout(drow, S.Layout.DenseColMajor)
    col = S.parse_plan("col-rr:kernel:0")
    with pytest.raises(ValueError):
        S.validate_plan(col, csr)
    S.validate_plan(col, padded)
    S.validate_plan(col, dcol)
    with pytest.raises(ValueError):
        S.validate_plan(col, drow)
    row = S.parse_plan("row-ch:kernel:0")
    S.validate_plan(row, csr)
    with pytest.raises(ValueError):
        S.validate_plan(row, dcol)
    ex = S.parse_plan("row-ch:example:0")
    S.validate_plan(ex, csr)
    S.validate_plan(ex, padded)
    with pytest.raises(ValueError):
        S.validate_plan(ex, drow)


def test_merge_models_matches_golden():
    reps = [r.copy() for r in GOLD["merge_reps"]]
    assert np.array_equal(S.hogwild.merge_models(reps), GOLD["merge_mean"])
    assert all(np.array_equal(r, GOLD["merge_mean"]) for r in reps)
    reps = [r.copy() for r in GOLD["merge_reps"]]
    assert np.array_equal(S.hogwild.merge_models(reps, [3.0, 1.0, 0.5, 2.0, 0.25]),
                          GOLD["merge_weighted"])
    with pytest.raises(ValueError):
        S.hogwild.merge_models([])


def test_validate_dataset():
    ds = S.fixtures.sparse_classification(10, 5, 2.0, 3)
    ds.validate()
    ds.labels[0] = 0.5
    with pytest.raises(ValueError):
        ds.validate()
