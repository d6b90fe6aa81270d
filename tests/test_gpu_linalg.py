"""GPU parity of the §4 operator API (proj/include/sgdbench/linalg.hpp:23-58)
against the reference's own linalg:: functions (oracle/_ref).

Mirrors proj/tests/test_linalg.cpp: matvec / matvec_transposed over every
layout, with and without a row subset, and the elementwise primitives. The
device reproduces the reference's summation order (per-row slot order; per
column sequential for DenseColMajor; 256-row block partials + the fixed
pairwise tree otherwise), so on f32-valued inputs the results are BIT-EXACT,
and the reference is itself bit-identical for any worker count (checked at 1
and 4), including exp / sigmoid (glibc's exp restated in libm_exp.hpp).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _make(S, layout, n, d, seed, avg=None):
    if avg is None:
        ds = S.fixtures.dense_classification(n, d, seed).rounded_f32()
    else:
        ds = S.fixtures.sparse_classification(n, d, avg, seed).rounded_f32()
    if ds.layout != layout:
        ds = S.convert_layout(ds, layout)
    return ds


# (layout, n, d, avg_nnz): n spans 1, one block, block edges and the pairwise
# tree's ragged cases (3, 5, 6, 7, 9 blocks).
CASES = [
    (0, 1, 5, None),
    (0, 256, 33, None),
    (0, 257, 33, None),
    (0, 256 * 5 + 3, 54, None),
    (0, 256 * 7, 17, None),
    (1, 256 * 6 + 1, 54, None),
    (1, 300, 9, None),
    (2, 256 * 9 - 1, 500, 12.0),
    (2, 2000, 3000, 40.0),
    (3, 256 * 3 + 7, 200, 6.0),
]


@pytest.mark.parametrize("layout,n,d,avg", CASES)
def test_matvec_bit_exact(sgdb, ref, dev, layout, n, d, avg):
    S = sgdb
    ds = _make(S, S.Layout(layout), n, d, 100 + n, avg)
    rng = np.random.default_rng(n)
    v = rng.standard_normal(d)
    dds = S.DeviceDataset(dev, ds)
    got = S.linalg.matvec(dds, v)
    assert np.array_equal(got, ref.matvec(ds, v, workers=1))
    assert np.array_equal(got, ref.matvec(ds, v, workers=4))
    rows = np.sort(rng.choice(n, size=max(1, n // 3), replace=False)).astype(np.uint32)
    assert np.array_equal(S.linalg.matvec(dds, v, rows), ref.matvec(ds, v, rows))


@pytest.mark.parametrize("layout,n,d,avg", CASES)
def test_matvec_transposed_bit_exact(sgdb, ref, dev, layout, n, d, avg):
    S = sgdb
    ds = _make(S, S.Layout(layout), n, d, 200 + n, avg)
    rng = np.random.default_rng(n + 1)
    a = rng.standard_normal(n)
    dds = S.DeviceDataset(dev, ds)
    got = S.linalg.matvec_transposed(dds, a)
    want = ref.matvec_transposed(ds, a, workers=1)
    assert np.array_equal(got, want)
    assert np.array_equal(want, ref.matvec_transposed(ds, a, workers=4))
    # Row subset in arbitrary (shuffled) order, a indexed by position.
    rows = rng.permutation(n)[: max(1, (2 * n) // 3)].astype(np.uint32)
    ap = rng.standard_normal(rows.size)
    assert np.array_equal(S.linalg.matvec_transposed(dds, ap, rows),
                          ref.matvec_transposed(ds, ap, rows))


def test_matvec_transposed_chunked_tree(sgdb, ref, dev):
    """d = 2^20: the block partials no longer fit one 256 MiB chunk (32 blocks),
    so the pairwise tree is carried across chunks on the per-coordinate stack."""
    S = sgdb
    n, d = 256 * 37 + 5, 1 << 20
    ds = _make(S, S.Layout.Csr, n, d, 7, 8.0)
    a = np.random.default_rng(3).standard_normal(n)
    got = S.linalg.matvec_transposed(S.DeviceDataset(dev, ds), a)
    assert np.array_equal(got, ref.matvec_transposed(ds, a, workers=8))


def test_empty_and_errors(sgdb, ref, dev):
    S = sgdb
    ds = _make(S, S.Layout.DenseRowMajor, 300, 10, 1)
    dds = S.DeviceDataset(dev, ds)
    with pytest.raises(ValueError, match="dimension mismatch"):
        S.linalg.matvec(dds, np.zeros(9))
    with pytest.raises(ValueError, match="dimension mismatch"):
        S.linalg.matvec_transposed(dds, np.zeros(299))
    # Empty row subset = all rows; zero-length a with n == 0 gives zeros.
    empty = S.Dataset(0, 4, S.Layout.Csr, np.zeros(0), np.zeros(0), np.zeros(0, np.uint32),
                      np.zeros(1, np.uint64))
    assert np.array_equal(S.linalg.matvec_transposed(S.DeviceDataset(dev, empty), np.zeros(0)),
                          np.zeros(4))
    with pytest.raises(ArithmeticError, match="division by zero at position 2"):
        S.linalg.ew_div(np.ones(4), np.array([1.0, 2.0, 0.0, 4.0]))
    with pytest.raises(ValueError, match="length mismatch"):
        S.linalg.ew_mul(np.ones(3), np.ones(4))
    with pytest.raises(ValueError, match="length mismatch"):
        S.linalg.axpy(np.ones(3), 0.5, np.ones(4))


def test_elementwise(sgdb, ref, dev):
    S = sgdb
    rng = np.random.default_rng(5)
    n = 100_003
    a = rng.standard_normal(n) * 30.0
    a[:6] = [0.0, -0.0, 1.0, 0.999999999, -745.5, 709.0]
    b = rng.standard_normal(n)
    b[b == 0.0] = 1.0
    Op = S.ElementwiseOp
    for op, bb, sc in [(Op.Mul, b, 0.0), (Op.Div, b, 0.0), (Op.Neg, None, 0.0),
                       (Op.AddScalar, None, -2.5), (Op.HingeIndicator, None, 0.0)]:
        got = S.linalg.elementwise(op, a, bb, sc)
        assert np.array_equal(got, ref.elementwise(int(op), a, bb, sc)), op
    for op in (Op.Exp, Op.Sigmoid):  # glibc's exp restated (libm_exp.hpp): bitwise too
        got = S.linalg.elementwise(op, a)
        assert np.array_equal(got, ref.elementwise(int(op), a)), op
    # The named wrappers route to the same kernels.
    assert np.array_equal(S.linalg.ew_add_scalar(3.0, a), ref.elementwise(4, a, None, 3.0))
    assert np.array_equal(S.linalg.ew_neg(a), -a)


def test_axpy_bit_exact(sgdb, ref, dev):
    S = sgdb
    rng = np.random.default_rng(9)
    w = rng.standard_normal(50_001)
    g = rng.standard_normal(50_001)
    want = ref.axpy(w, 0.37, g)
    S.linalg.axpy(w, 0.37, g)
    assert np.array_equal(w, want)


@pytest.mark.parametrize("task", [0, 1])
def test_primitive_chain_equals_batch_gradient(sgdb, ref, dev, task):
    """The paper's §4 chain (matvec -> elementwise -> matvec_transposed) built
    from the device primitives, step for step as sync_engine.cpp:27-40 chains
    them, reproduces the reference's batch gradient on the same rows, bit for
    bit (both tasks: exp is glibc's)."""
    S = sgdb
    la = S.linalg
    ds = _make(S, S.Layout.Csr, 2000, 800, 31, 20.0)
    dds = S.DeviceDataset(dev, ds)
    rng = np.random.default_rng(4)
    w = rng.standard_normal(800) * 0.1
    rows = np.sort(rng.choice(2000, 512, replace=False)).astype(np.uint32)
    y = ds.labels[rows]
    m = la.ew_mul(y, la.matvec(dds, w, rows))
    if task == 0:
        c = la.ew_mul(la.ew_sigmoid(la.ew_neg(m)), la.ew_neg(y))
    else:
        c = la.ew_mul(la.ew_hinge_indicator(m), la.ew_neg(y))
    g = la.matvec_transposed(dds, c, rows)
    assert np.array_equal(g, ref.batch_gradient(ds, task, rows, w))
