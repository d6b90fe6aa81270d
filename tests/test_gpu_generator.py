"""K9, the device generator of the 200M x 1000 configuration (BASELINE.json
configs[4]): device slices are bit-identical to the CPU restatement
(oracle/glm_oracle.cpp orc_philox_dense), and synchronous training on
device-generated data matches the oracle run on the restated slice."""
import numpy as np
import pytest

from conftest import rel, rel_l2

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,d,row_base,seed", [(3000, 1000, 0, 20250815), (2048, 1000, 123456789, 7),
                                               (777, 54, 5, 3), (129, 7, 1, 11)])
def test_generated_slice_is_bit_exact(sgdb, dev, orc, n, d, row_base, seed):
    S = sgdb
    dds = S.DeviceDataset.generate_dense(dev, n, d, seed, row_base=row_base,
                                         n_global=max(200_000_000, row_base + n))
    vals, labs = dds.read_dense(0, n)
    ref = orc.philox_dense(n, d, seed, row_base=row_base)
    assert np.array_equal(vals.astype(np.float64).ravel(), ref.values)
    assert np.array_equal(labs.astype(np.float64), ref.labels)


def test_generated_distribution():
    """uniform(-1,1) values, balanced labels, ~10% flips (fixtures.cpp:19-26)."""
    import oracle
    ds = oracle.oracle().philox_dense(20000, 100, 9, noise=0.0)
    noisy = oracle.oracle().philox_dense(20000, 100, 9, noise=0.1)
    v = ds.values
    assert v.min() >= -1.0 and v.max() < 1.0 and abs(v.mean()) < 0.01
    assert abs(ds.labels.mean()) < 0.05
    assert 0.08 < np.mean(ds.labels != noisy.labels) < 0.12


@pytest.mark.parametrize("batch", ["N", 4096])
def test_sync_on_generated_data_matches_oracle(sgdb, dev, orc, batch):
    S = sgdb
    n, d, seed = 20000, 1000, 20250815
    dds = S.DeviceDataset.generate_dense(dev, n, d, seed)
    b = n if batch == "N" else batch
    alpha = 1.0 / b / 10
    hp = S.Hyperparams(alpha=alpha, batch_b=b, epochs=4, task=S.Task.LR)
    r = S.sync.train(S.Task.LR, dds, hp, 5)
    host = orc.philox_dense(n, d, seed)
    om, ol, _ = orc.sync_train(host, 0, alpha, b, 4, 5)
    assert rel_l2(r.model, om[-1]) <= 1e-5
    for e in range(4):
        assert rel(r.trace.epochs[e].loss, ol[e]) <= 1e-6
