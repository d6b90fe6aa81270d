"""Ingestion → device pipeline, end to end on real files.

A LIBSVM text file is written (write_libsvm of a fixture, then edited to
carry the label codings, zero values and trailing blanks real files have),
parsed by the engine's host parser and by the reference's parse_libsvm
(bit-exact, proj/src/dataset.cpp:167-230), round-tripped through the binary
cache (save_binary / load_binary, :302-327), uploaded to the device and
trained; the trained models equal the reference's sync::train / hogwild::train
on the reference's own parse of the same file (fp32 tolerance). The
slot-major padded layout of a CSR upload is built on the device
(SGDB_UPLOAD_PADDED, csr_to_padded, :380-402) and serves the column access
paths exactly like a host-converted PaddedDense upload.
"""
import os

import numpy as np
import pytest

from conftest import rel, rel_l2

pytestmark = pytest.mark.gpu


def _libsvm_file(S, tmp_path):
    ds = S.fixtures.sparse_classification(1500, 400, 12.0, 77)
    text = S.write_libsvm(ds)
    lines = text.splitlines()
    # real-file features: label codings 0/2/+1, explicit zeros, extra spaces
    out = []
    for i, ln in enumerate(lines):
        lab, *feats = ln.split()
        if i % 7 == 0:
            lab = "0" if lab.startswith("-") else "+1"
        elif i % 11 == 0 and lab.startswith("-"):
            lab = "2"
        if i % 5 == 0 and feats:
            feats.append("401:0")  # a zero value: dropped by the parser, and d grows to 401
        out.append(" ".join([lab] + feats) + ("  " if i % 3 == 0 else ""))
    path = tmp_path / "data.libsvm"
    path.write_text("\n".join(out) + "\n")
    return str(path)


def test_libsvm_file_to_device_training(sgdb, dev, ref, tmp_path):
    S = sgdb
    path = _libsvm_file(S, tmp_path)
    text = open(path, "rb").read()
    ours = S.parse_libsvm(text)
    theirs, err_line = ref.parse_libsvm(text)
    assert err_line is None
    assert ours.n_examples == theirs.n_examples and ours.n_features == theirs.n_features
    np.testing.assert_array_equal(ours.labels, theirs.labels)
    np.testing.assert_array_equal(ours.values, theirs.values)
    np.testing.assert_array_equal(ours.indices, theirs.indices)
    np.testing.assert_array_equal(ours.row_offsets.astype(np.uint64), theirs.row_offsets.astype(np.uint64))
    # binary cache round trip, then the device
    cache = os.path.join(str(tmp_path), "data.sgdbds")
    S.save_binary(ours, cache)
    cached = S.load_binary(cache)
    np.testing.assert_array_equal(cached.values, ours.values)
    host = cached.rounded_f32()  # the reference trains on the same (fp32-rounded) parse
    dds = S.DeviceDataset(dev, host)
    hp = S.Hyperparams(alpha=0.05, batch_b=128, epochs=4, task=S.Task.SVM)
    r = S.sync.train(S.Task.SVM, dds, hp, 9)
    om, ol, _, div = ref.sync_train(host, 1, 0.05, 128, 4, 9)
    assert not div
    assert rel_l2(r.model, om) <= 1e-5
    assert rel(r.trace.final_loss(), ol[-1]) <= 1e-6
    plan = S.parse_plan("row-rr:kernel:0")
    plan.workers = 1
    h = S.hogwild.train(S.Task.LR, dds, S.Hyperparams(alpha=0.02, batch_b=1, epochs=2, task=S.Task.LR),
                        plan, 0)
    hm, hl, _, _ = ref.hogwild_train(host, 0, 0.02, 2, "row-rr:kernel:0", workers=1)
    assert rel_l2(h.model, hm) <= 1e-4


@pytest.mark.parametrize("plan_text", ["col-rr:kernel:0", "col-ch:kernel:0", "col-rr:block:0"])
def test_device_padded_conversion_equals_host_conversion(sgdb, dev, orc, plan_text):
    S = sgdb
    csr = S.fixtures.sparse_classification(700, 120, 9.0, 13).rounded_f32()
    host_padded = S.convert_layout(csr, S.Layout.PaddedDense)
    a = S.DeviceDataset(dev, host_padded)
    b = S.DeviceDataset(dev, csr, padded=True)
    plan = S.parse_plan(plan_text)
    plan.workers = 1
    hp = S.Hyperparams(alpha=0.03, batch_b=1, epochs=2, task=S.Task.SVM)
    ra = S.hogwild.train(S.Task.SVM, a, hp, plan, 0)
    rb = S.hogwild.train(S.Task.SVM, b, hp, plan, 0)
    np.testing.assert_array_equal(ra.model, rb.model)  # same layout on the device: same bits
    rr = "rr" in plan_text
    repl = 1 if ":block:" in plan_text else 0
    om, _, _ = orc.hogwild_serial(host_padded, 1, 0.03, 2, rr, repl, 0, 1)
    assert rel_l2(rb.model, om[-1]) <= 1e-4


def test_padded_upload_flag_rejections(sgdb, dev):
    S = sgdb
    dense = S.fixtures.dense_classification(50, 8, 2).rounded_f32()
    with pytest.raises(ValueError):
        S.DeviceDataset(dev, dense, padded=True)
    csr = S.fixtures.sparse_classification(50, 8, 3.0, 2).rounded_f32()
    with pytest.raises(S.UnsupportedError):
        S.DeviceDataset(dev, csr, padded=True, exact=True)
