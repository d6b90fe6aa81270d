"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the GLM SGD hot path.

Two ctypes-loaded libraries, both built by ``make -C oracle``:

* ``liboracle.so``  — ``oracle/glm_oracle.cpp``, our fp64 CPU restatement of the
  reference algorithms (each function cites /root/reference/proj file:line).
* ``_ref/libsgdbench_ref.so`` — the UNMODIFIED reference compiled from its own
  sources plus ``oracle/ref_capi.cpp`` wrappers (built only where
  /root/reference exists; the built file travels to the GPU box).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package — as the checker, never as the
thing measured or shipped. The product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(_HERE, "liboracle.so")
REF_SO = os.path.join(_HERE, "_ref", "libsgdbench_ref.so")

LR, SVM = 0, 1
DENSE_ROW, DENSE_COL, CSR, PADDED = 0, 1, 2, 3

_u64 = C.c_uint64
_i64 = C.c_int64
_dbl = C.c_double
_int = C.c_int
_vp = C.c_void_p
_P = C.POINTER


@dataclass
class HostData:
    """Plain numpy mirror of sgdbench::Dataset (include/sgdbench/dataset.hpp:42-61)."""

    n_examples: int
    n_features: int
    layout: int
    labels: np.ndarray
    values: np.ndarray
    indices: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    row_offsets: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    padded_width: int = 0


def _ptr(a, ct):
    if a is None or len(a) == 0:
        return None
    return a.ctypes.data_as(_P(ct))


class _Lib:
    def __init__(self, path, prefix):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        self.p = prefix
        L = self.lib
        f = getattr(L, f"{prefix}_ds_from_arrays")
        f.restype = _vp
        f.argtypes = [_u64, _u64, _int, _P(_dbl), _P(_dbl), _u64, _P(C.c_uint32), _u64,
                      _P(_u64), _u64, _u64]
        getattr(L, f"{prefix}_ds_free").argtypes = [_vp]
        getattr(L, f"{prefix}_ds_info").argtypes = [_vp, _P(_u64)]
        getattr(L, f"{prefix}_ds_copy").argtypes = [_vp, _P(_dbl), _P(_dbl), _P(C.c_uint32),
                                                     _P(_u64)]
        for name, args in (("fixture_dense", [_u64, _u64, _u64, _dbl]),
                           ("fixture_sparse", [_u64, _u64, _dbl, _u64, _dbl])):
            fn = getattr(L, f"{prefix}_{name}")
            fn.restype = _vp
            fn.argtypes = args
        fn = getattr(L, f"{prefix}_dataset_loss")
        fn.restype = _dbl
        fn.argtypes = [_vp, _int, _P(_dbl)]
        fn = getattr(L, f"{prefix}_last_error")
        fn.restype = C.c_char_p
        for name in ("point_coefficient", "point_loss_from_margin"):
            fn = getattr(L, f"{prefix}_{name}")
            fn.restype = _dbl
            fn.argtypes = [_int, _dbl, _dbl]
        fn = getattr(L, f"{prefix}_assign")
        fn.restype = _u64
        fn.argtypes = [_u64, _u64, _int, _u64, _P(C.c_uint32), _P(_u64)]
        fn = getattr(L, f"{prefix}_parse_libsvm")
        fn.restype = _int
        fn.argtypes = [C.c_char_p, _u64, _i64, _P(_vp), _P(_u64)]

    def fn(self, name):
        return getattr(self.lib, f"{self.p}_{name}")

    def err(self):
        return self.fn("last_error")().decode()

    # -- dataset marshalling -------------------------------------------------
    def to_handle(self, ds: HostData):
        labels = np.ascontiguousarray(ds.labels, np.float64)
        values = np.ascontiguousarray(ds.values, np.float64)
        indices = np.ascontiguousarray(ds.indices, np.uint32)
        offs = np.ascontiguousarray(ds.row_offsets, np.uint64)
        return self.fn("ds_from_arrays")(ds.n_examples, ds.n_features, ds.layout,
                                         _ptr(labels, _dbl), _ptr(values, _dbl), len(values),
                                         _ptr(indices, C.c_uint32), len(indices),
                                         _ptr(offs, _u64), len(offs), ds.padded_width)

    def from_handle(self, h, free=True) -> HostData:
        info = (_u64 * 7)()
        self.fn("ds_info")(h, info)
        n, d, layout, nv, ni, no, pw = (int(x) for x in info)
        labels = np.zeros(n, np.float64)
        values = np.zeros(nv, np.float64)
        indices = np.zeros(ni, np.uint32)
        offs = np.zeros(no, np.uint64)
        self.fn("ds_copy")(h, _ptr(labels, _dbl), _ptr(values, _dbl),
                           _ptr(indices, C.c_uint32), _ptr(offs, _u64))
        if free:
            self.fn("ds_free")(h)
        return HostData(n, d, layout, labels, values, indices, offs, pw)

    # -- fixtures -------------------------------------------------------------
    def fixture_dense(self, n, d, seed, noise=0.1) -> HostData:
        return self.from_handle(self.fn("fixture_dense")(n, d, seed, noise))

    def fixture_sparse(self, n, d, avg, seed, noise=0.1) -> HostData:
        return self.from_handle(self.fn("fixture_sparse")(n, d, avg, seed, noise))

    def dataset_loss(self, ds: HostData, task, w) -> float:
        h = self.to_handle(ds)
        try:
            w = np.ascontiguousarray(w, np.float64)
            return self.fn("dataset_loss")(h, task, _ptr(w, _dbl))
        finally:
            self.fn("ds_free")(h)

    def assign(self, n, workers, round_robin, k):
        total = self.fn("assign")(n, workers, int(round_robin), k, None, None)
        out = np.zeros(total, np.uint32)
        offs = np.zeros(workers + 1, np.uint64)
        self.fn("assign")(n, workers, int(round_robin), k, _ptr(out, C.c_uint32), _ptr(offs, _u64))
        return [out[int(offs[w]):int(offs[w + 1])].tolist() for w in range(workers)]

    def parse_libsvm(self, text: str | bytes, declared_d=None):
        """Returns (HostData, None) or (None, (kind, line, message))."""
        b = text.encode() if isinstance(text, str) else text
        h = _vp()
        line = _u64(0)
        rc = self.fn("parse_libsvm")(b, len(b), -1 if declared_d is None else declared_d,
                                     C.byref(h), C.byref(line))
        if rc == 0:
            return self.from_handle(h.value), None
        return None, ("parse" if rc == 1 else "other", int(line.value), self.err())


class Oracle(_Lib):
    """Our restatement (glm_oracle.cpp)."""

    def __init__(self):
        super().__init__(ORACLE_SO, "orc")
        L = self.lib
        L.orc_round_f32.argtypes = [_vp]
        L.orc_convert_layout.restype = _vp
        L.orc_convert_layout.argtypes = [_vp, _int]
        L.orc_schedule.argtypes = [_u64, _u64, _u64, _int, _P(C.c_uint32)]
        L.orc_batch_gradient.argtypes = [_vp, _int, _P(C.c_uint32), _u64, _P(_dbl), _P(_dbl)]
        L.orc_sync_train.restype = _u64
        L.orc_sync_train.argtypes = [_vp, _int, _dbl, _u64, _u64, _dbl, _u64, _int, _P(_dbl),
                                     _P(_dbl), _P(_dbl), _P(_int)]
        L.orc_hogwild_serial.restype = _u64
        L.orc_hogwild_serial.argtypes = [_vp, _int, _dbl, _u64, _dbl, _int, _int, _u64, _u64,
                                         _u64, _int, _P(_dbl), _P(_dbl), _P(_dbl), _P(_u64)]
        L.orc_merge_models.argtypes = [_P(_dbl), _u64, _u64, _P(_dbl), _P(_dbl)]
        L.orc_philox_hidden_model.argtypes = [_u64, _u64, _P(_dbl)]
        L.orc_philox_dense.argtypes = [_u64, _u64, _u64, _u64, _dbl, _P(_dbl), _P(_dbl)]
        L.orc_philox_dense_gradient.argtypes = [_u64, _u64, _u64, _u64, _dbl, _int, _P(_dbl),
                                                C.c_uint32, _P(_dbl), _P(_dbl)]

    def round_f32(self, ds: HostData) -> HostData:
        out = HostData(**ds.__dict__)
        out.values = ds.values.astype(np.float32).astype(np.float64)
        return out

    def convert_layout(self, ds: HostData, target) -> HostData:
        h = self.to_handle(ds)
        try:
            return self.from_handle(self.lib.orc_convert_layout(h, target))
        finally:
            self.lib.orc_ds_free(h)

    def schedule(self, seed, n, epochs, shuffle=True) -> np.ndarray:
        out = np.zeros(epochs * n, np.uint32)
        self.lib.orc_schedule(seed, n, epochs, int(shuffle), _ptr(out, C.c_uint32))
        return out.reshape(epochs, n)

    def batch_gradient(self, ds: HostData, task, rows, w) -> np.ndarray:
        h = self.to_handle(ds)
        try:
            rows = np.ascontiguousarray(rows if rows is not None else [], np.uint32)
            w = np.ascontiguousarray(w, np.float64)
            g = np.zeros(ds.n_features, np.float64)
            self.lib.orc_batch_gradient(h, task, _ptr(rows, C.c_uint32), len(rows),
                                        _ptr(w, _dbl), _ptr(g, _dbl))
            return g
        finally:
            self.lib.orc_ds_free(h)

    def sync_train(self, ds: HostData, task, alpha, batch_b, epochs, seed, decay=1.0,
                   shuffle=True, init=None):
        """Returns (models[epochs_run, d], losses[epochs_run], diverged)."""
        h = self.to_handle(ds)
        try:
            d = ds.n_features
            models = np.zeros((epochs, d), np.float64)
            losses = np.zeros(epochs, np.float64)
            div = _int(0)
            init_a = None if init is None else np.ascontiguousarray(init, np.float64)
            ran = self.lib.orc_sync_train(h, task, alpha, batch_b, epochs, decay, seed,
                                          int(shuffle), _ptr(init_a, _dbl), _ptr(models, _dbl),
                                          _ptr(losses, _dbl), C.byref(div))
            return models[:ran], losses[:ran], bool(div.value)
        finally:
            self.lib.orc_ds_free(h)

    def hogwild_serial(self, ds: HostData, task, alpha, epochs, round_robin, replication, k,
                       workers, group_size=32, offsets=True, decay=1.0, init=None):
        """Returns (models[epochs_run, d], losses, evals)."""
        h = self.to_handle(ds)
        try:
            d = ds.n_features
            models = np.zeros((epochs, d), np.float64)
            losses = np.zeros(epochs, np.float64)
            evals = np.zeros(epochs, np.uint64)
            init_a = None if init is None else np.ascontiguousarray(init, np.float64)
            ran = self.lib.orc_hogwild_serial(h, task, alpha, epochs, decay, int(round_robin),
                                              replication, k, workers, group_size, int(offsets),
                                              _ptr(init_a, _dbl), _ptr(models, _dbl),
                                              _ptr(losses, _dbl), _ptr(evals, _u64))
            return models[:ran], losses[:ran], evals[:ran]
        finally:
            self.lib.orc_ds_free(h)

    def philox_hidden_model(self, seed, d) -> np.ndarray:
        w = np.zeros(d, np.float64)
        self.lib.orc_philox_hidden_model(seed, d, _ptr(w, _dbl))
        return w

    def philox_dense(self, n, d, seed, row_base=0, noise=0.1) -> HostData:
        """Rows [row_base, row_base+n) of the device generator's dataset (K9 restatement)."""
        values = np.zeros(n * d, np.float64)
        labels = np.zeros(n, np.float64)
        self.lib.orc_philox_dense(n, d, row_base, seed, noise, _ptr(values, _dbl), _ptr(labels, _dbl))
        return HostData(n, d, DENSE_ROW, labels, values)

    def philox_dense_gradient(self, n, d, seed, task, w, row_base=0, noise=0.1, threads=None):
        """Full-batch gradient and loss at w over rows [row_base, row_base+n) of the
        device generator's dataset, streamed (rows regenerated, never stored)."""
        threads = threads or max(1, os.cpu_count() or 1)
        w = np.ascontiguousarray(w, np.float64)
        g = np.zeros(d, np.float64)
        loss = _dbl(0.0)
        self.lib.orc_philox_dense_gradient(n, d, row_base, seed, noise, task, _ptr(w, _dbl),
                                           threads, _ptr(g, _dbl), C.byref(loss))
        return g, float(loss.value)

    def merge_models(self, replicas: np.ndarray, weights=None) -> np.ndarray:
        reps = np.ascontiguousarray(replicas, np.float64)
        r, d = reps.shape
        out = np.zeros(d, np.float64)
        wts = None if weights is None else np.ascontiguousarray(weights, np.float64)
        self.lib.orc_merge_models(_ptr(reps.ravel(), _dbl), r, d, _ptr(wts, _dbl),
                                  _ptr(out, _dbl))
        return out


class Reference(_Lib):
    """The unmodified reference (oracle/_ref/libsgdbench_ref.so)."""

    def __init__(self):
        super().__init__(REF_SO, "ref")
        L = self.lib
        L.ref_sync_train.restype = _int
        L.ref_sync_train.argtypes = [_vp, _int, _dbl, _u64, _u64, _dbl, _u64, C.c_uint, _int,
                                     _P(_dbl), _P(_dbl), _P(_dbl), _P(_dbl), _P(_u64), _P(_int)]
        L.ref_sync_train_dump.restype = _int
        L.ref_sync_train_dump.argtypes = [_vp, _int, _dbl, _u64, _u64, _dbl, _u64, C.c_uint,
                                          _int, _P(_dbl), _P(_dbl)]
        L.ref_hogwild_train.restype = _int
        L.ref_hogwild_train.argtypes = [_vp, _int, _dbl, _u64, _dbl, C.c_char_p, _u64, _u64,
                                        _int, _u64, _int, _P(_dbl), _P(_dbl), _P(_dbl),
                                        _P(_dbl), _P(_u64), _P(_u64)]
        L.ref_batch_gradient.restype = _int
        L.ref_batch_gradient.argtypes = [_vp, _int, _P(C.c_uint32), _u64, _P(_dbl), C.c_uint,
                                         _P(_dbl)]
        L.ref_epoch_batch.restype = _dbl
        L.ref_epoch_batch.argtypes = [_vp, _int, _P(_dbl), _dbl, C.c_uint]
        L.ref_convert_layout.restype = _int
        L.ref_convert_layout.argtypes = [_vp, _int, _u64, _P(_vp)]
        L.ref_merge_models.argtypes = [_P(_dbl), _u64, _u64, _P(_dbl), _P(_dbl)]
        L.ref_hardware_threads.restype = C.c_uint
        L.ref_write_libsvm.restype = _u64
        L.ref_write_libsvm.argtypes = [_vp, C.c_char_p, _u64]
        L.ref_matvec.restype = _int
        L.ref_matvec.argtypes = [_vp, _P(C.c_uint32), _u64, _P(_dbl), C.c_uint, _P(_dbl)]
        L.ref_matvec_transposed.restype = _int
        L.ref_matvec_transposed.argtypes = [_vp, _P(C.c_uint32), _u64, _P(_dbl), _u64, C.c_uint,
                                            _P(_dbl)]
        L.ref_elementwise.restype = _int
        L.ref_elementwise.argtypes = [_int, _P(_dbl), _P(_dbl), _u64, _dbl, C.c_uint, _P(_dbl)]
        L.ref_axpy.argtypes = [_P(_dbl), _dbl, _P(_dbl), _u64, C.c_uint]

    def hardware_threads(self) -> int:
        return int(self.lib.ref_hardware_threads())

    def assign(self, n, workers, round_robin, k):
        # ref_assign takes the reference's Strategy enum (RoundRobin = 0, Chunk = 1).
        return super().assign(n, workers, 0 if round_robin else 1, k)

    def convert_layout(self, ds: HostData, target) -> HostData:
        h = self.to_handle(ds)
        try:
            out = _vp()
            if self.lib.ref_convert_layout(h, target, 0, C.byref(out)) != 0:
                raise RuntimeError(self.err())
            return self.from_handle(out.value)
        finally:
            self.lib.ref_ds_free(h)

    def write_libsvm(self, ds: HostData) -> str:
        h = self.to_handle(ds)
        try:
            size = self.lib.ref_write_libsvm(h, None, 0)
            buf = C.create_string_buffer(int(size) + 1)
            self.lib.ref_write_libsvm(h, buf, size)
            return buf.raw[:size].decode()
        finally:
            self.lib.ref_ds_free(h)

    def matvec(self, ds: HostData, v, rows=None, workers=1) -> np.ndarray:
        """linalg::matvec (linalg.cpp:30-44)."""
        h = self.to_handle(ds)
        try:
            rows = np.ascontiguousarray(rows if rows is not None else [], np.uint32)
            v = np.ascontiguousarray(v, np.float64)
            out = np.zeros(len(rows) if len(rows) else ds.n_examples, np.float64)
            if self.lib.ref_matvec(h, _ptr(rows, C.c_uint32), len(rows), _ptr(v, _dbl), workers,
                                   _ptr(out, _dbl)) != 0:
                raise RuntimeError(self.err())
            return out
        finally:
            self.lib.ref_ds_free(h)

    def matvec_transposed(self, ds: HostData, a, rows=None, workers=1) -> np.ndarray:
        """linalg::matvec_transposed (linalg.cpp:46-109)."""
        h = self.to_handle(ds)
        try:
            rows = np.ascontiguousarray(rows if rows is not None else [], np.uint32)
            a = np.ascontiguousarray(a, np.float64)
            out = np.zeros(ds.n_features, np.float64)
            if self.lib.ref_matvec_transposed(h, _ptr(rows, C.c_uint32), len(rows), _ptr(a, _dbl),
                                              len(a), workers, _ptr(out, _dbl)) != 0:
                raise RuntimeError(self.err())
            return out
        finally:
            self.lib.ref_ds_free(h)

    def elementwise(self, op, a, b=None, scalar=0.0, workers=1) -> np.ndarray:
        """linalg::elementwise / ew_sigmoid (op 5) / ew_hinge_indicator (op 6)."""
        a = np.ascontiguousarray(a, np.float64)
        b = None if b is None else np.ascontiguousarray(b, np.float64)
        out = np.zeros(len(a), np.float64)
        if self.lib.ref_elementwise(int(op), _ptr(a, _dbl), None if b is None else _ptr(b, _dbl),
                                    len(a), scalar, workers, _ptr(out, _dbl)) != 0:
            raise RuntimeError(self.err())
        return out

    def axpy(self, w, alpha, g, workers=1) -> np.ndarray:
        w = np.array(w, np.float64)
        g = np.ascontiguousarray(g, np.float64)
        self.lib.ref_axpy(_ptr(w, _dbl), alpha, _ptr(g, _dbl), len(w), workers)
        return w

    def batch_gradient(self, ds: HostData, task, rows, w, workers=1) -> np.ndarray:
        h = self.to_handle(ds)
        try:
            rows = np.ascontiguousarray(rows if rows is not None else [], np.uint32)
            w = np.ascontiguousarray(w, np.float64)
            g = np.zeros(ds.n_features, np.float64)
            if self.lib.ref_batch_gradient(h, task, _ptr(rows, C.c_uint32), len(rows),
                                           _ptr(w, _dbl), workers, _ptr(g, _dbl)) != 0:
                raise RuntimeError(self.err())
            return g
        finally:
            self.lib.ref_ds_free(h)

    def epoch_batch(self, ds: HostData, task, w, alpha, workers=1):
        h = self.to_handle(ds)
        try:
            w = np.array(w, np.float64)
            norm = self.lib.ref_epoch_batch(h, task, _ptr(w, _dbl), alpha, workers)
            return w, norm
        finally:
            self.lib.ref_ds_free(h)

    def sync_train(self, ds: HostData, task, alpha, batch_b, epochs, seed, decay=1.0,
                   workers=1, shuffle=True, init=None, handle=None):
        """sync::train verbatim. Returns (model, losses, seconds, diverged)."""
        h = handle if handle is not None else self.to_handle(ds)
        try:
            d = ds.n_features
            model = np.zeros(d, np.float64)
            losses = np.zeros(epochs, np.float64)
            secs = np.zeros(epochs, np.float64)
            ran = _u64(0)
            div = _int(0)
            init_a = None if init is None else np.ascontiguousarray(init, np.float64)
            if self.lib.ref_sync_train(h, task, alpha, batch_b, epochs, decay, seed, workers,
                                       int(shuffle), _ptr(init_a, _dbl), _ptr(model, _dbl),
                                       _ptr(losses, _dbl), _ptr(secs, _dbl), C.byref(ran),
                                       C.byref(div)) != 0:
                raise ValueError(self.err())
            k = int(ran.value)
            return model, losses[:k], secs[:k], bool(div.value)
        finally:
            if handle is None:
                self.lib.ref_ds_free(h)

    def sync_train_dump(self, ds: HostData, task, alpha, batch_b, epochs, seed, decay=1.0,
                        workers=1, shuffle=True):
        h = self.to_handle(ds)
        try:
            models = np.zeros((epochs, ds.n_features), np.float64)
            losses = np.zeros(epochs, np.float64)
            if self.lib.ref_sync_train_dump(h, task, alpha, batch_b, epochs, decay, seed,
                                            workers, int(shuffle), _ptr(models, _dbl),
                                            _ptr(losses, _dbl)) != 0:
                raise ValueError(self.err())
            return models, losses
        finally:
            self.lib.ref_ds_free(h)

    def hogwild_train(self, ds: HostData, task, alpha, epochs, plan: str, workers=1,
                      group_size=32, circular_offsets=True, merge_period=1, dual=False,
                      decay=1.0, init=None, handle=None):
        """hogwild::train / numa_dual_train verbatim. Returns (model, losses, seconds, evals)."""
        h = handle if handle is not None else self.to_handle(ds)
        try:
            d = ds.n_features
            model = np.zeros(d, np.float64)
            losses = np.zeros(epochs, np.float64)
            secs = np.zeros(epochs, np.float64)
            evals = np.zeros(epochs, np.uint64)
            ran = _u64(0)
            init_a = None if init is None else np.ascontiguousarray(init, np.float64)
            if self.lib.ref_hogwild_train(h, task, alpha, epochs, decay, plan.encode(), workers,
                                          group_size, int(circular_offsets), merge_period,
                                          int(dual), _ptr(init_a, _dbl), _ptr(model, _dbl),
                                          _ptr(losses, _dbl), _ptr(secs, _dbl),
                                          _ptr(evals, _u64), C.byref(ran)) != 0:
                raise ValueError(self.err())
            k = int(ran.value)
            return model, losses[:k], secs[:k], evals[:k]
        finally:
            if handle is None:
                self.lib.ref_ds_free(h)

    def warpsim_epoch(self, ds: HostData, task, alpha, plan: str, warp_width=32, segment_size=8,
                      offsets=True, w=None):
        """warpsim::simulate_epoch (proj/src/simd_sim.cpp): returns (w, stats dict)."""
        h = self.to_handle(ds)
        try:
            w = np.zeros(ds.n_features) if w is None else np.array(w, np.float64)
            st = np.zeros(4, np.uint64)
            L = self.lib
            L.ref_warpsim_epoch.argtypes = [_vp, _int, _dbl, C.c_char_p, _u64, _u64, _int, _P(_dbl), _P(_u64)]
            if L.ref_warpsim_epoch(h, task, alpha, plan.encode(), warp_width, segment_size, int(offsets),
                                   _ptr(w, _dbl), _ptr(st, _u64)) != 0:
                raise ValueError(self.err())
            return w, {"attempted_updates": int(st[0]), "surviving_updates": int(st[1]),
                       "memory_transactions": int(st[2]), "micro_steps": int(st[3])}
        finally:
            self.lib.ref_ds_free(h)

    def harness_run(self, ds: HostData, engine, task, alpha, batch_b, epochs, plan=None, workers=1,
                    repetitions=1, seed=0, optimal_loss=None):
        """harness::run (proj/src/harness.cpp): (losses, epochs_to {10,5,2,1: epoch|None}, l_used)."""
        h = self.to_handle(ds)
        try:
            L = self.lib
            L.ref_harness_run.argtypes = [_vp, _int, _int, _dbl, _u64, _u64, C.c_char_p, _u64, _u64, _u64,
                                          _dbl, _P(_dbl), _P(_u64), _P(C.c_int64), _P(_dbl)]
            losses = np.zeros(epochs, np.float64)
            n = _u64(0)
            et = np.zeros(4, np.int64)
            lu = _dbl(0)
            if L.ref_harness_run(h, engine, task, alpha, batch_b, epochs, (plan or "").encode(), workers,
                                 repetitions, seed, float("nan") if optimal_loss is None else optimal_loss,
                                 _ptr(losses, _dbl), C.byref(n), _ptr(et, C.c_int64), C.byref(lu)) != 0:
                raise ValueError(self.err())
            return (losses[:int(n.value)], {t: (int(e) or None) for t, e in zip((10, 5, 2, 1), et)},
                    float(lu.value))
        finally:
            self.lib.ref_ds_free(h)

    def estimate_optimal_loss(self, ds: HostData, task, epochs):
        """harness::estimate_optimal_loss over the default probes' step-size grid,
        `epochs` batch-GD epochs each (cache cleared first)."""
        h = self.to_handle(ds)
        try:
            L = self.lib
            L.ref_estimate_optimal_loss.restype = _dbl
            L.ref_estimate_optimal_loss.argtypes = [_vp, _int, _u64]
            return float(L.ref_estimate_optimal_loss(h, task, epochs))
        finally:
            self.lib.ref_ds_free(h)

    def grid_search_alpha(self, ds: HostData, engine, task, batch_b, epochs, grid, plan=None, workers=1,
                          seed=0, optimal_loss=None):
        """harness::grid_search_alpha: (best_alpha, converged, l_used)."""
        h = self.to_handle(ds)
        try:
            L = self.lib
            L.ref_grid_search_alpha.argtypes = [_vp, _int, _int, _u64, _u64, C.c_char_p, _u64, _u64, _dbl,
                                                _P(_dbl), _u64, _P(_dbl), _P(_int), _P(_dbl)]
            g = np.ascontiguousarray(grid, np.float64)
            best, conv, lu = _dbl(0), _int(0), _dbl(0)
            if L.ref_grid_search_alpha(h, engine, task, batch_b, epochs, (plan or "").encode(), workers, seed,
                                       float("nan") if optimal_loss is None else optimal_loss,
                                       _ptr(g, _dbl), len(g), C.byref(best), C.byref(conv),
                                       C.byref(lu)) != 0:
                raise ValueError(self.err())
            return float(best.value), bool(conv.value), float(lu.value)
        finally:
            self.lib.ref_ds_free(h)

    def count_transactions(self, lane_streams, segment_size):
        """warpsim::count_transactions (proj/src/simd_sim.cpp:89-104)."""
        flat = np.ascontiguousarray(np.concatenate([np.asarray(s, np.uint64) for s in lane_streams])
                                    if lane_streams else np.zeros(0, np.uint64), np.uint64)
        off = np.zeros(len(lane_streams) + 1, np.uint64)
        off[1:] = np.cumsum([len(s) for s in lane_streams])
        L = self.lib
        L.ref_count_transactions.restype = _u64
        L.ref_count_transactions.argtypes = [_P(_u64), _P(_u64), _u64, _u64]
        return int(L.ref_count_transactions(_ptr(flat, _u64), _ptr(off, _u64), len(lane_streams),
                                            segment_size))

    def merge_models(self, replicas: np.ndarray, weights=None) -> np.ndarray:
        reps = np.ascontiguousarray(replicas, np.float64)
        r, d = reps.shape
        out = np.zeros(d, np.float64)
        wts = None if weights is None else np.ascontiguousarray(weights, np.float64)
        self.lib.ref_merge_models(_ptr(reps.ravel(), _dbl), r, d, _ptr(wts, _dbl),
                                  _ptr(out, _dbl))
        return out


_ORACLE = None
_REF = None


def oracle() -> Oracle:
    global _ORACLE
    if _ORACLE is None:
        _ORACLE = Oracle()
    return _ORACLE


def reference_available() -> bool:
    return os.path.exists(REF_SO)


def reference() -> Reference:
    global _REF
    if _REF is None:
        _REF = Reference()
    return _REF
