"""Python mirror of the reference's C++ interface (proj/include/sgdbench/*.hpp).

Names, argument meaning and error behaviour follow the reference so that the
parity tests read like its own tests; every call goes through the C-ABI of
``include/sgdb.h`` (libsgdb_b200.so). Training runs on the GPU; the host
helpers (fixtures, LIBSVM parsing, layouts, assignment, plan grammar, the
mini-batch schedule) are host C++ in the same library.

    reference                         here
    ------------------------------    ------------------------------------
    sgdbench::Dataset                 Dataset (numpy arrays)
    fixtures::*_classification        fixtures.dense_classification / ...
    parse_libsvm / convert_layout     parse_libsvm / convert_layout / ...
    sync::train / batch_gradient      sync.train / sync.batch_gradient
    hogwild::train / numa_dual_train  hogwild.train / hogwild.numa_dual_train
    dataset_loss                      dataset_loss
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Callable, Optional, Sequence

import numpy as np

from . import _lib as L
from ._lib import check


# ---- enums -------------------------------------------------------------------
class Task(IntEnum):          # glm.hpp:15
    LR = 0
    SVM = 1


class Layout(IntEnum):        # dataset.hpp:13
    DenseRowMajor = 0
    DenseColMajor = 1
    Csr = 2
    PaddedDense = 3


class Strategy(IntEnum):      # dataset.hpp:133
    RoundRobin = 0
    Chunk = 1


class AccessPath(IntEnum):    # async_engine.hpp:17
    RowRR = 0
    RowCh = 1
    ColRR = 2
    ColCh = 3


class ModelReplication(IntEnum):  # async_engine.hpp:21
    Kernel = 0
    Block = 1
    Thread = 2
    Example = 3


def _lib():
    return L.load()


def _dptr(a):
    return None if a is None or a.size == 0 else a.ctypes.data_as(L.P(L.dbl))


def _u32ptr(a):
    return None if a is None or a.size == 0 else a.ctypes.data_as(L.P(L.u32))


def _u64ptr(a):
    return None if a is None or a.size == 0 else a.ctypes.data_as(L.P(L.u64))


# ---- Dataset -------------------------------------------------------------------
@dataclass
class Dataset:
    """sgdbench::Dataset (dataset.hpp:42-61) with numpy storage."""

    n_examples: int = 0
    n_features: int = 0
    layout: Layout = Layout.Csr
    labels: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float64))
    values: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float64))
    indices: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    row_offsets: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    padded_width: int = 0

    def __post_init__(self):
        self.layout = Layout(int(self.layout))
        self.labels = np.ascontiguousarray(self.labels, np.float64)
        self.values = np.ascontiguousarray(self.values, np.float64)
        self.indices = np.ascontiguousarray(self.indices, np.uint32)
        self.row_offsets = np.ascontiguousarray(self.row_offsets, np.uint64)

    def pad_sentinel(self) -> int:
        return int(self.n_features)

    def is_sparse_layout(self) -> bool:
        return self.layout in (Layout.Csr, Layout.PaddedDense)

    def view(self) -> L.DatasetView:
        """Borrowed C view (the arrays must outlive it)."""
        v = L.DatasetView()
        v.n_examples = self.n_examples
        v.n_features = self.n_features
        v.layout = int(self.layout)
        v.labels = _dptr(self.labels)
        v.values = _dptr(self.values)
        v.n_values = self.values.size
        v.indices = _u32ptr(self.indices)
        v.n_indices = self.indices.size
        v.row_offsets = _u64ptr(self.row_offsets)
        v.n_row_offsets = self.row_offsets.size
        v.padded_width = self.padded_width
        return v

    def nnz(self) -> int:
        if self.layout == Layout.Csr:
            return int(self.values.size)
        if self.layout == Layout.PaddedDense:
            return int(np.count_nonzero(self.indices != self.n_features))
        return int(np.count_nonzero(self.values))

    def validate(self) -> None:
        v = self.view()
        check(_lib().sgdb_validate_dataset(C.byref(v)))

    @staticmethod
    def _from_handle(h) -> "Dataset":
        lib = _lib()
        v = L.DatasetView()
        try:
            check(lib.sgdb_host_dataset_view(h, C.byref(v)))

            def arr(ptr, n, dt):
                if n == 0 or not ptr:
                    return np.zeros(0, dt)
                return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dt, copy=True)

            return Dataset(int(v.n_examples), int(v.n_features), Layout(v.layout),
                           arr(v.labels, v.n_examples, np.float64),
                           arr(v.values, v.n_values, np.float64),
                           arr(v.indices, v.n_indices, np.uint32),
                           arr(v.row_offsets, v.n_row_offsets, np.uint64), int(v.padded_width))
        finally:
            lib.sgdb_host_dataset_free(h)

    def rounded_f32(self) -> "Dataset":
        """Copy with values rounded to fp32 (the device storage precision)."""
        return Dataset(self.n_examples, self.n_features, self.layout, self.labels.copy(),
                       self.values.astype(np.float32).astype(np.float64), self.indices.copy(),
                       self.row_offsets.copy(), self.padded_width)


class ParseError(L.ParseError):
    pass


def parse_libsvm(text, declared_d: Optional[int] = None) -> Dataset:
    """parse_libsvm (dataset.cpp:167-230); raises _lib.ParseError with .line_number."""
    b = text.encode() if isinstance(text, str) else bytes(text)
    h = L.vp()
    line = L.u64(0)
    st = _lib().sgdb_parse_libsvm(b, len(b), -1 if declared_d is None else int(declared_d),
                                  C.byref(h), C.byref(line))
    check(st, int(line.value))
    return Dataset._from_handle(h)


def write_libsvm(ds: Dataset) -> str:
    v = ds.view()
    n = L.u64(0)
    check(_lib().sgdb_write_libsvm(C.byref(v), None, 0, C.byref(n)))
    buf = C.create_string_buffer(int(n.value) + 1)
    check(_lib().sgdb_write_libsvm(C.byref(v), buf, n.value, C.byref(n)))
    return buf.raw[: n.value].decode()


def save_binary(ds: Dataset, path: str) -> None:
    v = ds.view()
    check(_lib().sgdb_save_binary(C.byref(v), path.encode()))


def load_binary(path: str) -> Dataset:
    h = L.vp()
    check(_lib().sgdb_load_binary(path.encode(), C.byref(h)))
    return Dataset._from_handle(h)


def convert_layout(ds: Dataset, target: Layout, max_dense_bytes: int = 0) -> Dataset:
    v = ds.view()
    h = L.vp()
    check(_lib().sgdb_convert_layout(C.byref(v), int(target), max_dense_bytes, C.byref(h)))
    return Dataset._from_handle(h)


def assign(n: int, workers: int, strategy: Strategy, k: int) -> list[list[int]]:
    """assign (dataset.cpp:470-503): per-worker ordered id lists."""
    total = L.u64(0)
    check(_lib().sgdb_assign(n, workers, int(strategy), k, None, None, C.byref(total)))
    ids = np.zeros(int(total.value), np.uint32)
    offs = np.zeros(workers + 1, np.uint64)
    check(_lib().sgdb_assign(n, workers, int(strategy), k, _u32ptr(ids), _u64ptr(offs),
                             C.byref(total)))
    return [ids[int(offs[w]):int(offs[w + 1])].tolist() for w in range(workers)]


class fixtures:  # noqa: N801 — namespace mirror of sgdbench::fixtures
    @staticmethod
    def dense_classification(n, d, seed, label_noise=0.1) -> Dataset:
        h = L.vp()
        check(_lib().sgdb_fixture_dense(n, d, seed, label_noise, C.byref(h)))
        return Dataset._from_handle(h)

    @staticmethod
    def sparse_classification(n, d, avg_nnz, seed, label_noise=0.1) -> Dataset:
        h = L.vp()
        check(_lib().sgdb_fixture_sparse(n, d, avg_nnz, seed, label_noise, C.byref(h)))
        return Dataset._from_handle(h)


# ---- hyperparameters, plans, traces ---------------------------------------------
@dataclass
class Hyperparams:  # glm.hpp:22-35
    alpha: float = 0.01
    batch_b: int = 1
    epochs: int = 10
    task: Task = Task.LR
    step_decay: float = 1.0

    def step_size(self, epoch: int) -> float:
        a = self.alpha
        for _ in range(1, epoch):
            a *= self.step_decay
        return a

    def to_c(self, task=None) -> L.Hyper:
        return L.Hyper(self.alpha, self.batch_b, self.epochs,
                       int(self.task if task is None else task), self.step_decay)


@dataclass
class ExecutionPlan:  # async_engine.hpp:25-33
    access_path: AccessPath = AccessPath.RowCh
    model_replication: ModelReplication = ModelReplication.Kernel
    data_replication_k: int = 0
    workers: int = 1
    group_size: int = 32
    circular_offsets: bool = True
    merge_period_epochs: int = 1
    lanes_per_worker: int = 0  # device knob: 0 = auto

    def to_c(self) -> L.Plan:
        return L.Plan(int(self.access_path), int(self.model_replication), self.data_replication_k,
                      self.workers, self.group_size, int(self.circular_offsets),
                      self.merge_period_epochs, self.lanes_per_worker)

    @staticmethod
    def from_c(p: L.Plan) -> "ExecutionPlan":
        return ExecutionPlan(AccessPath(p.access_path), ModelReplication(p.replication),
                             int(p.data_replication_k), int(p.workers), int(p.group_size),
                             bool(p.circular_offsets), int(p.merge_period_epochs),
                             int(p.lanes_per_worker))


def parse_plan(text: str) -> ExecutionPlan:
    p = L.Plan()
    check(_lib().sgdb_parse_plan(text.encode(), C.byref(p)))
    return ExecutionPlan.from_c(p)


def plan_to_string(plan: ExecutionPlan) -> str:
    buf = C.create_string_buffer(64)
    p = plan.to_c()
    check(_lib().sgdb_plan_to_string(C.byref(p), buf, 64))
    return buf.value.decode()


def validate_plan(plan: ExecutionPlan, ds: Dataset) -> None:
    p = plan.to_c()
    check(_lib().sgdb_validate_plan(C.byref(p), int(ds.layout)))


@dataclass
class EpochRecord:  # trace.hpp:21-25
    epoch: int
    loss: float
    seconds: float


@dataclass
class LossTrace:  # trace.hpp:27-49
    epochs: list = field(default_factory=list)
    diverged: bool = False
    divergence_note: str = ""

    def losses(self) -> list[float]:
        return [e.loss for e in self.epochs]

    def final_loss(self) -> float:
        return self.epochs[-1].loss if self.epochs else 0.0

    def min_loss(self) -> float:
        return min((e.loss for e in self.epochs), default=0.0)

    def total_seconds(self) -> float:
        return sum(e.seconds for e in self.epochs)


class Schedule:
    """sync::train's mini-batch schedule: mt19937_64(seed) + std::shuffle per epoch."""

    def __init__(self, seed: int, n: int, shuffle: bool = True):
        self.n = n
        self._h = L.vp()
        check(_lib().sgdb_schedule_create(seed, n, int(shuffle), C.byref(self._h)))

    def next(self) -> np.ndarray:
        out = np.zeros(self.n, np.uint32)
        check(_lib().sgdb_schedule_next(self._h, _u32ptr(out)))
        return out

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                _lib().sgdb_schedule_free(self._h)
                self._h = None
        except Exception:  # interpreter teardown
            pass


# ---- device objects ---------------------------------------------------------------
class Device:
    """A device context: CUDA device + the stream all ops are queued on."""

    def __init__(self, ordinal: int = 0, stream: Optional[int] = None):
        """stream: a CUDA stream handle to queue every op on (e.g.
        torch.cuda.current_stream().cuda_stream); handle 0 — torch's default
        stream — means the legacy default stream (cudaStreamLegacy), not
        "create one". None: the context creates its own stream."""
        self._h = L.vp()
        if stream is not None and int(stream) == 0:
            stream = 1  # cudaStreamLegacy
        check(_lib().sgdb_ctx_create(ordinal, stream, C.byref(self._h)))
        self._allreduce_cb = None
        self.ordinal = ordinal

    @property
    def handle(self):
        return self._h

    @property
    def stream(self) -> int:
        s = L.vp()
        check(_lib().sgdb_ctx_stream(self._h, C.byref(s)))
        return int(s.value or 0)

    def synchronize(self):
        check(_lib().sgdb_ctx_synchronize(self._h))

    def launch_count(self) -> int:
        n = L.u64(0)
        check(_lib().sgdb_ctx_launch_count(self._h, C.byref(n)))
        return int(n.value)

    def set_profiling(self, enable: bool) -> None:
        """Per-launch CUDA-event timing of the library's kernels (clears records)."""
        check(_lib().sgdb_ctx_set_profiling(self._h, int(enable)))

    def kernel_stats(self) -> dict:
        """{kernel name: (launches, total ms)} since profiling was enabled."""
        out, n = {}, L.u64(0)
        check(_lib().sgdb_ctx_kernel_stats(self._h, 0, None, 0, None, None, C.byref(n)))
        for i in range(int(n.value)):
            name = C.create_string_buffer(128)
            cnt, ms = L.u64(0), L.dbl(0)
            check(_lib().sgdb_ctx_kernel_stats(self._h, i, name, 128, C.byref(cnt), C.byref(ms),
                                               None))
            out[name.value.decode()] = (int(cnt.value), float(ms.value))
        return out

    def resident_workers(self, dds: "DeviceDataset", lanes: int = 0) -> int:
        """Lane groups the Hogwild kernels keep resident for `lanes` lanes/worker."""
        n = L.u64(0)
        check(_lib().sgdb_ctx_resident_workers(self._h, dds.handle, lanes, C.byref(n)))
        return int(n.value)

    def set_allreduce(self, fn: Optional[Callable[[int, int, int, int], None]]):
        """fn(device_ptr, count, dtype(0=f32,1=f64), stream) sum-reduces in place."""
        if fn is None:
            self._allreduce_cb = None
            check(_lib().sgdb_ctx_set_allreduce(self._h, L.ALLREDUCE_FN(), None))
            return

        def tramp(_user, ptr, count, dtype, stream):
            try:
                fn(int(ptr), int(count), int(dtype), int(stream or 0))
                return 0
            except Exception:  # reported as a failed status by the engine
                import traceback
                traceback.print_exc()
                return 1

        self._allreduce_cb = L.ALLREDUCE_FN(tramp)
        check(_lib().sgdb_ctx_set_allreduce(self._h, self._allreduce_cb, None))

    @staticmethod
    def nccl_unique_id() -> bytes:
        """A fresh 128-byte NCCL id (rank 0 creates it, the host distributes it)."""
        buf = C.create_string_buffer(128)
        check(_lib().sgdb_nccl_get_unique_id(buf))
        return buf.raw

    def init_nccl(self, nranks: int, rank: int, uid: bytes) -> None:
        """Attach an in-library NCCL communicator (sgdb_ctx_init_nccl): the
        engine's gradient / model / loss reductions run as ncclAllReduce on
        this context's stream."""
        if len(uid) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        check(_lib().sgdb_ctx_init_nccl(self._h, nranks, rank, uid))

    def world(self) -> tuple[int, int]:
        """(rank, nranks) of the attached communicator ((0, 1) without one)."""
        r, n = L.i32(0), L.i32(0)
        check(_lib().sgdb_ctx_world(self._h, C.byref(r), C.byref(n)))
        return int(r.value), int(n.value)

    def close(self):
        if getattr(self, "_h", None):
            _lib().sgdb_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter teardown
            pass


_DEFAULT_EXACT: Optional[bool] = None


def set_default_precision(precision: str) -> None:
    """'fp32' (fused fp32 kernels, the default) or 'exact' (SGDB_UPLOAD_EXACT_FP64:
    fp64 in the reference's operation order, bit-identical results) for
    datasets uploaded without an explicit ``exact=``. The initial default
    comes from the SGDB_PRECISION environment variable."""
    global _DEFAULT_EXACT
    if precision not in ("fp32", "exact"):
        raise ValueError("precision must be 'fp32' or 'exact'")
    _DEFAULT_EXACT = precision == "exact"


def default_exact() -> bool:
    global _DEFAULT_EXACT
    if _DEFAULT_EXACT is None:
        import os
        _DEFAULT_EXACT = os.environ.get("SGDB_PRECISION", "fp32") in ("exact", "fp64")
    return _DEFAULT_EXACT


class DeviceDataset:
    """Device-resident dataset (fp32 storage; plus fp64 values in the exact
    mode), optionally a row shard."""

    def __init__(self, dev: Device, ds: Optional[Dataset], row_base: int = 0, n_global: int = 0,
                 exact: Optional[bool] = None, _handle=None, padded: bool = False):
        """padded=True (CSR input): the slot-major padded copy is built on the
        device (SGDB_UPLOAD_PADDED) and the dataset serves the column access
        paths like a PaddedDense upload."""
        self.dev = dev
        self.host = ds
        self.exact = bool(default_exact() if exact is None else exact) if _handle is None else False
        if _handle is not None:
            self._h = _handle
        else:
            self._h = L.vp()
            v = ds.view()
            flags = (L.SGDB_UPLOAD_EXACT_FP64 if self.exact else 0) | (L.SGDB_UPLOAD_PADDED if padded else 0)
            check(_lib().sgdb_dataset_upload_ex(dev.handle, C.byref(v), row_base, n_global, flags,
                                                C.byref(self._h)))
        n, d, nnz, rb, ng = (L.u64() for _ in range(5))
        check(_lib().sgdb_dataset_shape(self._h, C.byref(n), C.byref(d), C.byref(nnz),
                                        C.byref(rb), C.byref(ng)))
        self.n_local, self.n_features, self.nnz = int(n.value), int(d.value), int(nnz.value)
        self.row_base, self.n_global = int(rb.value), int(ng.value)
        self.layout = (Layout.PaddedDense if padded else ds.layout) if ds is not None else Layout.DenseRowMajor

    @classmethod
    def generate_dense(cls, dev: Device, n_local: int, d: int, seed: int, row_base: int = 0,
                       n_global: int = 0, label_noise: float = 0.1) -> "DeviceDataset":
        """K9: rows [row_base, row_base+n_local) of the Philox dense classification
        dataset generated on the device (sgdb_dataset_generate_dense)."""
        h = L.vp()
        check(_lib().sgdb_dataset_generate_dense(dev.handle, n_local, d, row_base, n_global, seed,
                                                 label_noise, C.byref(h)))
        return cls(dev, None, _handle=h)

    @property
    def handle(self):
        return self._h

    def read_dense(self, row0: int, nrows: int):
        """(values[nrows, d] float32, labels[nrows] float32) of a dense device dataset."""
        vals = np.zeros((nrows, self.n_features), np.float32)
        labs = np.zeros(nrows, np.float32)
        check(_lib().sgdb_dataset_read_dense(self.dev.handle, self._h, row0, nrows,
                                             vals.ctypes.data, labs.ctypes.data))
        return vals, labs

    def sweep_bytes(self) -> int:
        b = L.u64(0)
        check(_lib().sgdb_dataset_sweep_bytes(self._h, C.byref(b)))
        return int(b.value)

    def refresh_f32(self, values=None, labels=None, indices=None, row_offsets32=None,
                    device: Optional[Device] = None):
        """Async H2D re-copy of fp32 host arrays (pinned torch tensors or numpy), on
        `device`'s stream (default: the dataset's own context) — pass a context on a
        copy stream to overlap the transfer with epochs on another buffer."""
        def p(a):
            if a is None:
                return None
            return a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data
        ctx = (device or self.dev).handle
        check(_lib().sgdb_dataset_refresh_f32(ctx, self._h, p(values), p(labels), p(indices),
                                              p(row_offsets32)))

    def refresh_idx16(self, indices16, device: Optional[Device] = None):
        """Async H2D copy of 16-bit column ids (d <= 65536), widened on the device
        (sgdb_dataset_refresh_idx16); same stream rules as refresh_f32."""
        ptr = indices16.data_ptr() if hasattr(indices16, "data_ptr") else indices16.ctypes.data
        check(_lib().sgdb_dataset_refresh_idx16((device or self.dev).handle, self._h, ptr))

    def close(self):
        if getattr(self, "_h", None):
            _lib().sgdb_dataset_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter teardown
            pass


class DeviceModel:
    """Device model: fp32 working copy (d+1, guard slot) + fp64 master."""

    def __init__(self, dev: Device, d: int, init=None):
        self.dev = dev
        self.d = d
        self._h = L.vp()
        w = None if init is None else np.ascontiguousarray(init, np.float64)
        check(_lib().sgdb_model_create(dev.handle, d, _dptr(w), C.byref(self._h)))

    @property
    def handle(self):
        return self._h

    def get(self) -> np.ndarray:
        out = np.zeros(self.d, np.float64)
        check(_lib().sgdb_model_get(self.dev.handle, self._h, _dptr(out)))
        return out

    def set(self, w) -> None:
        w = np.ascontiguousarray(w, np.float64)
        check(_lib().sgdb_model_set(self.dev.handle, self._h, _dptr(w)))

    def device_ptrs(self) -> tuple[int, int]:
        a, b = L.vp(), L.vp()
        check(_lib().sgdb_model_device_ptrs(self._h, C.byref(a), C.byref(b)))
        return int(a.value), int(b.value)

    def close(self):
        if getattr(self, "_h", None):
            _lib().sgdb_model_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter teardown
            pass


# ---- device ops (layer 1) -------------------------------------------------------------
def sync_epoch(dds: DeviceDataset, model: DeviceModel, task: Task, alpha: float,
               order: Optional[np.ndarray], batch_b: int, check_finite: bool = True) -> bool:
    """One synchronous epoch. check_finite=False leaves the epoch fully
    asynchronous on the device stream (no flag read-back; returns True)."""
    o = None if order is None else np.ascontiguousarray(order, np.uint32)
    f = L.i32(1)
    check(_lib().sgdb_sync_epoch(dds.dev.handle, dds.handle, model.handle, int(task), alpha,
                                 _u32ptr(o), batch_b, C.byref(f) if check_finite else None))
    return bool(f.value)


def hogwild_epoch(dds: DeviceDataset, model: DeviceModel, task: Task, alpha: float,
                  plan: ExecutionPlan, segment: int = 0, segments: int = 1) -> int:
    """One Hogwild epoch (or segment `segment` of `segments`, see
    sgdb_hogwild_segment); returns the number of example evaluations."""
    p = plan.to_c()
    ev = L.u64(0)
    check(_lib().sgdb_hogwild_segment(dds.dev.handle, dds.handle, model.handle, int(task), alpha,
                                      C.byref(p), int(segment), int(segments), C.byref(ev)))
    return int(ev.value)


def device_loss(dds: DeviceDataset, model: DeviceModel, task: Task) -> float:
    out = L.dbl(0)
    check(_lib().sgdb_loss(dds.dev.handle, dds.handle, model.handle, int(task), C.byref(out)))
    return float(out.value)


def models_average(dev: Device, models: Sequence[DeviceModel], out: DeviceModel,
                   weights=None, refresh: bool = False) -> None:
    arr = (L.vp * len(models))(*[m.handle for m in models])
    w = None if weights is None else np.ascontiguousarray(weights, np.float64)
    check(_lib().sgdb_models_average(dev.handle, arr, len(models), _dptr(w), out.handle,
                                     int(refresh)))


def generate_hidden_model(seed: int, d: int) -> np.ndarray:
    """w_true of the device generator (sgdb_generate_hidden_model)."""
    out = np.zeros(d, np.float64)
    check(_lib().sgdb_generate_hidden_model(seed, d, _dptr(out)))
    return out


_DEFAULT_DEVICE: Optional[Device] = None


def default_device() -> Device:
    global _DEFAULT_DEVICE
    if _DEFAULT_DEVICE is None:
        _DEFAULT_DEVICE = Device(0)
    return _DEFAULT_DEVICE


def _as_device_dataset(ds, device) -> DeviceDataset:
    if isinstance(ds, DeviceDataset):
        return ds
    return DeviceDataset(device or default_device(), ds)


def dataset_loss(task: Task, ds, w, device: Optional[Device] = None) -> float:
    """dataset_loss (glm.cpp:85-94) on the device, fp64 accumulation."""
    dds = _as_device_dataset(ds, device)
    w = np.ascontiguousarray(w, np.float64)
    if w.size != dds.n_features:
        raise ValueError("model/dataset dim mismatch")
    m = DeviceModel(dds.dev, dds.n_features, w)
    return device_loss(dds, m, task)


def _options_struct(o, shuffle: bool):
    keep = []
    c = L.TrainOptions()
    c.workers = getattr(o, "workers", 1) if o else 1
    c.shuffle = int(shuffle)
    c.max_seconds = float(o.max_seconds) if o else 0.0
    if o is not None and o.initial_model is not None and len(o.initial_model):
        init = np.ascontiguousarray(o.initial_model, np.float64)
        keep.append(init)
        c.initial_model = _dptr(init)
        c.initial_model_len = init.size
    if o is not None and o.clock is not None:
        cb = L.CLOCK_FN(lambda _u: float(o.clock()))
        keep.append(cb)
        c.clock = cb
    if o is not None and o.epoch_hook is not None:
        hb = L.HOOK_FN(lambda _u, e, loss: o.epoch_hook(int(e), float(loss)))
        keep.append(hb)
        c.epoch_hook = hb
    return c, keep


def _trace(epochs: int, with_evals: bool):
    recs = (L.EpochRecord * max(1, epochs))()
    evals = np.zeros(max(1, epochs), np.uint64) if with_evals else None
    t = L.Trace()
    t.epochs = C.cast(recs, L.P(L.EpochRecord))
    t.evals_per_epoch = _u64ptr(evals) if with_evals else None
    t.capacity = epochs
    return t, recs, evals


def _loss_trace(t, recs) -> LossTrace:
    lt = LossTrace([EpochRecord(int(recs[i].epoch), float(recs[i].loss), float(recs[i].seconds))
                    for i in range(int(t.count))], bool(t.diverged),
                   t.divergence_note.decode(errors="replace"))
    return lt


# ---- sync_engine.hpp ------------------------------------------------------------------
@dataclass
class TrainOptions:  # sync_engine.hpp:15-25
    workers: int = 1
    shuffle: bool = True
    clock: Optional[Callable[[], float]] = None
    epoch_hook: Optional[Callable[[int, float], None]] = None
    max_seconds: float = 0.0
    initial_model: Optional[Sequence[float]] = None


@dataclass
class TrainResult:
    model: np.ndarray
    trace: LossTrace


class sync:  # noqa: N801 — namespace mirror of sgdbench::sync
    TrainOptions = TrainOptions
    TrainResult = TrainResult

    @staticmethod
    def train(task: Task, ds, hyper: Hyperparams, seed: int,
              options: Optional[TrainOptions] = None, device: Optional[Device] = None) -> TrainResult:
        """sync::train (sync_engine.cpp:56-121) with the epoch work on the GPU."""
        if isinstance(ds, Dataset) and ds.n_examples == 0:
            raise ValueError("cannot train on an empty dataset")
        dds = _as_device_dataset(ds, device)
        o = options or TrainOptions()
        c, keep = _options_struct(o, o.shuffle)
        t, recs, _ = _trace(hyper.epochs, False)
        model = np.zeros(dds.n_features, np.float64)
        h = hyper.to_c(task)
        check(_lib().sgdb_sync_train(dds.dev.handle, dds.handle, C.byref(h), seed, C.byref(c),
                                     _dptr(model), C.byref(t)))
        del keep
        return TrainResult(model, _loss_trace(t, recs))

    @staticmethod
    def batch_gradient(task: Task, ds, rows, w, workers: int = 1, transposed=None,
                       device: Optional[Device] = None) -> np.ndarray:
        """sync::batch_gradient (sync_engine.cpp:22-42); rows empty = all examples."""
        dds = _as_device_dataset(ds, device)
        w = np.ascontiguousarray(w, np.float64)
        if w.size != dds.n_features:
            raise ValueError("matvec: dimension mismatch")
        r = np.ascontiguousarray(rows if rows is not None else [], np.uint32)
        g = np.zeros(dds.n_features, np.float64)
        check(_lib().sgdb_batch_gradient(dds.dev.handle, dds.handle, int(task), _u32ptr(r),
                                         r.size, _dptr(w), int(transposed is not None),
                                         _dptr(g)))
        return g

    @staticmethod
    def epoch_batch(task: Task, ds, w: np.ndarray, alpha: float, workers: int = 1,
                    device: Optional[Device] = None) -> float:
        """sync::epoch_batch (sync_engine.cpp:44-54): updates w in place, returns ||g||."""
        dds = _as_device_dataset(ds, device)
        m = DeviceModel(dds.dev, dds.n_features, w)
        norm = L.dbl(0)
        check(_lib().sgdb_epoch_batch(dds.dev.handle, dds.handle, m.handle, int(task), alpha,
                                      C.byref(norm)))
        w[:] = m.get()
        return float(norm.value)


# ---- linalg.hpp ---------------------------------------------------------------------------
class ElementwiseOp(IntEnum):  # linalg.hpp:40 (+ the two fused ops)
    Mul = 0
    Div = 1
    Exp = 2
    Neg = 3
    AddScalar = 4
    Sigmoid = 5
    HingeIndicator = 6


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, np.float64)


class linalg:  # noqa: N801 — namespace mirror of sgdbench::linalg (linalg.hpp:23-58)
    """The §4 operator API on the device. `workers` is accepted for signature
    parity and ignored (the device decides its own parallelism); results follow
    the reference's summation order (see include/sgdb.h)."""

    @staticmethod
    def matvec(ds, v, rows=None, workers: int = 1, device: Optional[Device] = None) -> np.ndarray:
        """out_p = x_{rows[p]} . v (linalg.cpp:30-44)."""
        dds = _as_device_dataset(ds, device)
        v = _f64(v)
        r = np.ascontiguousarray(rows if rows is not None else [], np.uint32)
        out = np.zeros(r.size if r.size else dds.n_global, np.float64)
        check(_lib().sgdb_matvec(dds.dev.handle, dds.handle, _u32ptr(r), r.size, _dptr(v), v.size,
                                 _dptr(out)))
        return out

    @staticmethod
    def matvec_transposed(ds, a, rows=None, workers: int = 1,
                          device: Optional[Device] = None) -> np.ndarray:
        """X^T a over the rows, `a` indexed by position (linalg.cpp:46-109)."""
        dds = _as_device_dataset(ds, device)
        a = _f64(a)
        r = np.ascontiguousarray(rows if rows is not None else [], np.uint32)
        out = np.zeros(dds.n_features, np.float64)
        check(_lib().sgdb_matvec_transposed(dds.dev.handle, dds.handle, _u32ptr(r), r.size,
                                            _dptr(a), a.size, _dptr(out)))
        return out

    @staticmethod
    def elementwise(op: ElementwiseOp, a, b=None, scalar: float = 0.0, workers: int = 1,
                    device: Optional[Device] = None) -> np.ndarray:
        """elementwise (linalg.cpp:167-177); binary ops require equal lengths."""
        dev = device or default_device()
        a = _f64(a)
        binary = op in (ElementwiseOp.Mul, ElementwiseOp.Div)
        if binary:
            b = _f64(b)
            if b.size != a.size:
                name = "ew_mul" if op == ElementwiseOp.Mul else "ew_div"
                raise ValueError(f"{name}: length mismatch")
        out = np.zeros(a.size, np.float64)
        check(_lib().sgdb_elementwise(dev.handle, int(op), _dptr(a), _dptr(b) if binary else None,
                                      a.size, float(scalar), _dptr(out)))
        return out

    @staticmethod
    def ew_mul(a, b, workers: int = 1, device=None):
        return linalg.elementwise(ElementwiseOp.Mul, a, b, device=device)

    @staticmethod
    def ew_div(a, b, workers: int = 1, device=None):
        return linalg.elementwise(ElementwiseOp.Div, a, b, device=device)

    @staticmethod
    def ew_exp(a, workers: int = 1, device=None):
        return linalg.elementwise(ElementwiseOp.Exp, a, device=device)

    @staticmethod
    def ew_neg(a, workers: int = 1, device=None):
        return linalg.elementwise(ElementwiseOp.Neg, a, device=device)

    @staticmethod
    def ew_add_scalar(s: float, a, workers: int = 1, device=None):
        return linalg.elementwise(ElementwiseOp.AddScalar, a, scalar=s, device=device)

    @staticmethod
    def ew_sigmoid(a, workers: int = 1, device=None):
        return linalg.elementwise(ElementwiseOp.Sigmoid, a, device=device)

    @staticmethod
    def ew_hinge_indicator(a, workers: int = 1, device=None):
        return linalg.elementwise(ElementwiseOp.HingeIndicator, a, device=device)

    @staticmethod
    def axpy(w: np.ndarray, alpha: float, g, workers: int = 1, device=None) -> None:
        """w <- w - alpha g in place (linalg.cpp:179-183)."""
        dev = device or default_device()
        g = _f64(g)
        if not (isinstance(w, np.ndarray) and w.dtype == np.float64 and w.flags.c_contiguous):
            raise TypeError("axpy: w must be a contiguous float64 array (updated in place)")
        if w.size != g.size:
            raise ValueError("axpy: length mismatch")
        check(_lib().sgdb_axpy(dev.handle, _dptr(w), float(alpha), _dptr(g), w.size))


# ---- async_engine.hpp -------------------------------------------------------------------
@dataclass
class Options:  # async_engine.hpp:77-82
    clock: Optional[Callable[[], float]] = None
    epoch_hook: Optional[Callable[[int, float], None]] = None
    max_seconds: float = 0.0
    initial_model: Optional[Sequence[float]] = None


@dataclass
class Result:
    model: np.ndarray
    trace: LossTrace
    evals_per_epoch: list


class hogwild:  # noqa: N801 — namespace mirror of sgdbench::hogwild
    Options = Options
    Result = Result

    @staticmethod
    def _run(fn_name, task, ds, hyper, plan, seed, options, device):
        if isinstance(ds, Dataset):
            validate_plan(plan, ds)
            if ds.n_examples == 0:
                raise ValueError("cannot train on an empty dataset")
        dds = _as_device_dataset(ds, device)
        o = options or Options()
        c, keep = _options_struct(o, True)
        t, recs, evals = _trace(hyper.epochs, True)
        model = np.zeros(dds.n_features, np.float64)
        h = hyper.to_c(task)
        p = plan.to_c()
        check(getattr(_lib(), fn_name)(dds.dev.handle, dds.handle, C.byref(h), C.byref(p), seed,
                                       C.byref(c), _dptr(model), C.byref(t)))
        del keep
        n = int(t.count)
        return Result(model, _loss_trace(t, recs), [int(x) for x in evals[:n]])

    @staticmethod
    def train(task: Task, ds, hyper: Hyperparams, plan: ExecutionPlan, seed: int = 0,
              options: Optional[Options] = None, device: Optional[Device] = None) -> Result:
        """hogwild::train (async_engine.cpp:425-460): the GPU Hogwild kernels."""
        return hogwild._run("sgdb_hogwild_train", task, ds, hyper, plan, seed, options, device)

    @staticmethod
    def numa_dual_train(task: Task, ds, hyper: Hyperparams, plan: ExecutionPlan, seed: int = 0,
                        options: Optional[Options] = None,
                        device: Optional[Device] = None) -> Result:
        """hogwild::numa_dual_train (async_engine.cpp:462-520)."""
        return hogwild._run("sgdb_numa_dual_train", task, ds, hyper, plan, seed, options, device)

    @staticmethod
    def merge_models(replicas: list, weights=None) -> np.ndarray:
        """merge_models (async_engine.cpp:133-156): mean written back to every replica."""
        if not len(replicas):
            raise ValueError("merge_models: no replicas")
        d = len(replicas[0])
        if any(len(r) != d for r in replicas):
            raise ValueError("merge_models: dimension mismatch")
        if weights is not None:
            if len(weights) != len(replicas):
                raise ValueError("merge_models: weight count mismatch")
            total = 0.0
            for w in weights:  # sequential, as merge_models sums
                total += float(w)
            if total == 0.0:
                raise ValueError("merge_models: zero total weight")
        else:
            total = float(len(replicas))
        merged = np.zeros(d, np.float64)
        for i, r in enumerate(replicas):
            merged += (1.0 if weights is None else float(weights[i])) * np.asarray(r, np.float64)
        merged /= total
        for r in replicas:
            r[:] = merged
        return merged
