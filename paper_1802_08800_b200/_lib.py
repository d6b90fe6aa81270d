"""ctypes binding of libsgdb_b200.so (declarations: include/sgdb.h).

The library is built in-tree (``__graft_entry__.build()`` / ``make -C
paper_1802_08800_b200/csrc``). There is no fallback: importing the product
without the library raises, and every device op raises when CUDA is absent.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsgdb_b200.so")

u64, i64, i32, u32, dbl, vp = C.c_uint64, C.c_int64, C.c_int32, C.c_uint32, C.c_double, C.c_void_p
P = C.POINTER

SGDB_OK = 0
SGDB_UPLOAD_EXACT_FP64 = 1
SGDB_UPLOAD_PADDED = 2
STATUS_NAMES = {
    1: "invalid_argument", 2: "domain_error", 3: "parse_error", 4: "capacity_error",
    5: "runtime_error", 6: "cuda_error", 7: "unsupported",
}


class DatasetView(C.Structure):
    _fields_ = [("n_examples", u64), ("n_features", u64), ("layout", i32),
                ("labels", P(dbl)), ("values", P(dbl)), ("n_values", u64),
                ("indices", P(u32)), ("n_indices", u64),
                ("row_offsets", P(u64)), ("n_row_offsets", u64), ("padded_width", u64)]


class Hyper(C.Structure):
    _fields_ = [("alpha", dbl), ("batch_b", u64), ("epochs", u64), ("task", i32),
                ("step_decay", dbl)]


class Plan(C.Structure):
    _fields_ = [("access_path", i32), ("replication", i32), ("data_replication_k", u64),
                ("workers", u64), ("group_size", u64), ("circular_offsets", i32),
                ("merge_period_epochs", u64), ("lanes_per_worker", i32)]


class EpochRecord(C.Structure):
    _fields_ = [("epoch", u64), ("loss", dbl), ("seconds", dbl)]


class Trace(C.Structure):
    _fields_ = [("epochs", P(EpochRecord)), ("evals_per_epoch", P(u64)), ("capacity", u64),
                ("count", u64), ("diverged", i32), ("divergence_note", C.c_char * 160)]


CLOCK_FN = C.CFUNCTYPE(dbl, vp)
HOOK_FN = C.CFUNCTYPE(None, vp, u64, dbl)
ALLREDUCE_FN = C.CFUNCTYPE(i32, vp, vp, u64, i32, vp)


class TrainOptions(C.Structure):
    _fields_ = [("workers", u32), ("shuffle", i32), ("max_seconds", dbl),
                ("initial_model", P(dbl)), ("initial_model_len", u64),
                ("clock", CLOCK_FN), ("clock_user", vp),
                ("epoch_hook", HOOK_FN), ("hook_user", vp)]


# name -> (restype, argtypes); every function returns sgdb_status unless noted.
_S = i32
PROTOTYPES = {
    "sgdb_last_error": (C.c_char_p, []),
    "sgdb_version": (C.c_char_p, []),
    "sgdb_ctx_create": (_S, [i32, vp, P(vp)]),
    "sgdb_ctx_destroy": (_S, [vp]),
    "sgdb_ctx_stream": (_S, [vp, P(vp)]),
    "sgdb_ctx_synchronize": (_S, [vp]),
    "sgdb_ctx_launch_count": (_S, [vp, P(u64)]),
    "sgdb_ctx_set_allreduce": (_S, [vp, ALLREDUCE_FN, vp]),
    "sgdb_nccl_get_unique_id": (_S, [C.c_char_p]),
    "sgdb_ctx_init_nccl": (_S, [vp, i32, i32, C.c_char_p]),
    "sgdb_ctx_world": (_S, [vp, C.POINTER(i32), C.POINTER(i32)]),
    "sgdb_ctx_resident_workers": (_S, [vp, vp, i32, P(u64)]),
    "sgdb_ctx_set_profiling": (_S, [vp, i32]),
    "sgdb_ctx_kernel_stats": (_S, [vp, u64, C.c_char_p, u64, P(u64), P(dbl), P(u64)]),
    "sgdb_model_average_ranks": (_S, [vp, vp, u64]),
    "sgdb_dataset_upload": (_S, [vp, P(DatasetView), u64, u64, P(vp)]),
    "sgdb_dataset_upload_ex": (_S, [vp, P(DatasetView), u64, u64, u32, P(vp)]),
    "sgdb_dataset_refresh_f32": (_S, [vp, vp, vp, vp, vp, vp]),
    "sgdb_dataset_refresh_idx16": (_S, [vp, vp, vp]),
    "sgdb_dataset_free": (_S, [vp]),
    "sgdb_dataset_generate_dense": (_S, [vp, u64, u64, u64, u64, u64, dbl, P(vp)]),
    "sgdb_generate_hidden_model": (_S, [u64, u64, P(dbl)]),
    "sgdb_dataset_read_dense": (_S, [vp, vp, u64, u64, vp, vp]),
    "sgdb_dataset_sweep_bytes": (_S, [vp, P(u64)]),
    "sgdb_dataset_shape": (_S, [vp, P(u64), P(u64), P(u64), P(u64), P(u64)]),
    "sgdb_model_create": (_S, [vp, u64, P(dbl), P(vp)]),
    "sgdb_model_set": (_S, [vp, vp, P(dbl)]),
    "sgdb_model_get": (_S, [vp, vp, P(dbl)]),
    "sgdb_model_device_ptrs": (_S, [vp, P(vp), P(vp)]),
    "sgdb_model_free": (_S, [vp]),
    "sgdb_sync_epoch": (_S, [vp, vp, vp, i32, dbl, P(u32), u64, P(i32)]),
    "sgdb_batch_gradient": (_S, [vp, vp, i32, P(u32), u64, P(dbl), i32, P(dbl)]),
    "sgdb_epoch_batch": (_S, [vp, vp, vp, i32, dbl, P(dbl)]),
    "sgdb_hogwild_epoch": (_S, [vp, vp, vp, i32, dbl, P(Plan), P(u64)]),
    "sgdb_hogwild_segment": (_S, [vp, vp, vp, i32, dbl, P(Plan), u32, u32, P(u64)]),
    "sgdb_models_average": (_S, [vp, P(vp), u64, P(dbl), vp, i32]),
    "sgdb_loss": (_S, [vp, vp, vp, i32, P(dbl)]),
    "sgdb_matvec": (_S, [vp, vp, P(u32), u64, P(dbl), u64, P(dbl)]),
    "sgdb_matvec_transposed": (_S, [vp, vp, P(u32), u64, P(dbl), u64, P(dbl)]),
    "sgdb_elementwise": (_S, [vp, i32, P(dbl), P(dbl), u64, dbl, P(dbl)]),
    "sgdb_axpy": (_S, [vp, P(dbl), dbl, P(dbl), u64]),
    "sgdb_sync_train": (_S, [vp, vp, P(Hyper), u64, P(TrainOptions), P(dbl), P(Trace)]),
    "sgdb_hogwild_train": (_S, [vp, vp, P(Hyper), P(Plan), u64, P(TrainOptions), P(dbl),
                                P(Trace)]),
    "sgdb_numa_dual_train": (_S, [vp, vp, P(Hyper), P(Plan), u64, P(TrainOptions), P(dbl),
                                  P(Trace)]),
    "sgdb_fixture_dense": (_S, [u64, u64, u64, dbl, P(vp)]),
    "sgdb_fixture_sparse": (_S, [u64, u64, dbl, u64, dbl, P(vp)]),
    "sgdb_parse_libsvm": (_S, [C.c_char_p, u64, i64, P(vp), P(u64)]),
    "sgdb_write_libsvm": (_S, [P(DatasetView), vp, u64, P(u64)]),
    "sgdb_save_binary": (_S, [P(DatasetView), C.c_char_p]),
    "sgdb_load_binary": (_S, [C.c_char_p, P(vp)]),
    "sgdb_convert_layout": (_S, [P(DatasetView), i32, u64, P(vp)]),
    "sgdb_validate_dataset": (_S, [P(DatasetView)]),
    "sgdb_host_dataset_view": (_S, [vp, P(DatasetView)]),
    "sgdb_host_dataset_free": (_S, [vp]),
    "sgdb_assign": (_S, [u64, u64, i32, u64, P(u32), P(u64), P(u64)]),
    "sgdb_parse_plan": (_S, [C.c_char_p, P(Plan)]),
    "sgdb_plan_to_string": (_S, [P(Plan), C.c_char_p, u64]),
    "sgdb_validate_plan": (_S, [P(Plan), i32]),
    "sgdb_schedule_create": (_S, [u64, u64, i32, P(vp)]),
    "sgdb_schedule_next": (_S, [vp, P(u32)]),
    "sgdb_schedule_free": (_S, [vp]),
}

_LIB = None


def load():
    """Loads the in-tree library (raises if it has not been built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (or make -C paper_1802_08800_b200/csrc)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in PROTOTYPES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
    return _LIB


class SgdbError(RuntimeError):
    def __init__(self, status, message):
        super().__init__(f"[{STATUS_NAMES.get(status, status)}] {message}")
        self.status = status
        self.message = message


class ParseError(SgdbError, ValueError):
    """sgdbench::ParseError (dataset.hpp:22-26); .line_number is 1-based."""

    def __init__(self, status, message, line):
        super().__init__(status, message)
        self.line_number = line


class CapacityError(SgdbError):
    pass


class UnsupportedError(SgdbError):
    pass


class CudaError(SgdbError):
    pass


def check(status, line=None):
    """Raises the Python counterpart of the reference's exception type."""
    if status == SGDB_OK:
        return
    msg = load().sgdb_last_error().decode(errors="replace")
    if status == 1:
        raise ValueError(msg)  # std::invalid_argument
    if status == 2:
        raise ArithmeticError(msg)  # std::domain_error
    if status == 3:
        raise ParseError(status, msg, line)
    if status == 4:
        raise CapacityError(status, msg)
    if status == 7:
        raise UnsupportedError(status, msg)
    if status == 6:
        raise CudaError(status, msg)
    raise SgdbError(status, msg)
