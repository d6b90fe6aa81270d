"""B200-native GLM SGD engine (arXiv 1802.08800): synchronous mini-batch SGD and
Hogwild for logistic regression / linear SVM as hand-written sm_100a kernels
behind the C-ABI of include/sgdb.h, with the reference's interface mirrored in
Python (api.py) and C++ (include/sgdb_b200.hpp).

Importing requires the in-tree libsgdb_b200.so (no CPU fallback).
"""
from . import _lib
from .api import (  # noqa: F401
    AccessPath, Dataset, Device, DeviceDataset, DeviceModel, ElementwiseOp, EpochRecord,
    ExecutionPlan,
    Hyperparams, Layout, LossTrace, ModelReplication, Options, Result, Schedule, Strategy, Task,
    TrainOptions, TrainResult, assign, convert_layout, dataset_loss, default_device,
    device_loss, fixtures, generate_hidden_model, hogwild, hogwild_epoch, linalg, load_binary, models_average, parse_libsvm,
    parse_plan, plan_to_string, save_binary, set_default_precision, sync, sync_epoch,
    validate_plan, write_libsvm,
)
from ._lib import CapacityError, CudaError, ParseError, SgdbError, UnsupportedError  # noqa: F401
from . import harness  # noqa: F401,E402  (sgdbench::harness over the device engines)

_lib.load()

__all__ = [n for n in dir() if not n.startswith("_")]
