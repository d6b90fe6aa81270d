"""The C-ABI library loads, exports every entry point include/sgdb.h declares,
was built for sm_100a, and fails loudly (no CPU fallback) without a GPU."""
import os
import re
import subprocess

import pytest

import paper_1802_08800_b200 as S
from paper_1802_08800_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "sgdb.h")).read()
    return sorted(set(re.findall(r"\b(sgdb_[a-z0-9_]+)\s*\(", text)) - {"sgdb_status"})


def test_every_declared_symbol_is_exported():
    lib = _lib.load()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert len(declared_symbols()) >= 45


def test_every_declared_symbol_has_a_python_prototype():
    assert set(declared_symbols()) <= set(_lib.PROTOTYPES)


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_version():
    assert b"sm_100a" in _lib.load().sgdb_version()


def test_device_ops_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.CudaError):
        S.Device(0)


def test_status_mapping():
    with pytest.raises(ValueError):
        S.parse_plan("bogus")
    with pytest.raises(S.ParseError):
        S.parse_libsvm("x 1:1\n")
