import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libsgdb_b200.so on cuda:0)")
    config.addinivalue_line("markers", "slow: long-running")


def _gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _gpu_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle.oracle()


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.reference_available():
        pytest.skip("oracle/_ref not built")
    return oracle.reference()


@pytest.fixture(scope="session")
def sgdb():
    import paper_1802_08800_b200 as S
    return S


@pytest.fixture(scope="session")
def dev(sgdb):
    return sgdb.default_device()


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = max(np.linalg.norm(b), 1e-300)
    return float(np.linalg.norm(a - b) / den)


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def record(test, **values):
    """Append measured parity numbers (errors, epochs-to-1%) to
    gpurun_out/parity.jsonl when that directory exists (GPU runs), so the
    worst-case errors behind each green assertion can be committed."""
    import json
    out = os.path.join(ROOT, "gpurun_out")
    if not os.path.isdir(out):
        return
    with open(os.path.join(out, "parity.jsonl"), "a") as f:
        f.write(json.dumps({"test": test, **{k: (float(v) if isinstance(v, (np.floating, float))
                                                 else v) for k, v in values.items()}}) + "\n")
