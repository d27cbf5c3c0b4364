import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")


def _have_gpu() -> bool:
    try:
        from paper_2507_13204_b200 import _cabi

        return _cabi.device_count() > 0
    except Exception:
        return False


HAVE_GPU = _have_gpu()


def pytest_collection_modifyitems(config, items):
    if HAVE_GPU:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def same_bits(a, b) -> bool:
    """Bit equality of float64 data; all NaNs compare equal (NaN sign/payload is
    not part of the contract)."""
    a = np.array(a, dtype=np.float64, ndmin=1)
    b = np.array(b, dtype=np.float64, ndmin=1)
    if a.shape != b.shape:
        return False
    na, nb = np.isnan(a), np.isnan(b)
    return bool(np.array_equal(na, nb) and np.array_equal(a[~na].view(np.uint64), b[~nb].view(np.uint64)))


def assert_bits(a, b, what=""):
    if not same_bits(a, b):
        a = np.array(a, dtype=np.float64, ndmin=1)
        b = np.array(b, dtype=np.float64, ndmin=1)
        bad = np.flatnonzero(~((a == b) | (np.isnan(a) & np.isnan(b))).reshape(-1)) if a.shape == b.shape else []
        raise AssertionError(f"{what}: bit mismatch at {list(bad[:8])} "
                             f"got {a.reshape(-1)[bad[:4]] if len(bad) else a.shape} "
                             f"want {b.reshape(-1)[bad[:4]] if len(bad) else b.shape}")


@pytest.fixture(scope="session")
def corpus_golden():
    return np.load(os.path.join(GOLDEN, "corpus.npz"))


@pytest.fixture(scope="session")
def laplacian_golden():
    return np.load(os.path.join(GOLDEN, "laplacian.npz"))


@pytest.fixture(scope="session")
def pairwise_golden():
    return np.load(os.path.join(GOLDEN, "pairwise.npz"))


CORPUS = sorted(f[:-4] for f in os.listdir(os.path.join(ROOT, "paper_2507_13204_b200", "programs")))
SIZES = (1, 2, 3, 17, 257)


def corpus_case(golden, stem, n):
    """(inputs dict, wrt tuple, key prefix) of one stored corpus case."""
    key = f"{stem}/n{n}"
    prefix = key + "/in/"
    inputs = {}
    for k in golden.files:
        if k.startswith(prefix):
            v = golden[k]
            inputs[k[len(prefix):]] = float(v) if v.ndim == 0 else np.array(v)
    wrt = tuple(str(golden[key + "/wrt"]).split(","))
    return inputs, wrt, key


def free_port() -> int:
    """A TCP port the OS reports free on 127.0.0.1 (rendezvous of the multi-process tests)."""
    import socket

    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sock:
        sock.bind(("127.0.0.1", 0))
        return sock.getsockname()[1]
