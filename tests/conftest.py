"""Shared test plumbing.

* registers the ``gpu`` marker (tests that need a B200; run with ``-m gpu``);
* puts the repo root on sys.path so ``oracle`` and the package import;
* loads the golden fixtures produced by ``tests/golden/make_golden.py``.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402
import pytest  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def digest(*arrays) -> str:
    """Same digest recipe as tests/golden/make_golden.py."""
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


_KAT = None


def kat():
    global _KAT
    if _KAT is None:
        with np.load(os.path.join(GOLDEN, "kat_small.npz")) as z:
            _KAT = {k: z[k] for k in z.files}
    return _KAT


def golden_hashes() -> dict:
    with open(os.path.join(GOLDEN, "golden_hashes.json")) as fh:
        return json.load(fh)


def relative_error(actual, expected) -> float:
    """2-norm relative error (reference tests/conftest.py:75-79)."""
    norm = float(np.linalg.norm(expected))
    err = float(np.linalg.norm(np.asarray(actual) - np.asarray(expected)))
    return err / norm if norm > 0 else err


def have_cuda() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def K():
    return kat()


def pytest_collection_modifyitems(config, items):
    if have_cuda():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
