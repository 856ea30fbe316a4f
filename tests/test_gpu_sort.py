"""GPU: the hand-written stable radix sort behind the COO canonicalisation
(ds_sort.cu; the reference's stable np.lexsort, datamove.py:212) -- keys and
permutation equal numpy's stable argsort on tiles' edges, duplicates-heavy
and full-width keys."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_2209_06478_b200 import _native  # noqa: E402

DEV = torch.device("cuda", 0)


def gpu_sort(keys: np.ndarray, bits: int):
    lib = _native.load()
    n = keys.size
    kin = torch.from_numpy(keys.view(np.int64)).to(DEV)
    kout = torch.empty(max(n, 1), dtype=torch.int64, device=DEV)
    perm = torch.empty(max(n, 1), dtype=torch.int32, device=DEV)
    _native.check(lib.ds_radix_sort_pairs(kin.data_ptr() if n else None, n, bits,
                                          kout.data_ptr(), perm.data_ptr(),
                                          torch.cuda.current_stream(DEV).cuda_stream))
    torch.cuda.synchronize(DEV)
    return kout[:n].cpu().numpy().view(np.uint64), perm[:n].cpu().numpy()


@pytest.mark.parametrize("n", [0, 1, 31, 4095, 4096, 4097, 8192 + 17, 300_001])
@pytest.mark.parametrize("bits", [1, 8, 9, 20, 44, 64])
def test_radix_sort_matches_stable_argsort(n, bits):
    rng = np.random.default_rng(n * 131 + bits)
    hi = np.uint64((1 << bits) - 1) if bits < 64 else np.uint64(2**64 - 1)
    keys = rng.integers(0, hi, size=n, dtype=np.uint64, endpoint=True)
    if n > 8:   # heavy duplicates
        keys[rng.random(n) < 0.5] = keys[0]
    k, p = gpu_sort(keys, bits)
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(p, order)
    assert np.array_equal(k, keys[order])


def test_radix_sort_large_presorted_and_reversed():
    n = 3_000_000
    for keys in (np.arange(n, dtype=np.uint64), np.arange(n, dtype=np.uint64)[::-1].copy(),
                 np.repeat(np.arange(n // 1000, dtype=np.uint64), 1000)):
        k, p = gpu_sort(keys, 22)
        order = np.argsort(keys, kind="stable")
        assert np.array_equal(p, order) and np.array_equal(k, keys[order])
