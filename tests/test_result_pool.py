"""Host logic of cg()'s pinned result pool (solver._pinned_result): a buffer
handed out as a numpy array is reused only after every array / view over it
is gone, and the array keeps the buffer alive (no GPU: the pinned allocation
is replaced by a plain one)."""
import gc
import types

import numpy as np
import torch

from paper_2209_06478_b200 import solver as S


def test_result_pool_reuse_and_lifetime(monkeypatch):
    orig = torch.empty

    def fake_empty(*a, **k):
        k.pop("pin_memory", None)
        return orig(*a, **k)

    monkeypatch.setattr(torch, "empty", fake_empty)
    eng = types.SimpleNamespace()
    e1 = S._pinned_result(eng, 0, 8)
    a = np.ctypeslib.as_array(e1[1])
    a[:] = 1.0
    e2 = S._pinned_result(eng, 0, 8)
    assert e2 is not e1                      # a is alive: not reused
    v = a[2:4]
    del a
    assert S._pinned_result(eng, 0, 8) is e2  # e2 was never handed out as an array
    x = np.ctypeslib.as_array(e2[1])
    del v
    assert S._pinned_result(eng, 0, 8) is e1  # the last view of e1 died
    # the array outlives the engine and its pool
    del eng, e1, e2
    gc.collect()
    x[:] = 3.0
    assert float(x.sum()) == 24.0
