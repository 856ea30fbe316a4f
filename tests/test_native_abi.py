"""CPU-side checks of the C ABI boundary: the library loads (no GPU needed
to dlopen) and exports every symbol include/dynsparse_b200.h declares, with
the ctypes struct layouts matching the header."""

from __future__ import annotations

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "dynsparse_b200.h")


def declared_functions() -> list[str]:
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?(?:int|int64_t|void|char\s*\*|const\s+char\s*\*)\s*\*?\s*"
                       r"(ds_\w+)\s*\(", text, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_hot_path():
    names = declared_functions()
    for must in ("ds_spmv_csr", "ds_spmv_dia", "ds_spmv_coo", "ds_spmv", "ds_dot", "ds_waxpby",
                 "ds_convert_begin_coo", "ds_convert_finish_dia", "ds_gather", "ds_cg_update"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2209_06478_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert set(declared_functions()) == set(_native.EXPORTED_SYMBOLS)
    assert lib.ds_abi_version() == 1
    h = _native.load()
    assert h.ds_cg_workspace_bytes() > 0
    assert h.ds_last_error() is not None


def test_struct_layouts_match_header():
    from paper_2209_06478_b200 import _native
    assert ctypes.sizeof(_native.DsMatrix) == 4 + 4 + 8 * 3 + 8 * 4 + 8 + 4 + 4 + 8 + 8 * 9 + 8 + 8
    assert ctypes.sizeof(_native.DsCgScalars) == 8 * 8 + 4 * 4 + 8 + 4 + 4
    assert ctypes.sizeof(_native.DsPcgScalars) == 8 * 8 + 4 * 4
    assert _native.CG_SCALARS_BYTES % 8 == 0


def test_status_codes_map_to_reference_exceptions():
    from paper_2209_06478_b200 import _native, errors
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built")
    with pytest.raises(errors.DiaFillOverflow):
        _native.check(_native.DS_ERR_DIA_FILL_OVERFLOW)
    with pytest.raises(errors.StructurallyAbsentDiagonal) as e:
        _native.check(_native.DS_ERR_STRUCTURALLY_ABSENT_DIAG, index=7)
    assert e.value.index == 7
    with pytest.raises(errors.BreakdownZeroCurvature):
        _native.check(_native.DS_ERR_BREAKDOWN)
    with pytest.raises(errors.DeviceError):
        _native.check(_native.DS_ERR_CUDA)


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2209_06478_b200")
    for base, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                text = open(os.path.join(base, f)).read()
                assert "oracle" not in text.replace("Oracle", ""), f


def test_no_cuda_means_loud_failure():
    import torch

    import paper_2209_06478_b200 as ds
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    a = ds.build_csr(2, 2, [0, 1, 2], [0, 1], [1.0, 1.0])
    with pytest.raises(ds.DeviceError):
        ds.spmv(ds.SERIAL, a, ds.DenseVector([1.0, 2.0]), ds.DenseVector.zeros(2))
    with pytest.raises(ds.DeviceError):
        ds.convert(a, ds.FormatId.DIA)
