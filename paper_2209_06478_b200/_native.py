"""ctypes binding of the C ABI in include/dynsparse_b200.h.

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2209_06478_b200/csrc``) into ``paper_2209_06478_b200/_lib``.
There is deliberately no fallback: every compute entry point raises
``DeviceError`` when the library or a CUDA device is missing.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import (
    BreakdownZeroCurvature,
    DeviceError,
    DiaFillOverflow,
    IndexOutOfRange,
    StructurallyAbsentDiagonal,
)

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib")
LIB_PATH = os.environ.get("DS_NATIVE_LIB") or os.path.join(LIB_DIR, "libdynsparse_b200.so")
# (DS_NATIVE_LIB: an alternate build of the same library, for A/B timing runs)

DS_OK = 0
DS_ERR_INVALID_ARGUMENT = 1
DS_ERR_CUDA = 2
DS_ERR_DIA_FILL_OVERFLOW = 3
DS_ERR_STRUCTURALLY_ABSENT_DIAG = 4
DS_ERR_BREAKDOWN = 5
DS_ERR_NOT_SUPPORTED = 6
DS_ERR_INDEX_OUT_OF_RANGE = 7
DS_ERR_RETRY = 8   # a speculative fast path did not apply (handled by the caller)
DS_FILL_LIMIT_DEFAULT = -(2**63)   # include/dynsparse_b200.h: the reference default limit

DS_CG_STAGE_NONE, DS_CG_STAGE_PAP, DS_CG_STAGE_RR, DS_CG_STAGE_SETUP = 0, 1, 2, 3
DS_CG_STAGE_DEFERRED = 4

c_i32, c_i64, c_dbl, c_vp, c_int = (ctypes.c_int32, ctypes.c_int64, ctypes.c_double,
                                    ctypes.c_void_p, ctypes.c_int)
P_i64 = ctypes.POINTER(ctypes.c_int64)
P_i32 = ctypes.POINTER(ctypes.c_int32)


class DsMatrix(ctypes.Structure):
    """Mirror of ``ds_matrix``."""

    _fields_ = [
        ("format", c_i32), ("ndiags", c_i32),
        ("nrows", c_i64), ("ncols", c_i64), ("nnz", c_i64),
        ("idx0", c_vp), ("idx1", c_vp), ("values", c_vp), ("long_rows", c_vp),
        ("n_long", c_i64), ("rows_sorted", c_i32), ("max_row_len", c_i32),
        ("row_perm", c_vp), ("bins", c_i64 * 9), ("tiles", c_vp), ("ntiles", c_i64),
    ]


class DsCgScalars(ctypes.Structure):
    """Mirror of ``ds_cg_scalars`` (lives on the device; 96 bytes)."""

    _fields_ = [
        ("rr", c_dbl), ("pap", c_dbl), ("alpha", c_dbl), ("beta", c_dbl),
        ("scale", c_dbl), ("tol", c_dbl), ("bb", c_dbl), ("rr_new", c_dbl),
        ("iter", c_i32), ("max_iters", c_i32), ("done", c_i32), ("pad", c_i32),
        ("rr_used", c_dbl), ("iter_next", c_i32), ("pad2", c_i32),
    ]


CG_SCALARS_BYTES = ctypes.sizeof(DsCgScalars)


class DsPcgScalars(ctypes.Structure):
    """Mirror of ``ds_pcg_scalars`` (lives on the device; 80 bytes)."""

    _fields_ = [
        ("rtz", c_dbl), ("pap", c_dbl), ("rr", c_dbl), ("rtz_new", c_dbl),
        ("alpha", c_dbl), ("beta", c_dbl), ("scale", c_dbl), ("tol", c_dbl),
        ("iter", c_i32), ("max_iters", c_i32), ("done", c_i32), ("pad", c_i32),
    ]
P_mat = ctypes.POINTER(DsMatrix)

# name -> (restype, argtypes)
_SIGNATURES = {
    "ds_last_error": (ctypes.c_char_p, []),
    "ds_abi_version": (c_int, []),
    "ds_device_sm_count": (c_int, [P_i32]),
    "ds_csr_analyze": (c_int, [c_i64, c_vp, c_vp, P_i64, P_i32, c_vp]),
    "ds_spmv_csr": (c_int, [c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp,
                            c_int, c_vp]),
    "ds_spmv_dia": (c_int, [c_i64, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_int, c_vp]),
    "ds_spmv_coo": (c_int, [c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_int, c_vp, c_vp, c_int,
                            c_vp]),
    "ds_coo_order_flags": (c_int, [c_i64, c_vp, c_vp, P_i32, c_vp]),
    "ds_coo_max_run": (c_int, [c_i64, c_vp, P_i32, c_vp]),
    "ds_coo_long_runs": (c_int, [c_i64, c_vp, c_i32, c_vp, c_i64, P_i64, c_vp]),
    "ds_coo_long_run_threshold": (c_int, []),
    "ds_spmv_coo_sorted": (c_int, [c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp,
                                   c_int, c_vp]),
    "ds_csr_bins": (c_int, [c_i64, c_vp, c_vp, P_i64, c_vp]),
    "ds_csr_tiles_capacity": (c_i64, [c_i64, c_i64]),
    "ds_csr_tiles": (c_int, [c_i64, c_vp, c_vp, c_i64, P_i64, P_i64, c_vp]),
    "ds_dot_workspace_bytes": (c_i64, []),
    "ds_dot": (c_int, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "ds_waxpby": (c_int, [c_i64, c_dbl, c_vp, c_dbl, c_vp, c_vp, c_vp]),
    "ds_scan": (c_int, [c_i64, c_vp, c_vp, c_vp, c_vp]),
    "ds_extract_diag_csr": (c_int, [c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "ds_extract_diag_coo": (c_int, [c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "ds_update_diag_csr": (c_int, [c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, P_i64, c_vp]),
    "ds_update_diag_coo": (c_int, [c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, P_i64, c_vp]),
    "ds_dia_count_nonzero": (c_int, [c_i64, c_i64, c_i32, c_vp, c_vp, P_i64, c_vp]),
    "ds_dia_diag_column": (c_int, [c_i64, c_i32, c_i32, c_vp, c_vp, c_int, c_vp]),
    "ds_convert_begin_coo": (c_int, [c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_int, c_i64, c_vp,
                                     ctypes.POINTER(c_vp), P_i64, P_i64]),
    "ds_convert_begin_csr": (c_int, [c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_int, c_i64, c_vp,
                                     ctypes.POINTER(c_vp), P_i64, P_i64]),
    "ds_convert_begin_dia": (c_int, [c_i64, c_i64, c_i32, c_vp, c_vp, c_int, c_i64, c_vp,
                                     ctypes.POINTER(c_vp), P_i64, P_i64]),
    "ds_convert_begin_csr_dia_spec": (c_int, [c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_i64, c_vp,
                                              ctypes.POINTER(c_vp), P_i64]),
    "ds_convert_begin_coo_dia_spec": (c_int, [c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_i64, c_vp,
                                              ctypes.POINTER(c_vp), P_i64]),
    "ds_convert_direct": (c_int, [c_int, c_int, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp,
                                  c_vp, c_vp, P_i32]),
    "ds_convert_finish_coo": (c_int, [c_vp, c_vp, c_vp, c_vp]),
    "ds_convert_finish_csr": (c_int, [c_vp, c_vp, c_vp, c_vp]),
    "ds_convert_finish_dia": (c_int, [c_vp, c_vp, c_vp]),
    "ds_convert_abort": (None, [c_vp]),
    "ds_gather": (c_int, [c_i64, c_vp, c_vp, c_vp, c_vp]),
    "ds_symgs": (c_int, [c_i64, c_vp, c_vp, c_vp, c_vp, P_i64, c_int, c_vp, c_vp, c_vp]),
    "ds_symgs_ell_width": (c_int, [c_i64, c_vp, c_vp, ctypes.POINTER(c_i32), c_vp]),
    "ds_symgs_ell_fill": (c_int, [c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                  c_vp]),
    "ds_symgs_ell": (c_int, [c_i64, c_i32, c_vp, P_i64, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                             c_vp]),
    "ds_symgs_oell_fill": (c_int, [c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                   c_vp, c_vp]),
    "ds_symgs_oell": (c_int, [c_i64, c_i32, c_vp, c_vp, P_i64, c_int, c_vp, c_vp, c_vp, c_vp,
                              c_vp, c_vp]),
    "ds_pcg_alpha": (c_int, [c_vp, c_vp]),
    "ds_pcg_check": (c_int, [c_vp, c_vp, c_vp]),
    "ds_pcg_beta": (c_int, [c_vp, c_vp]),
    "ds_pcg_axpy": (c_int, [c_i64, c_vp, c_vp, c_vp, c_int, c_vp, c_vp, c_vp]),
    "ds_mg_restrict_residual": (c_int, [P_mat, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "ds_mg_restrict": (c_int, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "ds_mg_prolong": (c_int, [c_i64, c_vp, c_vp, c_vp, c_vp]),
    "ds_stencil_begin": (c_int, [c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_vp,
                                 ctypes.POINTER(c_vp), P_i64, P_i64]),
    "ds_stencil_finish": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "ds_csr_split_count": (c_int, [c_i64, c_i64, c_vp, c_vp, c_vp, P_i64, c_vp]),
    "ds_csr_split_fill": (c_int, [c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp,
                                  c_vp, c_vp, c_vp, c_vp]),
    "ds_spmv": (c_int, [P_mat, c_vp, c_vp, c_int, c_vp]),
    "ds_cg_workspace_bytes": (c_i64, []),
    "ds_cg_spmv_dot": (c_int, [P_mat, c_vp, c_vp, c_int, c_vp, c_vp, c_int, c_vp, c_vp, c_vp,
                               c_int, c_vp, c_vp]),
    "ds_cg_setup_residual": (c_int, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "ds_cg_setup_finalize": (c_int, [c_vp, c_vp, c_vp, c_int, c_dbl, c_i32, c_vp, c_vp]),
    "ds_cg_update": (c_int, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_int, c_vp,
                             c_vp]),
    "ds_cg_direction": (c_int, [c_i64, c_vp, c_vp, c_vp, c_vp]),
    "ds_cg_finalize": (c_int, [c_int, c_vp, c_vp, c_vp, c_int, c_vp]),
    "ds_cg_gather": (c_int, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "ds_cg_update_deferred": (c_int, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "ds_cg_direction_deferred": (c_int, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "ds_l2_persist": (c_int, [c_vp, c_i64, c_vp]),
    "ds_l2_persist_reset": (c_int, [c_vp]),
    "ds_probe_gather": (c_int, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "ds_cg_update_direction_deferred": (c_int, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                                c_vp, c_vp]),
    "ds_cg_update_gathered": (c_int, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_int, c_vp,
                                      c_vp, c_vp]),
    "ds_cg_direction_gathered": (c_int, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_int, c_vp, c_vp]),
    "ds_nccl_unique_id_bytes": (c_int, []),
    "ds_nccl_unique_id": (c_int, [ctypes.c_char_p, c_int]),
    "ds_nccl_comm_init": (c_int, [ctypes.c_char_p, c_int, c_int, ctypes.POINTER(c_vp)]),
    "ds_nccl_comm_destroy": (c_int, [c_vp]),
    "ds_halo_exchange": (c_int, [c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                 c_vp]),
    "ds_allgather_f64": (c_int, [c_vp, c_vp, c_i64, c_vp, c_vp]),
    "ds_while_graph_begin": (c_int, [c_vp, ctypes.POINTER(c_vp), ctypes.POINTER(ctypes.c_ulonglong)]),
    "ds_while_graph_end": (c_int, [c_vp, c_vp, ctypes.POINTER(c_vp)]),
    "ds_cg_while_continue": (c_int, [ctypes.c_ulonglong, c_vp, c_vp]),
    "ds_graph_exec_launch": (c_int, [c_vp, c_vp]),
    "ds_graph_destroy": (c_int, [c_vp, c_vp]),
    "ds_dia_to_entries": (c_int, [c_i64, c_i64, c_i32, c_vp, c_vp, c_int, c_vp, c_vp, c_vp, P_i64,
                                  c_vp]),
    "ds_radix_sort_pairs": (c_int, [c_vp, c_i64, c_int, c_vp, c_vp, c_vp]),
    "ds_ipc_handle_bytes": (c_int, []),
    "ds_ipc_export": (c_int, [c_vp, ctypes.c_char_p]),
    "ds_ipc_import": (c_int, [ctypes.c_char_p, ctypes.POINTER(c_vp)]),
    "ds_ipc_close": (c_int, [c_vp]),
    "ds_peer_allgather_f64": (c_int, [c_vp, c_int, c_int, c_int, c_vp, c_vp, c_vp, c_int, c_vp]),
    "ds_peer_halo_push": (c_int, [c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "ds_peer_wait_flags": (c_int, [c_int, c_vp, c_int, c_vp]),
}

DS_PEER_WAIT_SPIN, DS_PEER_WAIT_MEMOP = 0, 1
DS_PEER_MAX_RANKS, DS_PEER_MAX_NBR = 64, 26

EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_lock = threading.Lock()
_lib = None


def load():
    """Load (once) and return the ctypes handle; raise DeviceError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise DeviceError(
                    f"native extension missing at {LIB_PATH}; build it with "
                    "`python -c 'import __graft_entry__ as g; g.build()'`")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def last_error() -> str:
    msg = load().ds_last_error()
    return msg.decode(errors="replace") if msg else ""


def check(status: int, *, index: int | None = None) -> None:
    """Map a C status code onto the reference's exception classes."""
    if status == DS_OK:
        return
    msg = last_error()
    if status == DS_ERR_DIA_FILL_OVERFLOW:
        raise DiaFillOverflow(msg)
    if status == DS_ERR_STRUCTURALLY_ABSENT_DIAG:
        raise StructurallyAbsentDiagonal(int(index if index is not None else 0))
    if status == DS_ERR_BREAKDOWN:
        raise BreakdownZeroCurvature(msg)
    if status == DS_ERR_INDEX_OUT_OF_RANGE:
        raise IndexOutOfRange(msg)
    raise DeviceError(f"dynsparse native error {status}: {msg}")


def call(name: str, *args, **kw) -> None:
    check(getattr(load(), name)(*args), **kw)
