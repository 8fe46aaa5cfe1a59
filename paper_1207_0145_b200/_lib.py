"""ctypes binding of libmpsm_b200.so (the C ABI in include/mpsm_b200.h).

This is the reference-side binding a maintainer adds: it
replaces the numba call boundary of /root/reference/pkg/src/mpsm/_kernels.py.
There is no fallback: if the library is missing or no CUDA device is present,
every call raises.
"""

from __future__ import annotations

import ctypes
import os

from .core import ConfigurationError, DomainError, FormatError, InternalConsistencyError, MaterializeCapExceeded

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MPSM_LIB") or os.path.join(_HERE, "libmpsm_b200.so")

MPSM_OK = 0
ERR_DOMAIN, ERR_INTERNAL, ERR_CONFIG, ERR_CUDA, ERR_CAP, ERR_ARG, ERR_FORMAT, ERR_IO = -1, -2, -3, -4, -5, -6, -7, -8
MODE_AGGREGATE_MAX, MODE_COUNT, MODE_MATERIALIZE = 0, 1, 2
PAIR_COUNT, PAIR_BEST, PAIR_CHECKSUM, PAIR_START, PAIR_PROBES, PAIR_END, PAIR_EXAMINED, PAIR_EMITTED, PAIR_FLAGS = range(9)
PAIR_FIELDS = 9
FLAG_UNSORTED = 1

# every symbol include/mpsm_b200.h declares (checked by tests/test_boundary.py)
EXPORTS = (
    "mpsm_version", "mpsm_last_error", "mpsm_device_init", "mpsm_launch_count",
    "mpsm_profile_enable", "mpsm_profile_read",
    "mpsm_sort_workspace_bytes", "mpsm_sort_pass_count", "mpsm_sort_pairs", "mpsm_sort_packed",
    "mpsm_radix_histogram", "mpsm_domain_report", "mpsm_check_sorted",
    "mpsm_scatter_workspace_bytes", "mpsm_scatter_chunk",
    "mpsm_interp_lower_bound",
    "mpsm_join_workspace_bytes", "mpsm_join_pairs", "mpsm_join_pairs_packed",
    "mpsm_minmax_contiguous",
    "mpsm_ipc_get_handle", "mpsm_ipc_open_handle", "mpsm_ipc_close_handle",
    "mpsm_relfile_header", "mpsm_relfile_read", "mpsm_relfile_read_columns", "mpsm_relfile_write",
    "mpsm_deinterleave",
    "mpsm_upload_records", "mpsm_upload_bytes", "mpsm_sort_records", "mpsm_pack_records", "mpsm_partition_records",
    "mpsm_sort_segments_workspace_bytes", "mpsm_sort_pairs_segments", "mpsm_sort_packed_segments",
    "mpsm_sort_records_segments", "mpsm_sort_packed_dense", "mpsm_sort_records_dense",
    "mpsm_join_pairs_packed_hint", "mpsm_fetch_small",
)


class RunDesc(ctypes.Structure):
    _fields_ = [("keys", ctypes.c_void_p), ("pays", ctypes.c_void_p), ("n", ctypes.c_int64)]


_vp, _i64, _u64, _int, _sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, ctypes.c_size_t

_SIGS = {
    "mpsm_version": (_int, []),
    "mpsm_last_error": (ctypes.c_char_p, []),
    "mpsm_device_init": (_int, [_int]),
    "mpsm_launch_count": (_u64, []),
    "mpsm_fetch_small": (_int, [_vp, _vp, _i64, _vp, _i64, _vp]),
    "mpsm_profile_enable": (_int, [_int]),
    "mpsm_profile_read": (_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_u64)]),
    "mpsm_sort_workspace_bytes": (_int, [_i64, _int, ctypes.POINTER(_sz)]),
    "mpsm_sort_pass_count": (_int, [_int]),
    "mpsm_sort_pairs": (_int, [_vp, _vp, _i64, _u64, _u64, _int, _vp, _vp, _vp, _vp, _vp, _sz, _vp, _vp]),
    "mpsm_sort_packed": (_int, [_vp, _vp, _i64, _u64, _u64, _int, _vp, _vp, _vp, _sz, _vp, _vp, _vp]),
    "mpsm_radix_histogram": (_int, [_vp, _i64, _u64, _u64, _int, _int, _vp, _vp, _vp]),
    "mpsm_domain_report": (_int, [_vp, _i64, _u64, _u64, _vp, _vp]),
    "mpsm_check_sorted": (_int, [_vp, _i64, _vp, _vp]),
    "mpsm_scatter_workspace_bytes": (_int, [_i64, _int, ctypes.POINTER(_sz)]),
    "mpsm_scatter_chunk": (_int, [_vp, _vp, _i64, _u64, _int, _vp, _int, _int, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "mpsm_interp_lower_bound": (_int, [_vp, _i64, _vp, _i64, _vp, _vp, _vp]),
    "mpsm_join_workspace_bytes": (_int, [ctypes.POINTER(RunDesc), _int, ctypes.POINTER(RunDesc), _int,
                                         ctypes.POINTER(_sz)]),
    "mpsm_join_pairs": (_int, [ctypes.POINTER(RunDesc), _int, ctypes.POINTER(RunDesc), _int, _int, _int, _vp, _i64,
                               _vp, _vp, _sz, _vp]),
    "mpsm_join_pairs_packed": (_int, [ctypes.POINTER(RunDesc), _int, ctypes.POINTER(RunDesc), _int, _int, _u64, _int,
                                      _int, _vp, _i64, _vp, _vp, _sz, _vp]),
    "mpsm_minmax_contiguous": (_int, [_i64, _int, _vp, _vp, _vp, _i64, _vp]),
    "mpsm_ipc_get_handle": (_int, [_vp, _vp, ctypes.POINTER(_i64)]),
    "mpsm_ipc_open_handle": (_int, [_vp, ctypes.POINTER(_vp)]),
    "mpsm_ipc_close_handle": (_int, [_vp]),
    "mpsm_relfile_header": (_int, [ctypes.c_char_p, ctypes.POINTER(_u64), ctypes.POINTER(_i64)]),
    "mpsm_relfile_read": (_int, [ctypes.c_char_p, _u64, _vp, _int]),
    "mpsm_relfile_read_columns": (_int, [ctypes.c_char_p, _u64, _vp, _vp, _int]),
    "mpsm_relfile_write": (_int, [ctypes.c_char_p, _vp, _vp, _u64]),
    "mpsm_deinterleave": (_int, [_vp, _i64, _vp, _vp, _vp]),
    "mpsm_upload_records": (_int, [_vp, _vp, _i64, _u64, _u64, _int, _vp, _int, _int, _vp, _vp,
                                   ctypes.POINTER(_i64), ctypes.POINTER(_int)]),
    "mpsm_sort_records": (_int, [_vp, _i64, _int, _vp, _vp, _vp, _sz, _vp]),
    "mpsm_sort_segments_workspace_bytes": (_int, [_i64, _int, _int, ctypes.POINTER(_sz)]),
    "mpsm_sort_pairs_segments": (_int, [_vp, _vp, _i64, _int, _vp, _u64, _u64, _int, _vp, _vp, _vp, _vp, _vp, _sz, _vp,
                                        _vp]),
    "mpsm_sort_packed_segments": (_int, [_vp, _vp, _i64, _int, _vp, _u64, _u64, _int, _vp, _vp, _vp, _sz, _vp, _vp,
                                         _vp]),
    "mpsm_sort_records_segments": (_int, [_vp, _i64, _int, _vp, _int, _vp, _vp, _vp, _sz, _vp]),
    "mpsm_sort_packed_dense": (_int, [_vp, _vp, _i64, _u64, _u64, _int, _vp, _vp, _vp, _sz, _vp, _vp, _vp, _vp]),
    "mpsm_sort_records_dense": (_int, [_vp, _i64, _int, _vp, _vp, _vp, _sz, _vp, _vp]),
    "mpsm_join_pairs_packed_hint": (_int, [ctypes.POINTER(RunDesc), _int, ctypes.POINTER(RunDesc), _int, _int, _u64,
                                           _int, _int, _vp, _i64, _vp, _vp, _sz, _vp, _vp, _i64, _vp]),
    "mpsm_upload_bytes": (_u64, [_int]),
    "mpsm_pack_records": (_int, [_vp, _vp, _i64, _u64, _u64, _int, _vp, _vp, _vp, _vp]),
    "mpsm_partition_records": (_int, [_vp, _vp, _i64, _u64, _u64, _int, _int, _vp, _int, _int, _vp, _vp, _sz, _vp,
                                      _vp, _vp]),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load the library (no CUDA calls).  Raises if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1207_0145_b200.build` "
                "(there is no CPU fallback)"
            )
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc == MPSM_OK:
        return
    msg = load().mpsm_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == ERR_DOMAIN:
        raise DomainError(text)
    if rc == ERR_INTERNAL:
        raise InternalConsistencyError(text)
    if rc == ERR_CONFIG:
        raise ConfigurationError(text)
    if rc == ERR_CAP:
        raise MaterializeCapExceeded(text)
    if rc == ERR_ARG:
        raise ValueError(text)
    if rc == ERR_IO:
        raise OSError(text)
    if rc == ERR_FORMAT:
        raise FormatError(text)
    raise RuntimeError(f"CUDA failure in {what}: {msg}")


def launch_count() -> int:
    return int(load().mpsm_launch_count())


def profile_enable(on: bool) -> None:
    check(load().mpsm_profile_enable(int(bool(on))), "mpsm_profile_enable")


def profile_read(name: str):
    """-> (total device ms, launches) of one kernel family since profile_enable."""
    ms = ctypes.c_double(0)
    n = ctypes.c_uint64(0)
    check(load().mpsm_profile_read(name.encode(), ctypes.byref(ms), ctypes.byref(n)), "mpsm_profile_read")
    return float(ms.value), int(n.value)


def runs_array(runs) -> ctypes.Array:
    """runs: iterable of (keys_ptr, pays_ptr, n) -> RunDesc[]"""
    runs = list(runs)
    arr = (RunDesc * max(len(runs), 1))()
    for i, (k, p, n) in enumerate(runs):
        arr[i].keys = k
        arr[i].pays = p
        arr[i].n = n
    return arr
