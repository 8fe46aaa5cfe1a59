"""Relation files: the reference's MPSMREL1 format on the B200 input path.

Layout (``/root/reference/pkg/src/mpsm/bench.py:8-11``): magic ``MPSMREL1``,
u64 tuple count n, then n little-endian (key u64, payload u64) records.
``read_relation`` / ``write_relation`` keep the reference's semantics
(``bench.py:73-102``: exact-length check, ``FormatError`` with the byte
offset); the work is native (``csrc/relfile.cpp``: parallel ``pread``).
``load_relation`` is the device path: records land in pinned host memory,
move to HBM in one copy and are split into SoA columns on the GPU
(``mpsm_deinterleave``), ready for ``run_join``.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib
from .core import FormatError, Relation

MAGIC = b"MPSMREL1"


def _path(path) -> bytes:
    return os.fsencode(os.fspath(path))


def read_header(path) -> int:
    """Check magic and exact length like bench.read_relation; return n."""
    with open(path, "rb"):  # same OSError as the reference's open()
        pass
    n = ctypes.c_uint64(0)
    off = ctypes.c_int64(-1)
    rc = _lib.load().mpsm_relfile_header(_path(path), ctypes.byref(n), ctypes.byref(off))
    if rc == _lib.ERR_FORMAT:
        raise FormatError(_lib.load().mpsm_last_error().decode(errors="replace"), byte_offset=int(off.value))
    _lib.check(rc, "mpsm_relfile_header")
    return int(n.value)


def _read_records(path, n: int, dst_ptr: int, threads: int = 0) -> None:
    _lib.check(_lib.load().mpsm_relfile_read(_path(path), n, dst_ptr, threads), "mpsm_relfile_read")


def read_relation(path, threads: int = 0) -> Relation:
    """Load a relation into host memory (numpy), checking magic and length;
    the reading threads split the records into the two columns."""
    n = read_header(path)
    keys = np.empty(n, dtype="<u8")
    pays = np.empty(n, dtype="<u8")
    if n:
        _lib.check(_lib.load().mpsm_relfile_read_columns(_path(path), n, keys.ctypes.data, pays.ctypes.data, threads),
                   "mpsm_relfile_read_columns")
    return Relation(keys, pays)


def write_relation(rel: Relation, path) -> None:
    """Persist a relation bit-exactly (reference bench.write_relation)."""
    keys, pays = rel.keys, rel.payloads
    if hasattr(keys, "device") and getattr(keys.device, "type", "cpu") != "cpu":
        keys, pays = keys.cpu(), pays.cpu()
    keys = np.ascontiguousarray(np.asarray(keys).view(np.uint64))
    pays = np.ascontiguousarray(np.asarray(pays).view(np.uint64))
    _lib.check(_lib.load().mpsm_relfile_write(_path(path), keys.ctypes.data, pays.ctypes.data, int(keys.size)),
               "mpsm_relfile_write")


def load_relation(path, device=None, threads: int = 0) -> Relation:
    """Relation file -> pinned host buffer -> HBM -> SoA columns on the GPU."""
    import torch

    from . import device as D

    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    n = read_header(path)
    keys = torch.empty(n, dtype=torch.uint64, device=dev)
    pays = torch.empty(n, dtype=torch.uint64, device=dev)
    if n == 0:
        return Relation(keys, pays)
    host = torch.empty(2 * n, dtype=torch.int64, pin_memory=True)
    _read_records(path, n, host.data_ptr(), threads)
    rec = torch.empty(2 * n, dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        D.ensure_device()
        rec.copy_(host, non_blocking=True)
        _lib.check(_lib.load().mpsm_deinterleave(rec.data_ptr(), n, keys.data_ptr(), pays.data_ptr(),
                                                  D.stream_ptr()), "mpsm_deinterleave")
        torch.cuda.current_stream(dev).synchronize()
    return Relation(keys, pays)
