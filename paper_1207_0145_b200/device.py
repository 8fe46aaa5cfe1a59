"""Device-side operators: torch tensors in, C-ABI calls out.

PyTorch is only the carrier here (device memory, streams); every operator is
a call into libmpsm_b200.so.  Buffers are uint64 torch tensors on one CUDA
device; pointers and the current stream go through ctypes as plain integers.
"""

from __future__ import annotations

import ctypes
import threading
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from .core import ConfigurationError

U64 = torch.uint64
I64 = torch.int64

_init_lock = threading.Lock()
_inited = {}


_READY: dict = {}  # device index -> torch.device, once initialised


def ensure_device(device: Optional[torch.device] = None) -> torch.device:
    """Select the CUDA device and verify it is a B200 (sm_100).  Raises if none."""
    if device is None and _READY:  # per-join fast path: the current device, already initialised
        d = _READY.get(torch.cuda.current_device())
        if d is not None:
            return d
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1207_0145_b200 needs a CUDA device (B200); none is visible and there is no CPU path")
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    with _init_lock:
        if dev.index not in _inited:
            lib = _lib.load()
            with torch.cuda.device(dev):
                rc = lib.mpsm_device_init(dev.index)
            if rc < 0:
                _lib.check(rc, "mpsm_device_init")
            _inited[dev.index] = rc
            _READY[dev.index] = dev
    return dev


def stream_ptr(stream: Optional[torch.cuda.Stream] = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    if t is None:
        return None
    return int(t.data_ptr()) if t.numel() else None


class Workspace:
    """Grow-only scratch buffer per device (stream-ordered reuse)."""

    def __init__(self, device: torch.device):
        self.device = device
        self.buf = torch.empty(0, dtype=torch.uint8, device=device)

    def get(self, nbytes: int) -> torch.Tensor:
        nbytes = max(int(nbytes), 256)
        if self.buf.numel() < nbytes:
            self.buf = torch.empty(int(nbytes * 1.25) + 4096, dtype=torch.uint8, device=self.device)
        return self.buf


_ws = {}


def workspace(device: torch.device) -> Workspace:
    if device.index not in _ws:
        _ws[device.index] = Workspace(device)
    return _ws[device.index]


_WS_BYTES: dict = {}


def _sort_ws_bytes(n: int, width_bits: int) -> int:
    """mpsm_sort_workspace_bytes, memoised (a per-join ctypes round trip)"""
    key = (n, width_bits)
    v = _WS_BYTES.get(key)
    if v is None:
        sz = ctypes.c_size_t(0)
        _lib.check(_lib.load().mpsm_sort_workspace_bytes(n, width_bits, ctypes.byref(sz)), "sort workspace")
        v = int(sz.value)
        if len(_WS_BYTES) > 256:
            _WS_BYTES.clear()
        _WS_BYTES[key] = v
    return v


def new_bad_flag(device: torch.device) -> torch.Tensor:
    """int64[1] = -1 (all ones == UINT64_MAX: no out-of-domain key seen)."""
    return torch.full((1,), -1, dtype=I64, device=device)


_FLAGS_INIT = None


def new_join_flags(device: torch.device) -> torch.Tensor:
    """int64[3] = (-1, -1, 0): the public and private sides' out-of-domain
    flags (as new_bad_flag) and the payload-overflow flag (an int32 in the low
    half of the last word), set by one copy from a pinned template -- the
    per-join flags without a kernel launch each."""
    global _FLAGS_INIT
    if _FLAGS_INIT is None:
        _FLAGS_INIT = torch.tensor([-1, -1, 0], dtype=I64).pin_memory()
    f = torch.empty(3, dtype=I64, device=device)
    f.copy_(_FLAGS_INIT, non_blocking=True)
    return f


# ---------------------------------------------------------------- operators

def sort_pairs(in_k: torch.Tensor, in_p: torch.Tensor, lower: int, span_m1: int, width_bits: int,
               out_k: torch.Tensor, out_p: torch.Tensor, tmp_k: torch.Tensor, tmp_p: torch.Tensor,
               bad: Optional[torch.Tensor] = None) -> None:
    n = int(in_k.numel())
    if n == 0:
        return
    L = _lib.load()
    sz = ctypes.c_size_t(0)
    _lib.check(L.mpsm_sort_workspace_bytes(n, width_bits, ctypes.byref(sz)), "sort workspace")
    ws = workspace(in_k.device).get(sz.value)
    _lib.check(L.mpsm_sort_pairs(ptr(in_k), ptr(in_p), n, lower, span_m1, width_bits, ptr(out_k), ptr(out_p),
                                 ptr(tmp_k), ptr(tmp_p), ptr(ws), ws.numel(), ptr(bad), stream_ptr()),
               "mpsm_sort_pairs")


def sort_packed(in_k: torch.Tensor, in_p: torch.Tensor, lower: int, span_m1: int, width_bits: int,
                out_rec: torch.Tensor, tmp_rec: torch.Tensor, bad: Optional[torch.Tensor],
                overflow: torch.Tensor, dense: Optional[torch.Tensor] = None) -> None:
    """Sort into packed records (key - lower) << (64 - w) | payload; sets
    overflow[0] = 1 if a payload does not fit (caller falls back to SoA).
    dense (uint32[2], optional): the density probe of the sorted output
    (mpsm_sort_packed_dense)."""
    n = int(in_k.numel())
    L = _lib.load()
    if n == 0:
        if dense is not None:
            dense.copy_(torch.tensor([1, 0], dtype=torch.int32).view(torch.uint32))
        return
    ws = workspace(in_k.device).get(_sort_ws_bytes(n, width_bits))
    if dense is not None:
        _lib.check(L.mpsm_sort_packed_dense(ptr(in_k), ptr(in_p), n, lower, span_m1, width_bits, ptr(out_rec),
                                            ptr(tmp_rec), ptr(ws), ws.numel(), ptr(bad), ptr(overflow), ptr(dense),
                                            stream_ptr()), "mpsm_sort_packed_dense")
        return
    _lib.check(L.mpsm_sort_packed(ptr(in_k), ptr(in_p), n, lower, span_m1, width_bits, ptr(out_rec), ptr(tmp_rec),
                                  ptr(ws), ws.numel(), ptr(bad), ptr(overflow), stream_ptr()), "mpsm_sort_packed")


def sort_records(in_rec: torch.Tensor, width_bits: int, out_rec: torch.Tensor, tmp_rec: torch.Tensor,
                 dense: Optional[torch.Tensor] = None) -> None:
    """Sort packed records (key in the top width_bits bits); in, out, tmp
    distinct (in == out for an even pass count); dense as for sort_packed."""
    n = int(in_rec.numel())
    L = _lib.load()
    if n == 0:
        if dense is not None:
            dense.copy_(torch.tensor([1, 0], dtype=torch.int32).view(torch.uint32))
        return
    ws = workspace(in_rec.device).get(_sort_ws_bytes(n, width_bits))
    if dense is not None:
        _lib.check(L.mpsm_sort_records_dense(ptr(in_rec), n, width_bits, ptr(out_rec), ptr(tmp_rec), ptr(ws),
                                             ws.numel(), ptr(dense), stream_ptr()), "mpsm_sort_records_dense")
        return
    _lib.check(L.mpsm_sort_records(ptr(in_rec), n, width_bits, ptr(out_rec), ptr(tmp_rec), ptr(ws), ws.numel(),
                                   stream_ptr()), "mpsm_sort_records")


def _seg_ws(dev, n: int, nseg: int, width_bits: int) -> torch.Tensor:
    L = _lib.load()
    sz = ctypes.c_size_t(0)
    _lib.check(L.mpsm_sort_segments_workspace_bytes(n, nseg, width_bits, ctypes.byref(sz)), "sort workspace")
    return workspace(dev).get(sz.value)


def _offsets(offsets) -> np.ndarray:
    return np.ascontiguousarray(offsets, dtype=np.int64)


def sort_packed_segments(in_k, in_p, offsets, lower: int, span_m1: int, width_bits: int, out_rec, tmp_rec, bad,
                         overflow) -> None:
    """len(offsets) - 1 independent packed sorts of [offsets[s], offsets[s+1])
    in one launch sequence (segment s -> run s, in place of position)"""
    n = int(in_k.numel())
    if n == 0:
        return
    off = _offsets(offsets)
    ws = _seg_ws(in_k.device, n, off.shape[0] - 1, width_bits)
    _lib.check(_lib.load().mpsm_sort_packed_segments(ptr(in_k), ptr(in_p), n, off.shape[0] - 1, off.ctypes.data, lower,
                                                     span_m1, width_bits, ptr(out_rec), ptr(tmp_rec), ptr(ws),
                                                     ws.numel(), ptr(bad), ptr(overflow), stream_ptr()),
               "mpsm_sort_packed_segments")


def sort_records_segments(in_rec, offsets, width_bits: int, out_rec, tmp_rec) -> None:
    n = int(in_rec.numel())
    if n == 0:
        return
    off = _offsets(offsets)
    ws = _seg_ws(in_rec.device, n, off.shape[0] - 1, width_bits)
    _lib.check(_lib.load().mpsm_sort_records_segments(ptr(in_rec), n, off.shape[0] - 1, off.ctypes.data, width_bits,
                                                      ptr(out_rec), ptr(tmp_rec), ptr(ws), ws.numel(), stream_ptr()),
               "mpsm_sort_records_segments")


def sort_pairs_segments(in_k, in_p, offsets, lower: int, span_m1: int, width_bits: int, out_k, out_p, tmp_k, tmp_p,
                        bad) -> None:
    n = int(in_k.numel())
    if n == 0:
        return
    off = _offsets(offsets)
    ws = _seg_ws(in_k.device, n, off.shape[0] - 1, width_bits)
    _lib.check(_lib.load().mpsm_sort_pairs_segments(ptr(in_k), ptr(in_p), n, off.shape[0] - 1, off.ctypes.data, lower,
                                                    span_m1, width_bits, ptr(out_k), ptr(out_p), ptr(tmp_k),
                                                    ptr(tmp_p), ptr(ws), ws.numel(), ptr(bad), stream_ptr()),
               "mpsm_sort_pairs_segments")


def pack_records(keys: torch.Tensor, pays: torch.Tensor, lower: int, span_m1: int, width_bits: int,
                 out_rec: torch.Tensor, bad: torch.Tensor, overflow: torch.Tensor) -> None:
    """device columns -> packed records; domain / payload-width flags on device"""
    n = int(keys.numel())
    if n == 0:
        return
    _lib.check(_lib.load().mpsm_pack_records(ptr(keys), ptr(pays), n, lower, span_m1, width_bits, ptr(out_rec),
                                             ptr(bad), ptr(overflow), stream_ptr()), "mpsm_pack_records")


def partition_records(keys: torch.Tensor, pays: torch.Tensor, lower: int, span_m1: int, width_bits: int, shift: int,
                      sp: torch.Tensor, npart: int, out_rec: torch.Tensor, bad: torch.Tensor,
                      overflow: torch.Tensor) -> None:
    """private shard -> packed records grouped by partition (stable); sp:
    int32 splitter vector (bucket -> partition) on the device"""
    n = int(keys.numel())
    if n == 0:
        return
    L = _lib.load()
    sz = ctypes.c_size_t(0)
    _lib.check(L.mpsm_sort_workspace_bytes(n, width_bits, ctypes.byref(sz)), "sort workspace")
    ws = workspace(keys.device).get(sz.value)
    _lib.check(L.mpsm_partition_records(ptr(keys), ptr(pays), n, lower, span_m1, width_bits, shift, ptr(sp),
                                        int(sp.numel()), npart, ptr(out_rec), ptr(ws), ws.numel(), ptr(bad),
                                        ptr(overflow), stream_ptr()), "mpsm_partition_records")


def host_columns(a):
    """A host uint64 column as (keep-alive object, address), or None if `a`
    is not host-resident."""
    if isinstance(a, torch.Tensor):
        if a.device.type != "cpu":
            return None
        t = a.contiguous()
        if t.dtype not in (U64, torch.int64):
            return None
        return t, t.data_ptr()
    arr = np.ascontiguousarray(a)
    if arr.dtype not in (np.uint64, np.int64) or arr.ndim != 1:
        return None
    return arr, arr.ctypes.data


def upload_records(keys, pays, lower: int, span_m1: int, width_bits: int, out_rec: torch.Tensor,
                   threads: int = 0, gpu_pack_every: int = -1, ready: Optional[torch.cuda.Event] = None) -> tuple:
    """Host (key, payload) columns -> packed records on the device (half the
    PCIe bytes).  gpu_pack_every: every k-th chunk packed by the GPU from the
    mapped (pinned) columns; 0 = host only (use while the GPU is busy), -1 =
    default.  ready: event recorded when out_rec was allocated (the copies need
    not wait for work queued after it).  -> (first out-of-domain index or -1,
    payload overflow)."""
    hk, hp = host_columns(keys), host_columns(pays)
    n = int(out_rec.numel())
    bad = ctypes.c_int64(-1)
    ovf = ctypes.c_int(0)
    _lib.check(_lib.load().mpsm_upload_records(hk[1] if n else None, hp[1] if n else None, n, lower, span_m1,
                                               width_bits, ptr(out_rec), threads, gpu_pack_every, stream_ptr(),
                                               ready.cuda_event if ready is not None else None, ctypes.byref(bad),
                                               ctypes.byref(ovf)), "mpsm_upload_records")
    return int(bad.value), bool(ovf.value)


def radix_histogram(keys: torch.Tensor, lower: int, span_m1: int, shift: int, nbuckets: int,
                    counts: torch.Tensor, bad: Optional[torch.Tensor] = None) -> None:
    n = int(keys.numel())
    if n == 0:
        return
    _lib.check(_lib.load().mpsm_radix_histogram(ptr(keys), n, lower, span_m1, shift, nbuckets, ptr(counts), ptr(bad),
                                                stream_ptr()), "mpsm_radix_histogram")


def domain_report(keys: torch.Tensor, lower: int, span_m1: int) -> tuple:
    """(violation count, first index or -1) of a device key column
    (core.validate_relation's counts, computed on the GPU; synchronises)"""
    rep = torch.empty(2, dtype=U64, device=keys.device)
    _lib.check(_lib.load().mpsm_domain_report(ptr(keys), int(keys.numel()), lower, span_m1, ptr(rep), stream_ptr()),
               "mpsm_domain_report")
    cnt, first = (int(x) for x in rep.view(I64).cpu().tolist())
    return cnt, (first if cnt else -1)


def is_sorted(keys: torch.Tensor) -> bool:
    """keys[i] <= keys[i + 1] for all i (device check; synchronises)"""
    flag = torch.zeros(1, dtype=torch.int32, device=keys.device)
    _lib.check(_lib.load().mpsm_check_sorted(ptr(keys), int(keys.numel()), ptr(flag), stream_ptr()),
               "mpsm_check_sorted")
    return int(flag.item()) == 0


def scatter_chunk(keys, pays, lower: int, shift: int, sp: torch.Tensor, nbuckets: int, npart: int,
                  cursors: torch.Tensor, arena_k, arena_p, written: torch.Tensor) -> None:
    n = int(keys.numel())
    if n == 0:
        return
    L = _lib.load()
    sz = ctypes.c_size_t(0)
    _lib.check(L.mpsm_scatter_workspace_bytes(n, npart, ctypes.byref(sz)), "scatter workspace")
    ws = workspace(keys.device).get(sz.value)
    _lib.check(L.mpsm_scatter_chunk(ptr(keys), ptr(pays), n, lower, shift, ptr(sp), nbuckets, npart, ptr(cursors),
                                    ptr(arena_k), ptr(arena_p), ptr(written), ptr(ws), ws.numel(), stream_ptr()),
               "mpsm_scatter_chunk")


def interp_lower_bound(keys: torch.Tensor, targets: torch.Tensor):
    """-> (index int64 tensor, probes int64 tensor)"""
    nt = int(targets.numel())
    idx = torch.empty(nt, dtype=I64, device=keys.device)
    probes = torch.empty(nt, dtype=I64, device=keys.device)
    if nt:
        _lib.check(_lib.load().mpsm_interp_lower_bound(ptr(keys) or 0, int(keys.numel()), ptr(targets), nt, ptr(idx),
                                                       ptr(probes), stream_ptr()), "mpsm_interp_lower_bound")
    return idx, probes


def _run_descs(runs: Sequence[tuple]):
    return _lib.runs_array((ptr(k) or 0, ptr(p) or 0, int(k.numel())) for k, p in runs)


def join_pairs(priv: Sequence[tuple], pub: Sequence[tuple], swap: bool, mode: int,
               out: Optional[torch.Tensor] = None, cap: int = 0) -> torch.Tensor:
    """Merge-join every private run against every public run.

    priv/pub: sequences of (keys, pays) device tensors (sorted runs).
    Returns the uint64 [n_priv * n_pub, PAIR_FIELDS] pair-record tensor (device).
    """
    dev = (priv[0][0] if priv else pub[0][0]).device
    pa, ua = _run_descs(priv), _run_descs(pub)
    L = _lib.load()
    sz = ctypes.c_size_t(0)
    _lib.check(L.mpsm_join_workspace_bytes(pa, len(priv), ua, len(pub), ctypes.byref(sz)), "join workspace")
    ws = workspace(dev).get(sz.value)
    rec = torch.empty((len(priv) * len(pub), _lib.PAIR_FIELDS), dtype=U64, device=dev)
    _lib.check(L.mpsm_join_pairs(pa, len(priv), ua, len(pub), int(bool(swap)), int(mode), ptr(out), int(cap),
                                 ptr(rec), ptr(ws), ws.numel(), stream_ptr()), "mpsm_join_pairs")
    return rec


def join_pairs_packed(priv: Sequence[torch.Tensor], pub: Sequence[torch.Tensor], width_bits: int, lower: int,
                      swap: bool, mode: int, out: Optional[torch.Tensor] = None, cap: int = 0,
                      hint: Optional[tuple] = None) -> torch.Tensor:
    """join_pairs over runs of packed records (one uint64 tensor per run).
    hint: (dense uint32[2], whole sorted private array) the runs were cut
    from -- the density probe of its sort (mpsm_join_pairs_packed_hint)."""
    dev = (priv[0] if priv else pub[0]).device
    pa = _lib.runs_array((ptr(k) or 0, 0, int(k.numel())) for k in priv)
    ua = _lib.runs_array((ptr(k) or 0, 0, int(k.numel())) for k in pub)
    L = _lib.load()
    sz = ctypes.c_size_t(0)
    _lib.check(L.mpsm_join_workspace_bytes(pa, len(priv), ua, len(pub), ctypes.byref(sz)), "join workspace")
    ws = workspace(dev).get(sz.value)
    rec = torch.empty((len(priv) * len(pub), _lib.PAIR_FIELDS), dtype=U64, device=dev)
    if hint is not None:
        dense, base = hint
        _lib.check(L.mpsm_join_pairs_packed_hint(pa, len(priv), ua, len(pub), width_bits, lower, int(bool(swap)),
                                                 int(mode), ptr(out), int(cap), ptr(rec), ptr(ws), ws.numel(),
                                                 ptr(dense), ptr(base), int(base.numel()), stream_ptr()),
                   "mpsm_join_pairs_packed_hint")
        return rec
    _lib.check(L.mpsm_join_pairs_packed(pa, len(priv), ua, len(pub), width_bits, lower, int(bool(swap)), int(mode),
                                        ptr(out), int(cap), ptr(rec), ptr(ws), ws.numel(), stream_ptr()),
               "mpsm_join_pairs_packed")
    return rec


def minmax_contiguous(n: int, t: int, prefix: np.ndarray, edge: np.ndarray, cand: np.ndarray) -> list:
    prefix = np.ascontiguousarray(prefix, np.int64)
    edge = np.ascontiguousarray(edge, np.float64)
    cand = np.ascontiguousarray(cand, np.float64)
    out = np.zeros(t + 1, np.int64)
    rc = _lib.load().mpsm_minmax_contiguous(n, t, prefix.ctypes.data, edge.ctypes.data, cand.ctypes.data,
                                            cand.shape[0], out.ctypes.data)
    if rc == _lib.ERR_CONFIG:
        raise ConfigurationError(f"cannot split {n} buckets into {t} partitions")
    _lib.check(rc, "mpsm_minmax_contiguous")
    return out.tolist()


def to_device(a, device: torch.device, non_blocking: bool = False) -> torch.Tensor:
    """numpy uint64 / torch tensor -> contiguous uint64 tensor on device."""
    if isinstance(a, torch.Tensor):
        t = a if a.device == device else a.to(device, non_blocking=non_blocking)
        return t.contiguous()
    arr = np.ascontiguousarray(a, np.uint64)
    if arr.shape[0] == 0:
        return torch.empty(0, dtype=U64, device=device)
    return torch.from_numpy(arr).to(device, non_blocking=non_blocking)
