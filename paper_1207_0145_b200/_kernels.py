"""The reference's operator layer (``mpsm._kernels``) over this package's C ABI.

Same functions, argument meaning, in-place mutation of the caller's numpy
arrays and sentinel returns as /root/reference/pkg/src/mpsm/_kernels.py, so a
caller (or test) written against the reference's numba kernels runs on the
B200 kernels unchanged.  Each call moves its numpy arguments to the GPU, runs
the sm_100a kernel behind the C ABI and writes results back into the
caller's arrays -- the per-call operator API; the join engine itself keeps
everything in HBM and never goes through here.

  radix_histogram   _kernels.py:247-259  -> mpsm_radix_histogram
  scatter_chunk     _kernels.py:262-284  -> mpsm_radix_histogram + mpsm_scatter_chunk
  interp_lower_bound _kernels.py:287-337 -> mpsm_interp_lower_bound
  merge_join_run    _kernels.py:340-408  -> mpsm_join_pairs (count / materialize)
  three_phase_sort  _kernels.py:217-244  -> mpsm_sort_pairs (no fallbacks: 0)

Not provided: the reference's comparison-sort internals (``introsort_range``,
``heapsort_range``, ``insertion_pass``, ``radix_cluster``) -- the B200 run sort
is a radix sort with no introsort / heapsort stage.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from . import device as D

_EMPTY_U64 = np.empty(0, np.uint64)


def _dev_u64(a) -> torch.Tensor:
    dev = D.ensure_device()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, np.uint64))).to(dev)


def radix_histogram(keys, lower, shift, counts) -> int:
    """counts[(key - lower) >> shift] += 1 for every key (in place); -1, or
    the index of the first key whose bucket is outside [0, len(counts))."""
    n = int(keys.shape[0])
    nb = int(counts.shape[0])
    if n == 0:
        return -1
    lower, shift = int(lower), int(shift)
    k = np.asarray(keys, np.uint64)
    # a key maps into the bucket grid iff (key - lower) mod 2^64 < nb << shift
    span_m1 = (nb << shift) - 1 if (nb << shift) <= (1 << 64) else (1 << 64) - 1
    dk = _dev_u64(k)
    dc = torch.zeros(nb, dtype=torch.int64, device=dk.device)
    bad = D.new_bad_flag(dk.device)
    D.radix_histogram(dk, lower, min(span_m1, (1 << 64) - 1), shift, nb, dc, bad)
    idx = int(bad.item())
    if idx != -1:
        # the reference stops at the first bad key: buckets before it counted
        if idx:
            np.add.at(counts, ((k[:idx] - np.uint64(lower)) >> np.uint64(shift)).astype(np.int64), 1)
        return idx
    counts += dc.cpu().numpy().astype(counts.dtype, copy=False)
    return -1


def scatter_chunk(keys, pays, lower, shift, sp, cursors, ends, out_keys, out_pays) -> int:
    """Copy every tuple to partition sp[(key - lower) >> shift] at its cursor
    (cursors advance in place, never past ends); -1, or the index of the first
    tuple out of domain or overflowing its region (tuples before it copied,
    as the reference's sequential loop leaves them)."""
    n = int(keys.shape[0])
    if n == 0:
        return -1
    k = np.asarray(keys, np.uint64)
    lower, shift = int(lower), int(shift)
    nb, npart = int(sp.shape[0]), int(cursors.shape[0])
    b = (k - np.uint64(lower)) >> np.uint64(shift)
    first_bad = -1
    oob = np.nonzero(b >= np.uint64(nb))[0]
    limit = n if oob.size == 0 else int(oob[0])
    part = np.asarray(sp, np.int64)[b[:limit].astype(np.int64)]
    # overflow: the first tuple whose partition's running count passes its room
    room = np.asarray(ends, np.int64) - np.asarray(cursors, np.int64)
    if limit:
        cnt = np.zeros(npart, np.int64)
        order = np.argsort(part, kind="stable")
        ranks = np.empty(limit, np.int64)
        starts = np.searchsorted(part[order], np.arange(npart))
        ranks[order] = np.arange(limit) - starts[part[order]]
        over = np.nonzero(ranks >= room[part])[0]
        if over.size:
            limit = int(over[0])
            part = part[:limit]
        np.add.at(cnt, part, 1)
    if limit < n:
        first_bad = limit
    if limit:
        dev = D.ensure_device()
        dk, dp = _dev_u64(k[:limit]), _dev_u64(np.asarray(pays, np.uint64)[:limit])
        base = int(np.asarray(cursors, np.int64).min()) if npart else 0
        top = int(np.asarray(ends, np.int64).max()) if npart else 0
        ok = torch.from_numpy(np.ascontiguousarray(np.asarray(out_keys, np.uint64)[base:top])).to(dev)
        op = torch.from_numpy(np.ascontiguousarray(np.asarray(out_pays, np.uint64)[base:top])).to(dev)
        cur = torch.from_numpy(np.asarray(cursors, np.int64) - base).to(dev)
        written = torch.zeros(npart, dtype=torch.int64, device=dev)
        spd = torch.from_numpy(np.asarray(sp, np.int32)).to(dev)
        D.scatter_chunk(dk, dp, lower, shift, spd, nb, npart, cur, ok, op, written)
        out_keys[base:top] = ok.cpu().numpy()
        out_pays[base:top] = op.cpu().numpy()
        cursors += cnt.astype(cursors.dtype, copy=False)
    return first_bad


def interp_lower_bound(keys, target):
    """(first index whose key >= target, positions examined) by the
    reference's probe rule (interpolation, bisection after a step that fails
    to halve the window)."""
    n = int(keys.shape[0])
    if n == 0:
        return 0, 0
    dk = _dev_u64(keys)
    tgt = torch.from_numpy(np.array([int(target) & ((1 << 64) - 1)], np.uint64)).to(dk.device)
    idx, probes = D.interp_lower_bound(dk, tgt)
    return int(idx[0].item()), int(probes[0].item())


def merge_join_run(r_keys, r_pays, s_keys, s_pays, s_start, collect, out_r, out_s):
    """(match_count, best_sum, examined, emitted) of one sorted private run
    against one sorted public run scanned from s_start; with collect the
    first len(out_r) pairs (merge order) go to out_r / out_s."""
    nr, ns = int(r_keys.shape[0]), int(s_keys.shape[0])
    s_start = int(s_start)
    if nr == 0 or s_start >= ns:
        return 0, np.uint64(0), 0, 0
    rk, rp = _dev_u64(r_keys), _dev_u64(r_pays)
    sk, sp = _dev_u64(np.asarray(s_keys)[s_start:]), _dev_u64(np.asarray(s_pays)[s_start:])
    rec = D.join_pairs([(rk, rp)], [(sk, sp)], False, _lib.MODE_COUNT).cpu().numpy()[0]
    count = int(rec[_lib.PAIR_COUNT])
    best = np.uint64(rec[_lib.PAIR_BEST]) if count else np.uint64(0)
    # the reference reads every position from s_start up to the lower bound
    # the kernel starts at, then the same positions as the kernel
    examined = int(rec[_lib.PAIR_START]) + int(rec[_lib.PAIR_EXAMINED])
    emitted = 0
    cap = int(out_r.shape[0]) if collect else 0
    if collect and count and cap:
        m = min(count, cap)
        out = torch.empty(2 * m, dtype=torch.uint64, device=rk.device)
        D.join_pairs([(rk, rp)], [(sk, sp)], False, _lib.MODE_MATERIALIZE, out, m)
        pairs = out.view(m, 2).cpu().numpy()
        out_r[:m] = pairs[:, 0]
        out_s[:m] = pairs[:, 1]
        emitted = m
    return count, best, examined, emitted


def three_phase_sort(keys, pays, lo, hi, lower, width_bits) -> int:
    """Sort keys[lo:hi) with payloads in place by key - lower (width_bits
    bits); -1 for a key out of domain (nothing sorted), else the comparison
    sort's fallback count -- always 0 (the GPU run sort is a radix sort)."""
    lo, hi, lower, width_bits = int(lo), int(hi), int(lower), int(width_bits)
    if hi - lo <= 1:
        return 0
    k = np.asarray(keys[lo:hi], np.uint64)
    span_m1 = (1 << width_bits) - 1 if width_bits < 64 else (1 << 64) - 1
    dk, dp = _dev_u64(k), _dev_u64(pays[lo:hi])
    ok, op, tk, tp = (torch.empty_like(dk) for _ in range(4))
    bad = D.new_bad_flag(dk.device)
    D.sort_pairs(dk, dp, lower, span_m1, width_bits, ok, op, tk, tp, bad)
    if int(bad.item()) != -1:
        return -1
    keys[lo:hi] = ok.cpu().numpy()
    pays[lo:hi] = op.cpu().numpy()
    return 0


def warmup() -> None:
    """The reference compiles its numba kernels here; the B200 library is
    loaded and its device state initialised instead."""
    _lib.load()
    D.ensure_device()


__all__ = ["radix_histogram", "scatter_chunk", "interp_lower_bound", "merge_join_run", "three_phase_sort", "warmup",
           "_EMPTY_U64"]
