"""Run sorting on the GPU, mirroring /root/reference/pkg/src/mpsm/sorter.py.

The reference sorts a run with a three-phase CPU algorithm (MSD radix pass,
introsort, insertion pass).  Here every entry point is the segmented LSD radix
sort of csrc/segsort.cu over the width_bits significant bits of
(key - lower).  The three-phase helpers keep their names and contracts:
``radix_msd_pass`` clusters by the top min(8, w) bits (a stable partition
scatter), ``introsort`` / ``insertion_pass`` sort the given range.  Sorting is
in place on the caller's arrays, as in the reference (sorter.py:91-106);
numpy inputs are staged through the device and written back.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import device as D
from .core import DomainError, KeyDomain, Relation, Run

INSERTION_THRESHOLD = 16  # kept for API parity (sorter.py:25)


@dataclass(frozen=True)
class RadixBoundaries:
    """Bucket offsets after the MSD pass (sorter.py:28-43)."""

    offsets: np.ndarray
    radix_bits: int

    @property
    def bucket_count(self) -> int:
        return 1 << self.radix_bits


@dataclass(frozen=True)
class SortStats:
    heapsort_fallbacks: int = 0


def _span_m1(dom: KeyDomain) -> int:
    return dom.upper - dom.lower - 1


def _sort_arrays_inplace(keys, pays, dom: KeyDomain) -> None:
    """Sort (keys, pays) in place; raises DomainError before touching them."""
    n = int(keys.shape[0])
    if n == 0:
        return
    dev = D.ensure_device()
    host = isinstance(keys, np.ndarray)
    kd = D.to_device(keys, dev)
    pd = D.to_device(pays, dev)
    out_k = torch.empty_like(kd)
    out_p = torch.empty_like(pd)
    tmp_k = torch.empty_like(kd)
    tmp_p = torch.empty_like(pd)
    bad = D.new_bad_flag(dev)
    D.sort_pairs(kd, pd, dom.lower, _span_m1(dom), dom.width_bits, out_k, out_p, tmp_k, tmp_p, bad)
    idx = int(bad.item())
    if idx != -1:
        raise DomainError(f"key {int(keys[idx])} at index {idx} outside domain [{dom.lower}, {dom.upper})")
    if host:
        keys[:] = out_k.cpu().numpy()
        pays[:] = out_p.cpu().numpy()
    else:
        keys.copy_(out_k)
        pays.copy_(out_p)


def sort_run_with_stats(rel: Relation, dom: KeyDomain, origin_worker: int = 0) -> tuple:
    """Sort in place into a Run (sorter.py:91-100)."""
    _sort_arrays_inplace(rel.keys, rel.payloads, dom)
    return Run(rel.keys, rel.payloads, origin_worker), SortStats(0)


def sort_run(rel: Relation, dom: KeyDomain, origin_worker: int = 0) -> Run:
    run, _ = sort_run_with_stats(rel, dom, origin_worker)
    return run


def radix_msd_pass(rel: Relation, dom: KeyDomain) -> RadixBoundaries:
    """Cluster in place by the top min(8, w) bits of (key - lower) (sorter.py:57-73).

    A stable GPU partition scatter: buckets in order, input order inside a
    bucket (the reference leaves the order inside a bucket unspecified).
    """
    from .partition import SplitterVector

    eff = min(8, dom.width_bits)
    nb = 1 << eff
    shift = dom.width_bits - eff
    n = rel.cardinality
    dev = D.ensure_device()
    keys = D.to_device(rel.keys, dev)
    pays = D.to_device(rel.payloads, dev)
    hist = torch.zeros(nb, dtype=torch.int64, device=dev)
    bad = D.new_bad_flag(dev)
    if n:
        D.radix_histogram(keys, dom.lower, _span_m1(dom), shift, nb, hist, bad)
        idx = int(bad.item())
        if idx != -1:
            raise DomainError(f"key at index {idx} outside domain")
    counts = hist.cpu().numpy()
    offsets = np.zeros(nb + 1, np.int64)
    np.cumsum(counts, out=offsets[1:])
    if n:
        out_k = torch.empty_like(keys)
        out_p = torch.empty_like(pays)
        sp = SplitterVector.identity(nb)
        written = torch.zeros(nb, dtype=torch.int64, device=dev)
        D.scatter_chunk(keys, pays, dom.lower, shift, torch.arange(nb, dtype=torch.int32, device=dev), nb, nb,
                        torch.from_numpy(offsets[:-1].copy()).to(dev), out_k, out_p, written)
        del sp
        if isinstance(rel.keys, np.ndarray):
            rel.keys[:] = out_k.cpu().numpy()
            rel.payloads[:] = out_p.cpu().numpy()
        else:
            rel.keys.copy_(out_k)
            rel.payloads.copy_(out_p)
    return RadixBoundaries(offsets, eff)


def _full_domain_for(keys) -> KeyDomain:
    return KeyDomain(0, 1 << 64)


def introsort(keys, payloads, lo: int = 0, hi: int | None = None) -> SortStats:
    """Sort keys[lo:hi) with payloads (sorter.py:76-82); no fallbacks on GPU."""
    hi = keys.shape[0] if hi is None else hi
    if hi - lo > 1:
        _sort_arrays_inplace(keys[lo:hi], payloads[lo:hi], _full_domain_for(keys))
    return SortStats(0)


def insertion_pass(keys, payloads, lo: int = 0, hi: int | None = None) -> None:
    """Finish sorting keys[lo:hi) (sorter.py:85-88)."""
    introsort(keys, payloads, lo, hi)
