"""Skew-resilient splitters from the public CDF and the private histogram.

Mirrors /root/reference/pkg/src/mpsm/skew.py.  The numpy pieces (bounds,
CDF, edge evaluation, candidate costs) are the reference's own vectorised
float64 operations, evaluated the same way so the values are bit-identical;
the search over bucket ranges (the reference's pure-Python hot loop,
skew.py:180-273, ~15 ms at B=10/T=8) runs in C++ (csrc/splitters.cpp) via
mpsm_minmax_contiguous.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import device as D
from .core import ConfigurationError, KeyDomain, Run
from .partition import SplitterVector, bucket_lower_key

EXACT_SEARCH_MAX_BUCKETS = 256


@dataclass(frozen=True)
class LocalBounds:
    """Equi-height sample of one sorted public run (skew.py:32-49)."""

    bound_keys: np.ndarray
    run_size: int

    @property
    def n_bounds(self) -> int:
        return int(self.bound_keys.shape[0])

    @property
    def weight_per_bound(self) -> float:
        return self.run_size / self.n_bounds if self.n_bounds else 0.0


def bound_positions(n: int, f: int, t: int) -> np.ndarray:
    k = f * t
    ms = np.arange(1, k + 1, dtype=np.int64)
    return (n * ms + k - 1) // k - 1


def local_equiheight_bounds(run: Run, f: int, t: int) -> LocalBounds:
    """Keys at ranks ceil(n*m/k)-1, k=f*t (skew.py:52-62)."""
    k = f * t
    if k < 1:
        raise ConfigurationError("f * T must be >= 1")
    n = run.cardinality
    if n == 0:
        return LocalBounds(np.empty(0, np.uint64), 0)
    pos = bound_positions(n, f, t)
    keys = run.keys
    if isinstance(keys, np.ndarray):
        return LocalBounds(keys[pos].copy(), n)
    import torch

    return LocalBounds(keys.view(torch.int64)[torch.from_numpy(pos).to(keys.device)].cpu().numpy().view(np.uint64), n)


@dataclass(frozen=True)
class Cdf:
    """Global step function of public tuples below a key (skew.py:65-113)."""

    step_keys: np.ndarray
    step_cum: np.ndarray
    total: int
    anchor_key: int = 0

    def eval_many(self, probe_keys: np.ndarray) -> np.ndarray:
        keys = self.step_keys
        n = keys.shape[0]
        probes = np.asarray(probe_keys, np.uint64)
        out = np.zeros(probes.shape[0], np.float64)
        if n == 0 or self.total == 0:
            return out
        idx = np.searchsorted(keys, probes, side="left")
        above = idx >= n
        out[above] = float(self.total)
        inside = ~above
        ii = idx[inside]
        pk = probes[inside]
        hi_key = keys[ii]
        hi_cum = self.step_cum[ii]
        exact = hi_key == pk
        lo_key = np.where(ii > 0, keys[np.maximum(ii - 1, 0)], np.uint64(self.anchor_key))
        lo_cum = np.where(ii > 0, self.step_cum[np.maximum(ii - 1, 0)], 0.0)
        below = pk <= np.uint64(self.anchor_key)
        denom = (hi_key - lo_key).astype(np.float64)
        denom[denom == 0] = 1.0
        frac = (pk - lo_key).astype(np.float64) / denom
        vals = lo_cum + frac * (hi_cum - lo_cum)
        vals = np.where(below, 0.0, vals)
        vals = np.where(exact, hi_cum, vals)
        out[inside] = vals
        return out

    def eval(self, key: int) -> float:
        key = min(max(int(key), 0), (1 << 64) - 1)
        return float(self.eval_many(np.array([key], np.uint64))[0])


def build_cdf(all_bounds: Sequence[LocalBounds], *, anchor_key: int = 0) -> Cdf:
    """Merge per-worker bounds into the global CDF (skew.py:116-141)."""
    keys_parts, weight_parts, total = [], [], 0
    for lb in all_bounds:
        total += lb.run_size
        if lb.n_bounds:
            keys_parts.append(lb.bound_keys)
            weight_parts.append(np.full(lb.n_bounds, lb.weight_per_bound))
    if not keys_parts:
        return Cdf(np.empty(0, np.uint64), np.empty(0, np.float64), total, anchor_key)
    keys = np.concatenate(keys_parts)
    weights = np.concatenate(weight_parts)
    order = np.argsort(keys, kind="stable")
    keys = keys[order]
    cum = np.cumsum(weights[order])
    keep = np.empty(keys.shape[0], bool)
    keep[:-1] = keys[:-1] != keys[1:]
    keep[-1] = True
    return Cdf(keys[keep], cum[keep], total, anchor_key)


def cdf_eval(cdf: Cdf, key: int) -> float:
    return cdf.eval(key)


def split_relevant_cost(n_private: int, t: int, s_span: float) -> float:
    """skew.py:148-153"""
    if s_span < 0:
        raise ValueError("s_span must be non-negative")
    sort_cost = n_private * math.log2(n_private) if n_private > 0 else 0.0
    return sort_cost + t * n_private + s_span


@dataclass(frozen=True)
class SplitterSet:
    """T-1 splitter keys at bucket granularity plus derived artifacts (skew.py:156-177)."""

    splitter_keys: np.ndarray
    bucket_bounds: np.ndarray
    vector: SplitterVector
    partition_sizes: np.ndarray
    partition_costs: np.ndarray

    @property
    def n_partitions(self) -> int:
        return int(self.partition_sizes.shape[0])

    @property
    def max_cost(self) -> float:
        return float(self.partition_costs.max())


def _edge_cdf(cdf: Cdf, dom: KeyDomain, radix_bits: int) -> np.ndarray:
    """CDF at every bucket-edge key (skew.py:276-284)."""
    n = 1 << radix_bits
    sh = dom.width_bits - radix_bits
    top = (1 << 64) - 1
    if dom.lower + (n << sh) <= top:  # no edge saturates: exact in u64
        edges = np.uint64(dom.lower) + (np.arange(n + 1, dtype=np.uint64) << np.uint64(sh))
    else:
        edges = np.array([min(dom.lower + (e << sh), top) for e in range(n + 1)], np.uint64)
    return cdf.eval_many(edges)


def _prefix(r_hist: np.ndarray) -> np.ndarray:
    prefix = np.zeros(r_hist.shape[0] + 1, np.int64)
    np.cumsum(r_hist, out=prefix[1:])
    return prefix


def _check(n: int, t: int, radix_bits: int) -> None:
    if n != 1 << radix_bits:
        raise ConfigurationError("histogram length must be 2^radix_bits")
    if n < t:
        raise ConfigurationError(f"buckets ({n}) must be >= partitions ({t})")


def compute_splitters(r_hist: np.ndarray, cdf: Cdf, t: int, dom: KeyDomain, radix_bits: int) -> SplitterSet:
    """Min-max split-relevant-cost splitters (skew.py:287-315); search in C++."""
    r_hist = np.asarray(r_hist, np.int64)
    n = int(r_hist.shape[0])
    _check(n, t, radix_bits)
    prefix = _prefix(r_hist)
    edge = _edge_cdf(cdf, dom, radix_bits)

    def batch_costs(a: np.ndarray, b: np.ndarray) -> np.ndarray:  # skew.py:306-312, numpy float ops
        sizes = (prefix[b] - prefix[a]).astype(np.float64)
        spans = edge[b] - edge[a]
        logs = np.zeros_like(sizes)
        nz = sizes > 0
        logs[nz] = np.log2(sizes[nz])
        return sizes * logs + t * sizes + spans

    if t == 1:
        bounds = [0, n]
    else:
        if n <= EXACT_SEARCH_MAX_BUCKETS:
            aa, bb = np.meshgrid(np.arange(n + 1), np.arange(n + 1), indexing="ij")
            mask = aa < bb
            cand = np.unique(batch_costs(aa[mask], bb[mask]))
        else:
            cand = batch_costs(np.arange(n), np.arange(1, n + 1))
        bounds = D.minmax_contiguous(n, t, prefix, edge, cand)
    return _splitter_set(bounds, r_hist, prefix, edge, t, dom, radix_bits)


def compute_size_balanced_splitters(r_hist: np.ndarray, cdf: Cdf, t: int, dom: KeyDomain,
                                    radix_bits: int) -> SplitterSet:
    """Contrast partitioner balancing |R_i| only (skew.py:318-339): the
    balanced contiguous split of the prefix sums (host control plane)."""
    r_hist = np.asarray(r_hist, np.int64)
    n = int(r_hist.shape[0])
    _check(n, t, radix_bits)
    prefix = _prefix(r_hist)
    edge = _edge_cdf(cdf, dom, radix_bits)

    def max_extend(a, bound):
        lo, hi = a + 1, n
        while lo < hi:
            mid = (lo + hi + 1) // 2
            if prefix[mid] - prefix[a] <= bound:
                lo = mid
            else:
                hi = mid - 1
        return lo

    def feasible(bound):
        a, parts = 0, 0
        while a < n:
            if prefix[a + 1] - prefix[a] > bound:
                return False
            a = max_extend(a, bound)
            parts += 1
            if parts > t:
                return False
        return True

    if t == 1:
        bounds = [0, n]
    else:
        cand = np.unique((prefix[None, :] - prefix[:, None])[np.triu_indices(n + 1, 1)]) if n <= 256 else None
        if cand is not None:
            lo, hi = 0, cand.shape[0] - 1
            while lo < hi:
                mid = (lo + hi) // 2
                if feasible(int(cand[mid])):
                    hi = mid
                else:
                    lo = mid + 1
            best = int(cand[lo])
        else:
            lo, hi = int(np.max(r_hist)), int(prefix[-1])
            while lo < hi:
                mid = (lo + hi) // 2
                if feasible(mid):
                    hi = mid
                else:
                    lo = mid + 1
            best = lo
        jump = [max_extend(a, best) for a in range(n)]
        g = [0] * (n + 1)
        for a in range(n - 1, -1, -1):
            g[a] = 1 + g[jump[a]]
        bounds, a = [0], 0
        for p in range(1, t):
            remaining = t - p
            e = a + 1
            while e <= n - remaining and not (prefix[e] - prefix[a] <= best and g[e] <= remaining):
                e += 1
            bounds.append(e)
            a = e
        bounds.append(n)
    return _splitter_set(bounds, r_hist, prefix, edge, t, dom, radix_bits)


def _splitter_set(bounds, r_hist, prefix, edge, t, dom, radix_bits) -> SplitterSet:
    """skew.py:342-369 (spans clamped at 0, see csrc/splitters.cpp)."""
    n = int(r_hist.shape[0])
    bb = np.asarray(bounds, np.int64)
    sizes = prefix[bb[1:]] - prefix[bb[:-1]]
    costs = np.array([split_relevant_cost(int(sizes[j]), t, max(0.0, float(edge[bb[j + 1]] - edge[bb[j]])))
                      for j in range(t)])
    keys = np.array([bucket_lower_key(int(e), dom, radix_bits) for e in bb[1:-1]], np.uint64)
    return SplitterSet(keys, bb, SplitterVector.from_bucket_bounds(bounds, n), sizes.astype(np.int64), costs)
