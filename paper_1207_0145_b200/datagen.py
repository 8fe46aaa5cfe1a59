"""Seeded input generators for the join benchmark configurations.

These are the synthetic stand-ins for the paper's datasets (PAPER.md
290-310; the paper's data is synthetic, so nothing is missing).  All draw
from numpy's PCG64, seeded explicitly, so identical arguments give
bit-identical relations:

* ``gen_fk``        -- BASELINE.json configs 1-3 and 5: R keys a
  seeded permutation of 1..|R|, S keys iid uniform in [1, |R|], payloads
  uniform in [0, 2^32).  R draws from PCG64(2*seed), S from PCG64(2*seed+1),
  the reference harness's seed convention (bench.py:142-144).
* ``gen_skewed_8020`` -- restates the reference generator
  (datagen.py:65-84): 80 % of the keys uniform in the hot 20 % tail of the
  domain (high or low end), the rest uniform in the remainder.  Config 4 uses
  R = low, S = high.  tests/test_oracle_golden.py checks the oracle's copy reproduces the
  reference's arrays bit for bit (fingerprints in tests/golden/golden.json).
* ``gen_uniform`` / ``gen_location_skew`` -- datagen.py:58-62, 87-105.
"""

from __future__ import annotations

import numpy as np

from .core import ConfigurationError, KeyDomain, Relation

PAYLOAD_UPPER = 1 << 32


def _rng(seed) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def gen_fk(n_r: int, n_s: int, seed: int = 0) -> tuple:
    """Foreign-key join inputs: (R, S, KeyDomain(1, n_r + 1))."""
    rr = _rng(2 * seed)
    r_keys = rr.permutation(n_r).astype(np.uint64)
    r_keys += np.uint64(1)
    r_pays = rr.integers(0, PAYLOAD_UPPER, n_r, dtype=np.uint64)
    rs = _rng(2 * seed + 1)
    s_keys = rs.integers(1, n_r + 1, n_s, dtype=np.uint64)
    s_pays = rs.integers(0, PAYLOAD_UPPER, n_s, dtype=np.uint64)
    return Relation(r_keys, r_pays), Relation(s_keys, s_pays), KeyDomain(1, n_r + 1)


def gen_uniform(n: int, dom: KeyDomain, seed: int = 0) -> Relation:
    rng = _rng(seed)
    keys = rng.integers(dom.lower, dom.upper, n, dtype=np.uint64)
    return Relation(keys, rng.integers(0, PAYLOAD_UPPER, n, dtype=np.uint64))


def gen_skewed_8020(n: int, dom: KeyDomain, direction: str, seed: int = 0) -> Relation:
    """80 % of keys in the 20 % high (or low) tail, uniform within segments."""
    if direction not in ("high", "low"):
        raise ConfigurationError("direction must be 'high' or 'low'")
    rng = _rng(seed)
    cut = dom.lower + (dom.width * 4) // 5
    hot = rng.random(n) < 0.8
    n_hot = int(np.count_nonzero(hot))
    keys = np.empty(n, np.uint64)
    if direction == "high":
        keys[hot] = rng.integers(cut, dom.upper, n_hot, dtype=np.uint64)
        keys[~hot] = rng.integers(dom.lower, cut, n - n_hot, dtype=np.uint64)
    else:
        edge = dom.lower + dom.width - (dom.width * 4) // 5
        keys[hot] = rng.integers(dom.lower, edge, n_hot, dtype=np.uint64)
        keys[~hot] = rng.integers(edge, dom.upper, n - n_hot, dtype=np.uint64)
    return Relation(keys, rng.integers(0, PAYLOAD_UPPER, n, dtype=np.uint64))


def gen_location_skew(rel: Relation, t: int, seed: int = 0) -> Relation:
    """Chunk i of t holds the i-th key quantile, shuffled inside the chunk."""
    if t < 1:
        raise ConfigurationError("t must be >= 1")
    order = np.argsort(rel.keys, kind="stable")
    keys = rel.keys[order].copy()
    pays = rel.payloads[order].copy()
    rng = _rng([seed, 0x10C])
    n = rel.cardinality
    base, rem = divmod(n, t)
    start = 0
    for i in range(t):
        size = base + (1 if i < rem else 0)
        perm = rng.permutation(size)
        keys[start:start + size] = keys[start:start + size][perm]
        pays[start:start + size] = pays[start:start + size][perm]
        start += size
    return Relation(keys, pays)


def gen_negcorr(n_r: int, n_s: int, dom: KeyDomain, seed: int = 0) -> tuple:
    """Config 4: R skewed low, S skewed high (negatively correlated)."""
    return gen_skewed_8020(n_r, dom, "low", seed=2 * seed), gen_skewed_8020(n_s, dom, "high", seed=2 * seed + 1)


DISTRIBUTIONS = ("uniform", "skew-80-20-high", "skew-80-20-low", "location-sorted-clusters")


class GenSpec:
    """Everything needed to regenerate a relation (datagen.py:33-47)."""

    def __init__(self, cardinality: int, key_domain: KeyDomain, distribution: str = "uniform", seed: int = 0,
                 location_threads: int = 4):
        if cardinality < 0:
            raise ConfigurationError("cardinality must be non-negative")
        if distribution not in DISTRIBUTIONS:
            raise ConfigurationError(f"unknown distribution {distribution!r}")
        self.cardinality = cardinality
        self.key_domain = key_domain
        self.distribution = distribution
        self.seed = seed
        self.location_threads = location_threads


def generate(spec: GenSpec) -> Relation:
    """datagen.py:108-118"""
    if spec.distribution == "uniform":
        return gen_uniform(spec.cardinality, spec.key_domain, spec.seed)
    if spec.distribution == "skew-80-20-high":
        return gen_skewed_8020(spec.cardinality, spec.key_domain, "high", spec.seed)
    if spec.distribution == "skew-80-20-low":
        return gen_skewed_8020(spec.cardinality, spec.key_domain, "low", spec.seed)
    base = gen_uniform(spec.cardinality, spec.key_domain, spec.seed)
    return gen_location_skew(base, spec.location_threads, spec.seed)


def fk_range_device(n_r: int, n_s: int, r_range: tuple, s_range: tuple, seed: int, device) -> tuple:
    """Positions [r_range) of R and [s_range) of S of a counter-based FK
    workload generated on the GPU (any range of any size, independently):
    R keys are a bijective Feistel permutation of [0, n_r) (cycle walking)
    plus 1, S keys splitmix64(seed, pos) mod n_r plus 1, payloads splitmix64
    masked to 32 bits.  -> (R, S) Relations with CUDA uint64 columns."""
    import math

    import torch

    def mix(x):
        x = x + (0x9E3779B97F4A7C15 - (1 << 64))  # int64 arithmetic wraps
        x = (x ^ (x >> 30).bitwise_and((1 << 34) - 1)) * -4658895280553007687  # 0xBF58476D1CE4E5B9
        x = (x ^ (x >> 27).bitwise_and((1 << 37) - 1)) * -7723592293110705685  # 0x94D049BB133111EB
        return x ^ (x >> 31).bitwise_and((1 << 33) - 1)

    half = max(1, math.ceil(math.log2(max(n_r, 2)) / 2))
    mask = (1 << half) - 1

    def feistel(x):
        l, r_ = x >> half, x & mask
        for rnd in range(4):
            l, r_ = r_, l ^ (mix(r_ + (seed * 4 + rnd) * 0x1000193) & mask)
        return (l << half) | r_

    ra, rb = r_range
    sa, sb = s_range
    pos = torch.arange(ra, rb, dtype=torch.int64, device=device)
    k = feistel(pos)
    while True:
        bad = k >= n_r
        if not bool(bad.any()):
            break
        k = torch.where(bad, feistel(k), k)
    r_keys = (k + 1).view(torch.uint64)
    r_pays = (mix(pos + (2 * seed + 11) * (1 << 40)) & 0xFFFFFFFF).view(torch.uint64)
    del pos, k
    spos = torch.arange(sa, sb, dtype=torch.int64, device=device)
    hs = mix(spos + (2 * seed + 1) * (1 << 41))
    s_keys = ((hs & 0x7FFFFFFFFFFFFFFF) % n_r + 1).view(torch.uint64)
    del hs
    s_pays = (mix(spos + (2 * seed + 13) * (1 << 42)) & 0xFFFFFFFF).view(torch.uint64)
    return Relation(r_keys, r_pays), Relation(s_keys, s_pays)


def fk_shard_chunked(n_r: int, n_s: int, rank: int, world: int, seed: int, device, chunk: int = 1 << 27) -> tuple:
    """Position-shard `rank` of `world` of the counter-based FK workload
    (fk_range_device), generated chunk by chunk into preallocated columns so
    the generator's temporaries stay small (config 5: 6.4G S tuples)."""
    import torch

    from .core import chunk_bounds

    (ra, rb), (sa, sb) = chunk_bounds(n_r, world)[rank], chunk_bounds(n_s, world)[rank]
    cols = [torch.empty(n, dtype=torch.uint64, device=device) for n in (rb - ra, rb - ra, sb - sa, sb - sa)]
    for a in range(ra, rb, chunk):
        b = min(rb, a + chunk)
        r, _ = fk_range_device(n_r, n_s, (a, b), (0, 0), seed, device)
        cols[0][a - ra:b - ra].copy_(r.keys)
        cols[1][a - ra:b - ra].copy_(r.payloads)
    for a in range(sa, sb, chunk):
        b = min(sb, a + chunk)
        _, s = fk_range_device(n_r, n_s, (0, 0), (a, b), seed, device)
        cols[2][a - sa:b - sa].copy_(s.keys)
        cols[3][a - sa:b - sa].copy_(s.payloads)
    return Relation(cols[0], cols[1]), Relation(cols[2], cols[3])


def skewed_8020_range_device(n: int, dom: KeyDomain, direction: str, pos_range: tuple, seed: int, device,
                             chunk: int = 1 << 27) -> Relation:
    """Positions [pos_range) of an 80-20 skewed relation generated on the GPU
    (counter-based, any range independently): the distribution of
    gen_skewed_8020 / the reference's datagen.py:65-84 (80 % of the keys
    uniform in the hot 20 % tail of the domain, high or low end, the rest
    uniform in the remainder, payloads uniform 32-bit), not its numpy stream.
    The multi-GPU bench builds config 4 shards with it."""
    import torch

    if direction not in ("high", "low"):
        raise ConfigurationError("direction must be 'high' or 'low'")
    M = 0x7FFFFFFFFFFFFFFF

    def mix(x):
        x = x + (0x9E3779B97F4A7C15 - (1 << 64))
        x = (x ^ (x >> 30).bitwise_and((1 << 34) - 1)) * -4658895280553007687
        x = (x ^ (x >> 27).bitwise_and((1 << 37) - 1)) * -7723592293110705685
        return x ^ (x >> 31).bitwise_and((1 << 33) - 1)

    w = dom.width
    if direction == "high":
        cut = dom.lower + (w * 4) // 5
        hot_lo, hot_n, cold_lo, cold_n = cut, dom.upper - cut, dom.lower, cut - dom.lower
    else:
        edge = dom.lower + w - (w * 4) // 5
        hot_lo, hot_n, cold_lo, cold_n = dom.lower, edge - dom.lower, edge, dom.upper - edge
    a0, b0 = pos_range
    keys = torch.empty(b0 - a0, dtype=torch.uint64, device=device)
    pays = torch.empty(b0 - a0, dtype=torch.uint64, device=device)
    for a in range(a0, b0, chunk):
        b = min(b0, a + chunk)
        pos = torch.arange(a, b, dtype=torch.int64, device=device)
        u = mix(pos + (3 * seed + 1) * (1 << 40)) & M
        hot = (u % 1000) < 800
        v = mix(pos + (3 * seed + 2) * (1 << 41)) & M
        k = torch.where(hot, hot_lo + v % hot_n, cold_lo + v % max(cold_n, 1))
        keys[a - a0:b - a0].copy_(k.view(torch.uint64))
        pays[a - a0:b - a0].copy_((mix(pos + (3 * seed + 3) * (1 << 42)) & 0xFFFFFFFF).view(torch.uint64))
    return Relation(keys, pays)


def gen_fk_device(n_r: int, n_s: int, seed: int = 0, device=None, rank: int = 0, world: int = 1) -> tuple:
    """FK workload generated on the GPU (counter-based; a rank builds only its
    position shard): -> (R, S, KeyDomain) with CUDA uint64 columns.  Not the
    numpy stream of gen_fk -- same distribution (R keys a permutation of
    [1, n_r], S keys uniform over them, 32-bit payloads)."""
    import torch

    from .distributed import fk_shard_device

    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    r, s = fk_shard_device(n_r, n_s, rank, world, seed, dev)
    return r, s, KeyDomain(1, n_r + 1)
