"""CPU oracle for the MPSM join hot path -- TEST INFRASTRUCTURE ONLY.

This module is the checker the CUDA product path is compared against.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it; the product package
``paper_1207_0145_b200`` never does (tests/test_boundary.py checks that).

It restates, in plain C (``mpsm_oracle.c``, loaded through ctypes) and numpy,
the reference package at /root/reference/pkg/src/mpsm:

* kernels          -> _kernels.py:30-408   (C, mpsm_oracle.c)
* skew control     -> skew.py:52-369       (numpy/python, below)
* P-MPSM / B-MPSM  -> engine.py:181-433    (python driver below, T logical
                      workers run sequentially or on a thread pool; ctypes
                      releases the GIL so the C kernels run in parallel)

plus the checksum of SURVEY.md 8(a) a13 (sum mod 2^64 of
splitmix64(r_pay ^ rotl64(s_pay, 17)) over matched pairs).

Parity pin: tests/test_oracle_golden.py checks this restatement against the
fixtures in tests/golden/ that tests/golden/make_golden.py produced by running
the reference itself (count, max, materialized pairs -> checksum, worker
statistics, splitters, interpolation probes, sort/partition known answers).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

U64P = ctypes.POINTER(ctypes.c_uint64)
I64P = ctypes.POINTER(ctypes.c_int64)


def build(force: bool = False) -> str:
    """Compile mpsm_oracle.c into oracle/liboracle.so (gcc, -O2)."""
    src = os.path.join(_HERE, "mpsm_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(
            ["gcc", "-O2", "-fPIC", "-shared", "-o", _LIB_PATH, src],
            cwd=_HERE,
        )
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_three_phase_sort.restype = ctypes.c_int64
        L.orc_three_phase_sort.argtypes = [U64P, U64P, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int64]
        L.orc_radix_histogram.restype = ctypes.c_int64
        L.orc_radix_histogram.argtypes = [U64P, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64, I64P, ctypes.c_int64]
        L.orc_scatter_chunk.restype = ctypes.c_int64
        L.orc_scatter_chunk.argtypes = [U64P, U64P, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64, I64P,
                                        ctypes.c_int64, I64P, I64P, U64P, U64P]
        L.orc_interp_lower_bound.restype = ctypes.c_int64
        L.orc_interp_lower_bound.argtypes = [U64P, ctypes.c_int64, ctypes.c_uint64, I64P]
        L.orc_merge_join_run.restype = None
        L.orc_merge_join_run.argtypes = [U64P, U64P, ctypes.c_int64, U64P, U64P, ctypes.c_int64, ctypes.c_int64,
                                         ctypes.c_int, U64P, U64P, ctypes.c_int64, ctypes.c_int, U64P]
        L.orc_fk_gather.restype = ctypes.c_int64
        L.orc_fk_gather.argtypes = [U64P, U64P, ctypes.c_int64, U64P, U64P, ctypes.c_int64, ctypes.c_uint64, U64P]
        L.orc_pairs_checksum.restype = ctypes.c_uint64
        L.orc_pairs_checksum.argtypes = [U64P, U64P, ctypes.c_int64]
        L.orc_pair_hash.restype = ctypes.c_uint64
        L.orc_pair_hash.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        _lib = L
    return _lib


def _u64(a: np.ndarray):
    assert a.dtype == np.uint64 and a.flags.c_contiguous
    return a.ctypes.data_as(U64P)


def _i64(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(I64P)


# ---------------------------------------------------------------- kernels ---

def pair_hash(r_pay: int, s_pay: int) -> int:
    return int(lib().orc_pair_hash(r_pay, s_pay))


def pair_hash_np(r_pays: np.ndarray, s_pays: np.ndarray) -> np.ndarray:
    """Vectorized splitmix64(r ^ rotl(s,17)) (numpy uint64 wraps mod 2^64)."""
    r = r_pays.astype(np.uint64)
    s = s_pays.astype(np.uint64)
    with np.errstate(over="ignore"):
        x = r ^ ((s << np.uint64(17)) | (s >> np.uint64(47)))
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def pairs_checksum(r_pays: np.ndarray, s_pays: np.ndarray) -> int:
    r = np.ascontiguousarray(r_pays, np.uint64)
    s = np.ascontiguousarray(s_pays, np.uint64)
    return int(lib().orc_pairs_checksum(_u64(r), _u64(s), r.shape[0]))


def three_phase_sort(keys: np.ndarray, pays: np.ndarray, lower: int, width_bits: int) -> int:
    """In-place run sort (_kernels.py:217); returns fallbacks or -1 (domain)."""
    return int(lib().orc_three_phase_sort(_u64(keys), _u64(pays), 0, keys.shape[0], lower, width_bits))


def radix_histogram(keys: np.ndarray, lower: int, shift: int, counts: np.ndarray) -> int:
    return int(lib().orc_radix_histogram(_u64(keys), keys.shape[0], lower, shift, _i64(counts), counts.shape[0]))


def scatter_chunk(keys, pays, lower, shift, sp, cursors, ends, out_keys, out_pays) -> int:
    return int(lib().orc_scatter_chunk(_u64(keys), _u64(pays), keys.shape[0], lower, shift, _i64(sp),
                                       sp.shape[0], _i64(cursors), _i64(ends), _u64(out_keys), _u64(out_pays)))


def interp_lower_bound(keys: np.ndarray, target: int):
    probes = ctypes.c_int64(0)
    idx = lib().orc_interp_lower_bound(_u64(keys), keys.shape[0], int(target), ctypes.byref(probes))
    return int(idx), int(probes.value)


def merge_join_run(r_keys, r_pays, s_keys, s_pays, s_start, collect=False, out_r=None, out_s=None, swap=False):
    """Returns (count, best, examined, emitted, checksum) (_kernels.py:340-408 + checksum)."""
    res = np.zeros(5, np.uint64)
    if out_r is None:
        out_r = np.empty(0, np.uint64)
        out_s = np.empty(0, np.uint64)
    lib().orc_merge_join_run(_u64(r_keys), _u64(r_pays), r_keys.shape[0], _u64(s_keys), _u64(s_pays),
                             s_keys.shape[0], int(s_start), int(bool(collect)), _u64(out_r), _u64(out_s),
                             out_r.shape[0], int(bool(swap)), _u64(res))
    return int(res[0]), int(res[1]), int(res[2]), int(res[3]), int(res[4])


def fk_gather(r_keys, r_pays, s_keys, s_pays, lower: int):
    """Independent FK checker: (count, max or None, checksum)."""
    res = np.zeros(5, np.uint64)
    rc = lib().orc_fk_gather(_u64(r_keys), _u64(r_pays), r_keys.shape[0], _u64(s_keys), _u64(s_pays),
                             s_keys.shape[0], lower, _u64(res))
    if rc != -1:
        raise ValueError("R keys are not a permutation of the domain prefix")
    count = int(res[0])
    return count, (int(res[1]) if count else None), int(res[4])


# ------------------------------------------------------------ skew (numpy) ---

def width_bits(lower: int, upper: int) -> int:
    return (upper - lower - 1).bit_length()  # core.py:82-84


def local_equiheight_bounds(run_keys: np.ndarray, f: int, t: int):
    """skew.py:52-62: keys at ranks ceil(n*m/k)-1, k=f*t; (keys, run_size)."""
    k = f * t
    n = run_keys.shape[0]
    if n == 0:
        return np.empty(0, np.uint64), 0
    ms = np.arange(1, k + 1, dtype=np.int64)
    pos = (n * ms + k - 1) // k - 1
    return run_keys[pos].copy(), n


@dataclass
class Cdf:
    step_keys: np.ndarray
    step_cum: np.ndarray
    total: int
    anchor_key: int = 0

    def eval_many(self, probes: np.ndarray) -> np.ndarray:
        """skew.py:79-109 (same float operations in the same order)."""
        keys = self.step_keys
        n = keys.shape[0]
        probes = np.asarray(probes, np.uint64)
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


def build_cdf(bounds, anchor_key: int = 0) -> Cdf:
    """skew.py:116-141; bounds = list of (keys, run_size)."""
    kp, wp, total = [], [], 0
    for keys, size in bounds:
        total += size
        if keys.shape[0]:
            kp.append(keys)
            wp.append(np.full(keys.shape[0], size / keys.shape[0]))
    if not kp:
        return Cdf(np.empty(0, np.uint64), np.empty(0, np.float64), total, anchor_key)
    keys = np.concatenate(kp)
    w = np.concatenate(wp)
    order = np.argsort(keys, kind="stable")
    keys = keys[order]
    cum = np.cumsum(w[order])
    keep = np.empty(keys.shape[0], bool)
    keep[:-1] = keys[:-1] != keys[1:]
    keep[-1] = True
    return Cdf(keys[keep], cum[keep], total, anchor_key)


def split_cost(n_private: int, t: int, span: float) -> float:
    """skew.py:148-153"""
    if span < 0:
        raise ValueError("s_span must be non-negative")  # skew.py:150-151
    return (n_private * math.log2(n_private) if n_private > 0 else 0.0) + t * n_private + span


def _minmax_contiguous(n, t, seg_cost, batch_costs):
    """skew.py:180-273: min over max segment cost, lexicographically smallest bounds."""
    if t > n:
        raise ValueError(f"cannot split {n} buckets into {t} partitions")
    if t == 1:
        return [0, n]

    def max_extend(a, bound):
        lo, hi = a + 1, n
        while lo < hi:
            mid = (lo + hi + 1) // 2
            if seg_cost(a, mid) <= bound:
                lo = mid
            else:
                hi = mid - 1
        return lo

    def feasible(bound):
        if seg_cost(0, 1) > bound:
            return False
        a, parts = 0, 0
        while a < n:
            if seg_cost(a, a + 1) > bound:
                return False
            a = max_extend(a, bound)
            parts += 1
            if parts > t:
                return False
        return True

    if n <= 256:
        aa, bb = np.meshgrid(np.arange(n + 1), np.arange(n + 1), indexing="ij")
        mask = aa < bb
        cand = np.unique(batch_costs(aa[mask], bb[mask]))
        lo, hi = 0, cand.shape[0] - 1
        while lo < hi:
            mid = (lo + hi) // 2
            if feasible(float(cand[mid])):
                hi = mid
            else:
                lo = mid + 1
        best = float(cand[lo])
    else:
        singles = batch_costs(np.arange(n), np.arange(1, n + 1))
        lo_c, hi_c = float(singles.max()), float(seg_cost(0, n))
        for _ in range(80):
            mid = 0.5 * (lo_c + hi_c)
            if feasible(mid):
                hi_c = mid
            else:
                lo_c = mid
            if hi_c - lo_c <= 1e-9 * max(1.0, abs(hi_c)):
                break
        best = hi_c
    jump = [max_extend(a, best) for a in range(n)]
    g = [0] * (n + 1)
    for a in range(n - 1, -1, -1):
        g[a] = 1 + g[jump[a]]
    bounds, a = [0], 0
    for p in range(1, t):
        remaining = t - p
        e = a + 1
        limit = n - remaining
        while e <= limit:
            if seg_cost(a, e) <= best and g[e] <= remaining:
                break
            e += 1
        if e > limit:
            raise RuntimeError("no feasible boundary at the optimal bound")
        bounds.append(e)
        a = e
    bounds.append(n)
    return bounds


def edge_cdf(cdf: Cdf, lower: int, wbits: int, radix_bits: int) -> np.ndarray:
    """skew.py:276-284"""
    n = 1 << radix_bits
    sh = wbits - radix_bits
    top = (1 << 64) - 1
    edges = np.array([min(lower + (e << sh), top) for e in range(n + 1)], np.uint64)
    return cdf.eval_many(edges)


def compute_splitters(r_hist: np.ndarray, cdf: Cdf, t: int, lower: int, wbits: int, radix_bits: int):
    """skew.py:287-315; returns bucket_bounds (list of t+1 ints)."""
    n = int(r_hist.shape[0])
    prefix = np.zeros(n + 1, np.int64)
    np.cumsum(r_hist, out=prefix[1:])
    ec = edge_cdf(cdf, lower, wbits, radix_bits)

    def seg_cost(a, b):
        return split_cost(int(prefix[b] - prefix[a]), t, float(ec[b] - ec[a]))

    def batch_costs(a, b):
        sizes = (prefix[b] - prefix[a]).astype(np.float64)
        spans = ec[b] - ec[a]
        logs = np.zeros_like(sizes)
        nz = sizes > 0
        logs[nz] = np.log2(sizes[nz])
        return sizes * logs + t * sizes + spans

    return _minmax_contiguous(n, t, seg_cost, batch_costs)


# --------------------------------------------------------- engine (python) ---

@dataclass
class OracleStats:
    worker: int
    tuples_sorted_public: int = 0
    tuples_sorted_private: int = 0
    tuples_scattered: int = 0
    public_tuples_examined: int = 0
    probe_tuples_examined: int = 0
    s_runs_with_matches: int = 0


@dataclass
class OracleResult:
    match_count: int
    aggregate_max: Optional[int]
    checksum: int
    materialized: Optional[np.ndarray] = None
    worker_stats: list = field(default_factory=list)
    bucket_bounds: Optional[list] = None


def _chunks(n: int, t: int):
    base, rem = divmod(n, t)
    out, start = [], 0
    for i in range(t):
        size = base + (1 if i < rem else 0)
        out.append((start, start + size))
        start += size
    return out


def join(r_keys, r_pays, s_keys, s_pays, *, threads=1, lower=0, upper=1 << 32, radix_bits=10,
         cdf_fanout=4, algorithm="p-mpsm", role_policy="auto", query_mode="aggregate-max",
         materialize_cap=1 << 20, parallel=False) -> OracleResult:
    """Restatement of engine.run_pmpsm / run_bmpsm (engine.py:279-433, 195-276).

    Workers run their phases in barrier order; with parallel=True each phase's
    T worker calls go to a thread pool (the C kernels release the GIL).
    Raises ValueError for domain violations (the reference raises DomainError).
    """
    t = threads
    wbits = width_bits(lower, upper)
    for keys in (r_keys, s_keys):
        if keys.shape[0] and (int(keys.min()) < lower or (upper < 1 << 64 and int(keys.max()) >= upper)):
            raise ValueError("key outside domain")
    if role_policy == "r-private":
        swapped = False
    elif role_policy == "s-private":
        swapped = True
    else:
        swapped = not (r_keys.shape[0] <= s_keys.shape[0])
    pk, pp, uk, up = (s_keys, s_pays, r_keys, r_pays) if swapped else (r_keys, r_pays, s_keys, s_pays)
    pub_ch = _chunks(uk.shape[0], t)
    priv_ch = _chunks(pk.shape[0], t)
    stats = [OracleStats(i) for i in range(t)]
    pool = ThreadPoolExecutor(t) if parallel and t > 1 else None

    def each(fn):
        if pool is None:
            return [fn(i) for i in range(t)]
        return list(pool.map(fn, range(t)))

    def sort_copy(keys, pays, a, b):
        k = np.ascontiguousarray(keys[a:b]).copy()
        p = np.ascontiguousarray(pays[a:b]).copy()
        if three_phase_sort(k, p, lower, wbits) < 0:
            raise ValueError("key outside domain")
        return k, p

    try:
        pub_runs = each(lambda i: sort_copy(uk, up, *pub_ch[i]))
        for i in range(t):
            stats[i].tuples_sorted_public = pub_ch[i][1] - pub_ch[i][0]
        bucket_bounds = None
        if algorithm == "b-mpsm":
            priv_runs = each(lambda i: sort_copy(pk, pp, *priv_ch[i]))
        else:
            bits = min(radix_bits, wbits)
            bounds = [local_equiheight_bounds(pub_runs[i][0], cdf_fanout, t) for i in range(t)]
            cdf = build_cdf(bounds, anchor_key=lower)
            shift = wbits - bits
            hists = []
            for i in range(t):
                c = np.zeros(1 << bits, np.int64)
                a, b = priv_ch[i]
                if b > a and radix_histogram(np.ascontiguousarray(pk[a:b]), lower, shift, c) >= 0:
                    raise ValueError("key outside domain")
                hists.append(c)
            ghist = np.sum(hists, axis=0)
            bucket_bounds = compute_splitters(ghist, cdf, t, lower, wbits, bits)
            sp = np.empty(1 << bits, np.int64)
            for j in range(t):
                sp[bucket_bounds[j]:bucket_bounds[j + 1]] = j
            counts = np.zeros((t, t), np.int64)
            for i in range(t):
                np.add.at(counts[i], sp, hists[i])
            starts = np.zeros_like(counts)
            if t > 1:
                starts[1:] = np.cumsum(counts[:-1], axis=0)
            run_base = np.zeros(t + 1, np.int64)
            np.cumsum(counts.sum(axis=0), out=run_base[1:])
            ak = np.empty(int(run_base[-1]), np.uint64)
            ap = np.empty(int(run_base[-1]), np.uint64)

            def scat(i):
                a, b = priv_ch[i]
                cur = (run_base[:-1] + starts[i]).astype(np.int64)
                ends = cur + counts[i]
                if b > a:
                    bad = scatter_chunk(np.ascontiguousarray(pk[a:b]), np.ascontiguousarray(pp[a:b]), lower, shift,
                                        sp, cur, ends, ak, ap)
                    if bad >= 0:
                        raise RuntimeError("scatter overflow")
                if not np.array_equal(cur, ends):
                    raise RuntimeError("scatter underflow")

            each(scat)
            priv_runs = each(lambda i: sort_copy(ak, ap, int(run_base[i]), int(run_base[i + 1])))
            for i in range(t):
                stats[i].tuples_scattered = priv_ch[i][1] - priv_ch[i][0]

        collect = query_mode == "materialize"

        def join_worker(i):
            rk, rp = priv_runs[i]
            st = stats[i]
            st.tuples_sorted_private = rk.shape[0]
            cnt, best, csum = 0, 0, 0
            outs = []
            if rk.shape[0] == 0:
                return cnt, best, csum, outs
            for k in range(t):
                sk, spp = pub_runs[(i + k) % t]
                if sk.shape[0] == 0:
                    continue
                start, probes = interp_lower_bound(sk, int(rk[0]))
                st.probe_tuples_examined += probes
                st.public_tuples_examined += probes
                if collect:
                    o_r = np.empty(materialize_cap, np.uint64)
                    o_s = np.empty(materialize_cap, np.uint64)
                else:
                    o_r = o_s = None
                c, b, ex, em, cs = merge_join_run(rk, rp, sk, spp, start, collect, o_r, o_s, swapped)
                st.public_tuples_examined += ex
                if c > 0:
                    st.s_runs_with_matches += 1
                    if cnt == 0 or b > best:
                        best = b
                    cnt += c
                    csum = (csum + cs) & ((1 << 64) - 1)
                    if collect:
                        if em < c:
                            raise OverflowError("materialize cap exceeded")
                        outs.append(np.stack([o_r[:em], o_s[:em]], axis=1))
            return cnt, best, csum, outs

        partials = each(join_worker)
    finally:
        if pool is not None:
            pool.shutdown()
    count = sum(p[0] for p in partials)
    agg = None
    if query_mode == "aggregate-max" and count > 0:
        agg = max(p[1] for p in partials if p[0] > 0)
    csum = sum(p[2] for p in partials) & ((1 << 64) - 1)
    mat = None
    if collect:
        if count > materialize_cap:
            raise OverflowError("materialize cap exceeded")
        pieces = [x for p in partials for x in p[3] if x.shape[0]]
        mat = np.concatenate(pieces, axis=0) if pieces else np.empty((0, 2), np.uint64)
    return OracleResult(count, agg, csum, mat, stats, bucket_bounds)


# ----------------------------------------------------------- generators ---

def gen_fk(n_r: int, n_s: int, seed: int = 0):
    """SURVEY.md 8(d) FK generator: R = PCG64(2*seed), S = PCG64(2*seed+1)."""
    rr = np.random.Generator(np.random.PCG64(2 * seed))
    r_keys = (rr.permutation(n_r) + 1).astype(np.uint64)
    r_pays = rr.integers(0, 1 << 32, n_r, dtype=np.uint64)
    rs = np.random.Generator(np.random.PCG64(2 * seed + 1))
    s_keys = rs.integers(1, n_r + 1, n_s, dtype=np.uint64)
    s_pays = rs.integers(0, 1 << 32, n_s, dtype=np.uint64)
    return r_keys, r_pays, s_keys, s_pays
