"""GPU MPSM join engine -- the drop-in for the reference's run_join / run_pmpsm /
run_bmpsm (/root/reference/pkg/src/mpsm/engine.py:279-466).

Same signatures, phases, result semantics and statistics.  The T logical
workers of the reference (cfg.threads) are kept: T public runs (S chunked by
position, core.py:263-279) and, for P-MPSM, T private partitions chosen by
the reference's CDF/histogram splitters.  One host thread issues the work of
all workers to the GPU in barrier order (engine.py:380-419); there are no
worker threads and no barriers to deadlock on (SURVEY.md finding 7).

Per phase, device work only (csrc/):
  sort_public   LSD radix sort of every public chunk into its run
  sort_private  the private input sorted as ONE run (P-MPSM; B-MPSM: per
                chunk), first pass fused with the domain check; the host
                computes the splitters meanwhile
  histogram     2^B bucket counts of the private input (k_radix_hist, over
                the packed records for host inputs), queued with the public
                runs' bound keys ahead of the private sort
  splitters     host: CDF from f*T bounds per public run + C++ min-max search
  scatter       none on one GPU: the range partition sends contiguous key
                ranges to the partitions in worker order and the run sort is
                stable, so partition p's run is the slice [run_base[p],
                run_base[p+1]) of the sorted private run -- the same tuples in
                the same order as the reference's arena + per-partition sort
                (partition.py:233-276, engine.py:396-409).  The multi-GPU
                engine (distributed.py) does move tuples: there the partition
                is a real scatter into per-rank send buffers + all-to-all.
  join          merge-path merge-join of every (private, public) run pair with
                fused COUNT / MAX / checksum and the Run order check (no
                materialisation unless asked)
"""

from __future__ import annotations

import os
import threading
import time
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np
import torch

from . import _lib
from . import device as D
from .core import (
    ConfigurationError,
    DomainError,
    InternalConsistencyError,
    JoinConfig,
    JoinResult,
    KeyDomain,
    MaterializeCapExceeded,
    PackedRelation,
    Relation,
    Run,
    WorkerStats,
    chunk_bounds,
    validate_relation,
)
from .partition import combine_counts, effective_radix_bits
from .skew import LocalBounds, bound_positions, build_cdf, compute_splitters

PhaseHook = Optional[Callable[[int, str], None]]
MASK64 = (1 << 64) - 1


@dataclass(frozen=True)
class RoleAssignment:
    """Which input plays the private (partitioned) role (engine.py:55-66)."""

    private: str

    @property
    def public(self) -> str:
        return "s" if self.private == "r" else "r"

    @property
    def swapped(self) -> bool:
        return self.private == "s"


def choose_roles(n_r: int, n_s: int, policy: str = "auto") -> RoleAssignment:
    """Smaller relation private, ties keep R (engine.py:69-78)."""
    if policy == "r-private":
        return RoleAssignment("r")
    if policy == "s-private":
        return RoleAssignment("s")
    if policy != "auto":
        raise ConfigurationError(f"unknown role policy {policy!r}")
    return RoleAssignment("r" if n_r <= n_s else "s")


@dataclass(frozen=True)
class PhaseStep:
    name: str
    barrier_after: bool


@dataclass(frozen=True)
class PhasePlan:
    algorithm: str
    steps: tuple

    def __post_init__(self) -> None:
        names = [s.name for s in self.steps]
        if "join" in names and "sort_public" in names:
            i_pub = names.index("sort_public")
            if not self.steps[i_pub].barrier_after or names.index("join") < i_pub:
                raise ConfigurationError("join must start after the public-sort barrier")


def plan_phases(algorithm: str) -> PhasePlan:
    """engine.py:100-121"""
    if algorithm == "b-mpsm":
        return PhasePlan(algorithm, (PhaseStep("sort_public", True), PhaseStep("sort_private", False),
                                     PhaseStep("join", False)))
    if algorithm == "p-mpsm":
        return PhasePlan(algorithm, (PhaseStep("sort_public", True), PhaseStep("histogram", True),
                                     PhaseStep("scatter", True), PhaseStep("sort_private", False),
                                     PhaseStep("join", False)))
    raise ConfigurationError(f"no phase plan for algorithm {algorithm!r}")


# ------------------------------------------------------------ run helpers

def _keys_of(run):
    if isinstance(run, (Run, Relation)):
        return run.keys, run.payloads
    return run, None


def interpolation_search(run, target: int) -> int:
    """First index with key >= target (engine.py:124-128), on the GPU with the
    reference's probe rule."""
    keys, _ = _keys_of(run)
    dev = D.ensure_device()
    kd = D.to_device(keys if not isinstance(keys, (list, tuple)) else np.asarray(keys, np.uint64), dev)
    tg = torch.from_numpy(np.array([int(target) & MASK64], np.uint64)).to(dev)
    idx, _ = D.interp_lower_bound(kd, tg)
    return int(idx.item())


def merge_join(r_run: Run, s_run: Run, s_start: int, emit: Callable[[int, int], None]) -> int:
    """emit(r_payload, s_payload) once per matching pair; returns the pair
    count (engine.py:131-166).  The pairs are produced by the GPU merge kernel
    (materialize mode) from s_start on and then handed to emit on the host."""
    dev = D.ensure_device()
    rk, rp = D.to_device(r_run.keys, dev), D.to_device(r_run.payloads, dev)
    sk, sp = D.to_device(s_run.keys, dev), D.to_device(s_run.payloads, dev)
    sk, sp = sk[s_start:], sp[s_start:]
    if rk.numel() == 0 or sk.numel() == 0:
        return 0
    rec = D.join_pairs([(rk, rp)], [(sk, sp)], False, _lib.MODE_COUNT)
    count = int(rec[0, _lib.PAIR_COUNT].item())
    if count:
        out = torch.empty(2 * count, dtype=torch.uint64, device=dev)
        D.join_pairs([(rk, rp)], [(sk, sp)], False, _lib.MODE_MATERIALIZE, out, count)
        pairs = out.view(count, 2).cpu().numpy()
        for a, b in pairs.tolist():
            emit(a, b)
    return count


# ----------------------------------------------------------------- engine

_EV_POOL = threading.local()  # per thread and device: timing events reused join after join


class _Timeline:
    """CUDA events at phase boundaries (engine.py:421-432 keys).  The events
    come from a per-thread pool (creating one costs as much host time as a
    kernel launch, and a join's first launch waits behind it); a join reads
    its timings before it returns, so the next join of the thread may reuse
    them."""

    def __init__(self):
        self.ev = {}
        pools = getattr(_EV_POOL, "pools", None)
        if pools is None:
            pools = _EV_POOL.pools = {}
        dev = torch.cuda.current_device()
        self.pool = pools.setdefault(dev, [])
        self.used = 0

    def mark(self, name: str) -> None:
        if self.used < len(self.pool):
            e = self.pool[self.used]
        else:
            e = torch.cuda.Event(enable_timing=True)
            self.pool.append(e)
        self.used += 1
        e.record()
        self.ev[name] = e

    def seconds(self, a: str, b: str) -> float:
        return self.ev[a].elapsed_time(self.ev[b]) / 1e3


def _prepare(r: Relation, s: Relation, cfg: JoinConfig):
    roles = choose_roles(r.cardinality, s.cardinality, cfg.role_policy)
    private, public = (r, s) if roles.private == "r" else (s, r)
    return cfg.key_domain, roles, private, public


def _domain_report(rel: Relation, dom: KeyDomain) -> tuple:
    """(violations, first index) of one relation: on the GPU for device
    columns, numpy for host columns (the error path only)"""
    if rel.cardinality == 0 or isinstance(rel, PackedRelation):  # records were validated when packed
        return 0, -1
    keys = rel.keys
    if isinstance(keys, torch.Tensor) and keys.is_cuda:
        return D.domain_report(keys, dom.lower, dom.upper - dom.lower - 1)
    rep = validate_relation(rel, dom)
    return rep.violation_count, (rep.sample_indices[0] if rep.sample_indices else -1)


def raise_domain_error(r: Relation, s: Relation, dom: KeyDomain) -> None:
    """The reference's DomainError, r checked before s (engine.py:181-190).
    Called once a fused domain check (first sort pass / histogram / upload)
    has flagged an out-of-domain key."""
    for name, rel in (("r", r), ("s", s)):
        cnt, first = _domain_report(rel, dom)
        if cnt:
            raise DomainError(f"relation {name} has {cnt} out-of-domain keys (first at index {first})")
    raise InternalConsistencyError("a domain check flagged a key that a recount does not find")


# packed 8-B records (key - lower) << (64 - w) | payload are used whenever the
# key width allows it and every payload fits; a join that meets a wide payload
# is re-run on (key, payload) pairs.  MPSM_PACK=0 forces the pair layout.
PACK_RECORDS = os.environ.get("MPSM_PACK", "1") != "0"
# host-resident inputs of a packed join cross PCIe as packed records (host
# threads pack while earlier chunks copy: half the bytes, device.upload_records)
# MPSM_HOST_PACK=0 copies the columns instead.
HOST_PACK = os.environ.get("MPSM_HOST_PACK", "1") != "0"

# device copies of the public runs' equi-height bound positions, per (device,
# chunk layout, fanout, workers): a host -> device copy from pageable memory
# would wait for the public sort queued before it
_BOUND_POS: dict = {}


def _bound_positions_device(chunks, f: int, t: int, dev) -> Optional[torch.Tensor]:
    key = (str(dev), tuple(chunks), f, t)
    pos = _BOUND_POS.get(key)
    if pos is None:
        parts = [bound_positions(b - a, f, t) + a for a, b in chunks if b > a]
        if not parts:
            return None
        host = torch.from_numpy(np.concatenate(parts).astype(np.int64)).pin_memory()
        pos = host.to(dev, non_blocking=True)
        if len(_BOUND_POS) > 64:
            _BOUND_POS.clear()
        _BOUND_POS[key] = pos
    return pos


_PASSES: dict = {}


def _pass_count(width_bits: int) -> int:
    v = _PASSES.get(width_bits)
    if v is None:
        v = _PASSES[width_bits] = int(_lib.load().mpsm_sort_pass_count(width_bits))
    return v


_STATUS_BUF: dict = {}


def _pinned_status(n: int) -> torch.Tensor:
    """pinned int64[n] for fetch_status, reused across joins (read back and
    copied out before the next join of the thread can write it)"""

    key = threading.get_ident()
    h = _STATUS_BUF.get(key)
    if h is None or h.numel() < n:
        h = torch.empty(max(n, 64), dtype=torch.int64, pin_memory=True)
        if len(_STATUS_BUF) > 64:
            _STATUS_BUF.clear()
        _STATUS_BUF[key] = h
    return h[:n]


class _PackOverflow(Exception):
    """a payload does not fit the packed record: rerun on (key, payload) pairs"""


class JoinContext:
    """Device buffers and state of one join on one GPU.

    Runs are (keys, payloads) tensor pairs, or (records, None) in packed mode.

    The private side of P-MPSM is sorted as ONE run and cut at the partition
    boundaries: the range partition (partition.py:233-276) sends contiguous
    key ranges to the partitions in worker order and the stable run sort keeps
    input order among equal keys, so sorting the whole private input and
    cutting it at run_base yields exactly the runs the arena + per-partition
    sorts produce (same tuples in the same order), without the scatter pass.
    The bucket histogram that feeds the splitters is computed before the
    private sort is queued and read back behind an event, so the host's
    splitter search overlaps the sort.
    """

    def __init__(self, r: Relation, s: Relation, cfg: JoinConfig, phase_hook: PhaseHook, packed: bool,
                 variant: str = "p-mpsm"):
        self.cfg = cfg
        self.hook = phase_hook
        self.dev = D.ensure_device()
        self.r, self.s = r, s
        self.dom, self.roles, private, public = _prepare(r, s, cfg)
        self.t = cfg.threads
        self.variant = variant
        self.wbits = self.dom.width_bits
        self.packed = bool(packed) and 1 <= self.wbits <= 63
        for rel in (r, s):
            if isinstance(rel, PackedRelation):
                if rel.key_domain != self.dom:
                    raise ConfigurationError("a PackedRelation's key domain must be the join's key domain")
                if not self.packed:
                    raise ConfigurationError("PackedRelation inputs need the packed record layout (MPSM_PACK=1)")
        # record inputs sorted in place (even pass count: the last pass lands
        # back in the input buffer)
        self._inplace = _pass_count(self.wbits) % 2 == 0
        self.pw = 64 - self.wbits
        self.span_m1 = self.dom.upper - self.dom.lower - 1
        # the private side is sorted whole (P-MPSM) or per chunk (B-MPSM);
        # host inputs of it are staged after the public sort is queued, so
        # that upload overlaps the public sort
        self._private = private
        self.priv_rec = None
        self.n_priv = private.cardinality
        # the private upload buffer is allocated now, before the public sort is
        # queued: its copies then need not wait for that sort
        self._priv_buf = self._priv_ready = None
        if self.packed and HOST_PACK and not isinstance(private, PackedRelation) \
                and D.host_columns(private.keys) is not None:
            self._priv_buf = torch.empty(self.n_priv, dtype=torch.uint64, device=self.dev)
            self._priv_ready = torch.cuda.Event()
            self._priv_ready.record()
        self.pub_rec = self._upload(public, True)
        if self.pub_rec is None:
            self.pub_k = D.to_device(public.keys, self.dev)
            self.pub_p = D.to_device(public.payloads, self.dev)
            self.n_pub = int(self.pub_k.numel())
        else:
            self.n_pub = int(self.pub_rec.numel())
        self.pub_chunks = chunk_bounds(self.n_pub, self.t)
        self.priv_chunks = chunk_bounds(self.n_priv, self.t)
        self.stats = [WorkerStats(i) for i in range(self.t)]
        # the two sides' domain flags and the payload-overflow flag in one
        # int64[3] (one copy; fetch_status reads them back with one copy)
        self.flags = D.new_join_flags(self.dev)
        self.bad_pub, self.bad_priv = self.flags[0:1], self.flags[1:2]
        self.overflow = self.flags[2:3].view(torch.int32)[0:1]
        self.tmp = []
        self.tl = _Timeline()

    def stage_private(self) -> None:
        """private input -> device (packed records or columns)"""
        private = self._private
        # the GPU is sorting the public run: host threads pack every chunk
        self.priv_rec = self._upload(private, True, gpu_pack_every=0, buf=self._priv_buf, ready=self._priv_ready)
        if self.priv_rec is None:
            self.priv_k = D.to_device(private.keys, self.dev)
            self.priv_p = D.to_device(private.payloads, self.dev)
        self._private = None

    def _upload(self, rel: Relation, allowed: bool, gpu_pack_every: int = -1, buf=None, ready=None):
        """host columns -> packed records on the device, or None (columns path)"""
        if isinstance(rel, PackedRelation):
            return rel.records
        if not (allowed and self.packed and HOST_PACK):
            return None
        hk, hp = D.host_columns(rel.keys), D.host_columns(rel.payloads)
        if hk is None or hp is None or hk[0].shape[0] != hp[0].shape[0]:
            return None
        rec = buf if buf is not None else torch.empty(int(hk[0].shape[0]), dtype=torch.uint64, device=self.dev)
        bad, ovf = D.upload_records(hk[0], hp[0], self.dom.lower, self.span_m1, self.wbits, rec,
                                    gpu_pack_every=gpu_pack_every, ready=ready)
        if bad >= 0:
            raise_domain_error(self.r, self.s, self.dom)
        if ovf:
            raise _PackOverflow()
        return rec

    def check_domain(self) -> None:
        """raise the reference's DomainError if a fused check flagged a key
        (synchronises on the two flags unless fetch_status read them)"""
        st = getattr(self, "_status", None)
        flags = (st[1], st[2]) if st is not None else (int(self.bad_priv.item()), int(self.bad_pub.item()))
        if flags != (-1, -1):
            raise_domain_error(self.r, self.s, self.dom)

    def fetch_status(self) -> None:
        """after the join is queued: the pair records and the three device
        flags (domain, payload width) into pinned host memory, one stream
        synchronisation for all of them"""
        n = int(self.rec.numel())
        h = _pinned_status(n + 3)
        # one kernel writes both into the pinned buffer (mpsm_fetch_small):
        # bad_pub, bad_priv, overflow (low half) after the pair records
        _lib.check(_lib.load().mpsm_fetch_small(h.data_ptr(), self.rec.data_ptr(), n, self.flags.data_ptr(), 3,
                                                D.stream_ptr()), "mpsm_fetch_small")
        torch.cuda.current_stream().synchronize()
        v = h.numpy()
        self._rec_host = v[:n].view(np.uint64).copy()
        self._status = (int(v[n + 2]) & 0xFFFFFFFF, int(v[n + 1]), int(v[n]))  # overflow, bad_priv, bad_pub

    def _hook(self, i: int, phase: str) -> None:
        if self.hook:
            self.hook(i, phase)

    def _empty(self, n: int) -> torch.Tensor:
        return torch.empty(n, dtype=torch.uint64, device=self.dev)

    def _tmp(self, width: int) -> list:
        """ping-pong buffers of the run sorts, shared by all phases"""
        if not self.tmp or self.tmp[0].numel() < width:
            self.tmp = [self._empty(width) for _ in range(1 if self.packed else 2)]
        return self.tmp

    def _alloc_runs(self, n: int) -> tuple:
        return (self._empty(n), None) if self.packed else (self._empty(n), self._empty(n))

    def _sort_into(self, in_k, in_p, dst: tuple, a: int, b: int, bad, dense=None) -> tuple:
        """sort in_k/in_p (length b-a; in_p None: in_k holds packed records)
        into dst[.][a:b]; returns the run.  dense: the sort's density probe
        of its output (packed layouts)"""
        n = b - a
        tmp = self._tmp(n)
        if in_p is None:
            out = dst[0][a:b]
            D.sort_records(in_k, self.wbits, out, tmp[0][:n], dense)
            return (out, None)
        if self.packed:
            out = dst[0][a:b]
            D.sort_packed(in_k, in_p, self.dom.lower, self.span_m1, self.wbits, out, tmp[0][:n], bad,
                          self.overflow, dense)
            return (out, None)
        ok, op = dst[0][a:b], dst[1][a:b]
        if n:
            D.sort_pairs(in_k, in_p, self.dom.lower, self.span_m1, self.wbits, ok, op, tmp[0][:n], tmp[1][:n], bad)
        return (ok, op)

    def _store_for(self, rel, rec, n: int) -> tuple:
        """where the runs of a side go: in place for consumed record inputs"""
        if isinstance(rel, PackedRelation) and self._inplace:
            return (rec, None)
        return self._alloc_runs(n)

    def _sort_segments(self, chunks, rec, k, p, dst: tuple, bad) -> list:
        """every chunk [a, b) sorted into dst[.][a:b] by ONE segmented sort
        (mpsm_sort_*_segments: one count / scan / scatter launch per pass for
        all chunks); returns the runs"""
        n = chunks[-1][1] if chunks else 0
        off = [a for a, _ in chunks] + [n]
        tmp = self._tmp(n)
        if n:
            if rec is not None:
                D.sort_records_segments(rec, off, self.wbits, dst[0], tmp[0][:n])
            elif self.packed:
                D.sort_packed_segments(k, p, off, self.dom.lower, self.span_m1, self.wbits, dst[0], tmp[0][:n], bad,
                                       self.overflow)
            else:
                D.sort_pairs_segments(k, p, off, self.dom.lower, self.span_m1, self.wbits, dst[0], dst[1],
                                      tmp[0][:n], tmp[1][:n], bad)
        return [(dst[0][a:b], None if dst[1] is None else dst[1][a:b]) for a, b in chunks]

    def sort_public(self):
        """phase 1: every public chunk -> sorted run (engine.py:389-395); T > 1
        chunks in one segmented sort."""
        public = self.s if self.roles.private == "r" else self.r
        self.pub_store = self._store_for(public, self.pub_rec, self.n_pub)
        if self.t > 1:
            self._tmp(self.n_pub)
            for i, (a, b) in enumerate(self.pub_chunks):
                self._hook(i, "sort_public")
                self.stats[i].tuples_sorted_public = b - a
            k, p = (None, None) if self.pub_rec is not None else (self.pub_k, self.pub_p)
            self.pub_runs = self._sort_segments(self.pub_chunks, self.pub_rec, k, p, self.pub_store, self.bad_pub)
            return
        self._tmp(max((b - a for a, b in self.pub_chunks), default=0))
        self.pub_runs = []
        for i, (a, b) in enumerate(self.pub_chunks):
            self._hook(i, "sort_public")
            if self.pub_rec is not None:
                run = self._sort_into(self.pub_rec[a:b], None, self.pub_store, a, b, self.bad_pub)
            else:
                run = self._sort_into(self.pub_k[a:b], self.pub_p[a:b], self.pub_store, a, b, self.bad_pub)
            self.pub_runs.append(run)
            self.stats[i].tuples_sorted_public = b - a

    def _sort_private_range(self, a: int, b: int, dense=None) -> tuple:
        if self.priv_rec is not None:
            return self._sort_into(self.priv_rec[a:b], None, self.priv_store, a, b, self.bad_priv, dense)
        return self._sort_into(self.priv_k[a:b], self.priv_p[a:b], self.priv_store, a, b, self.bad_priv, dense)

    def _private_rel(self):
        return self.r if self.roles.private == "r" else self.s

    def sort_private_chunks(self):
        """B-MPSM phase 2: each private chunk sorted into its run (engine.py:297-309),
        all chunks in one segmented sort."""
        self.priv_store = self._store_for(self._private_rel(), self.priv_rec, self.n_priv)
        for i, (a, b) in enumerate(self.priv_chunks):
            self._hook(i, "sort_private")
            self.stats[i].tuples_sorted_private = b - a
        if self.t == 1:
            self.priv_runs = [self._sort_private_range(0, self.n_priv)]
            return
        k, p = (None, None) if self.priv_rec is not None else (self.priv_k, self.priv_p)
        self.priv_runs = self._sort_segments(self.priv_chunks, self.priv_rec, k, p, self.priv_store, self.bad_priv)

    def sort_private_whole(self):
        """P-MPSM: the whole private input -> one sorted run (cut by partition()).
        Packed: the sort also reports whether its output is dense (consecutive
        keys, the FK case), which the join then need not read R to decide."""
        self.priv_store = self._store_for(self._private_rel(), self.priv_rec, self.n_priv)
        self.priv_dense = torch.empty(2, dtype=torch.uint32, device=self.dev) if self.packed else None
        self.priv_whole = self._sort_private_range(0, self.n_priv, self.priv_dense)

    def queue_histogram(self):
        """P-MPSM, T > 1, before the private sort is queued: the 2^B bucket
        histogram of the private input (partition.py:110-122; over the packed
        records when the private side was uploaded as records) and the
        equi-height bound keys of the public runs (skew.py:52-62), both copied
        to pinned host memory behind one event -- the host computes the
        splitters while the GPU sorts the private run."""
        t, dom = self.t, self.dom
        for i in range(t):
            self._hook(i, "histogram")
        bits = effective_radix_bits(dom, self.cfg.radix_bits)
        if (1 << bits) < t:
            raise ConfigurationError(f"effective radix bits {bits} give fewer buckets than {t} workers")
        nb = 1 << bits
        f = self.cfg.cdf_fanout
        hist = torch.zeros(nb, dtype=torch.int64, device=self.dev)
        if self.n_priv:
            if self.priv_rec is not None:  # records: the bucket is the top bits of the record
                D.radix_histogram(self.priv_rec, 0, (1 << 64) - 1, self.pw + self.wbits - bits, nb, hist, None)
            else:
                D.radix_histogram(self.priv_k, dom.lower, self.span_m1, self.wbits - bits, nb, hist, self.bad_priv)
        pos = _bound_positions_device(self.pub_chunks, f, t, self.dev)
        bk = self.pub_store[0].view(torch.int64)[pos] if pos is not None else None
        h_hist = torch.empty(nb, dtype=torch.int64, pin_memory=True)
        h_hist.copy_(hist, non_blocking=True)
        h_bk = None
        if bk is not None:
            h_bk = torch.empty(bk.numel(), dtype=torch.int64, pin_memory=True)
            h_bk.copy_(bk, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._hist_pending = (ev, h_hist, h_bk, bits, hist, bk)

    def partition(self):
        """P-MPSM phase 2 (engine.py:359-374, 396-406) on the host, from the
        queued histogram and bounds: splitters, cursors; the partition runs
        are slices of the sorted private run (cut_partitions)."""
        t, dom, f = self.t, self.dom, self.cfg.cdf_fanout
        ev, h_hist, h_bk, bits, _, _ = self._hist_pending
        ev.synchronize()  # the histogram and the bounds only, not the private sort behind them
        hist = h_hist.numpy().copy()
        bk = np.empty(0, np.uint64) if h_bk is None else h_bk.numpy().view(np.uint64).copy()
        if self.packed:
            bk = (bk >> np.uint64(self.pw)) + np.uint64(dom.lower)
        self._hist_pending = None
        bounds, off = [], 0
        for a, b in self.pub_chunks:
            if b > a:
                bounds.append(LocalBounds(bk[off:off + f * t], b - a))
                off += f * t
            else:
                bounds.append(LocalBounds(np.empty(0, np.uint64), 0))
        cdf = build_cdf(bounds, anchor_key=dom.lower)
        ss = compute_splitters(hist, cdf, t, dom, bits)
        self.splitters = ss
        cursors = combine_counts([hist], ss.vector.sp, t)
        cursors.verify_disjoint()
        self.cursors = cursors
        for i, (a, b) in enumerate(self.priv_chunks):
            self._hook(i, "scatter")
            self.stats[i].tuples_scattered = b - a
        return cursors.run_base

    def cut_partitions(self, run_base):
        """P-MPSM phase 3 (engine.py:405-409): partition p's run is
        [run_base[p], run_base[p+1]) of the sorted private run."""
        k, p = self.priv_whole
        self.priv_runs = []
        for i in range(self.t):
            a, b = int(run_base[i]), int(run_base[i + 1])
            self._hook(i, "sort_private")
            self.priv_runs.append((k[a:b], None if p is None else p[a:b]))
            self.stats[i].tuples_sorted_private = b - a

    def _join(self, mode: int, out=None, cap: int = 0):
        if self.packed:
            dense = getattr(self, "priv_dense", None)
            hint = (dense, self.priv_whole[0]) if dense is not None and self.n_priv > 0 else None
            return D.join_pairs_packed([r[0] for r in self.priv_runs], [r[0] for r in self.pub_runs], self.wbits,
                                       self.dom.lower, self.roles.swapped, mode, out, cap, hint)
        return D.join_pairs(self.priv_runs, self.pub_runs, self.roles.swapped, mode, out, cap)

    def join(self):
        """phase 4 (engine.py:228-276, 410-419) for all workers in one launch sequence."""
        for i in range(self.t):
            self._hook(i, "join")
        mode = {"aggregate-max": _lib.MODE_AGGREGATE_MAX, "count": _lib.MODE_COUNT,
                "materialize": _lib.MODE_COUNT}[self.cfg.query_mode]
        self.rec = self._join(mode)

    def materialize(self, total: int) -> np.ndarray:
        if total == 0:
            return np.empty((0, 2), np.uint64)
        out = self._empty(2 * total)
        self._join(_lib.MODE_MATERIALIZE, out, total)
        return out.view(total, 2).cpu().numpy()

    def packed_overflowed(self) -> bool:
        st = getattr(self, "_status", None)
        ovf = st[0] if st is not None else int(self.overflow.item())
        return self.packed and ovf != 0

    def finalize(self, timings: dict) -> JoinResult:
        """engine.py:195-225 plus the checksum and per-worker statistics."""
        t = self.t
        rec_h = self._rec_host if getattr(self, "_rec_host", None) is not None else self.rec.cpu().numpy()
        rec = rec_h.reshape(t, t, _lib.PAIR_FIELDS).astype(object)
        self.check_domain()
        if any(int(f) & _lib.FLAG_UNSORTED for f in rec[:, :, _lib.PAIR_FLAGS].ravel()):
            raise InternalConsistencyError("run keys are not sorted ascending (found by the merge-join walk)")
        count, agg, csum = 0, None, 0
        for i in range(t):
            st = self.stats[i]
            ci, bi = 0, 0
            n_priv_i = int(self.priv_runs[i][0].numel())
            for j in range(t):
                n_pub_j = int(self.pub_runs[j][0].numel())
                if n_priv_i == 0 or n_pub_j == 0:
                    continue
                c = int(rec[i, j, _lib.PAIR_COUNT])
                st.probe_tuples_examined += int(rec[i, j, _lib.PAIR_PROBES])
                st.public_tuples_examined += int(rec[i, j, _lib.PAIR_PROBES]) + int(rec[i, j, _lib.PAIR_EXAMINED])
                if c > 0:
                    st.s_runs_with_matches += 1
                    b = int(rec[i, j, _lib.PAIR_BEST])
                    if ci == 0 or b > bi:
                        bi = b
                    ci += c
                    csum = (csum + int(rec[i, j, _lib.PAIR_CHECKSUM])) & MASK64
            count += ci
            if ci > 0 and self.cfg.query_mode == "aggregate-max":
                agg = bi if agg is None or bi > agg else agg
        materialized = None
        if self.cfg.query_mode == "materialize":
            if count > self.cfg.materialize_cap:
                raise MaterializeCapExceeded(f"join produced {count} pairs, cap is {self.cfg.materialize_cap}")
            materialized = self.materialize(count)
        for st in self.stats:
            st.sort_public_seconds = timings.get("sort_public", 0.0)
            st.sort_private_seconds = timings.get("sort_private", 0.0)
            st.join_seconds = timings.get("join", 0.0)
        return JoinResult(match_count=int(count), aggregate_max=agg, materialized=materialized,
                          phase_timings=timings, worker_stats=self.stats, checksum=int(csum))


def _run(variant: str, r: Relation, s: Relation, cfg: JoinConfig, phase_hook: PhaseHook,
         packed: Optional[bool] = None) -> JoinResult:
    try:
        ctx = JoinContext(r, s, cfg, phase_hook, PACK_RECORDS if packed is None else packed, variant)
        ctx.tl.mark("t0")
        ctx.sort_public()
        ctx.tl.mark("public")
        # with host inputs the private upload runs while the GPU sorts the
        # public run
        ctx.stage_private()
    except _PackOverflow:
        return _run(variant, r, s, cfg, phase_hook, packed=False)
    if variant == "b-mpsm":
        ctx.tl.mark("partitioned")
        ctx.sort_private_chunks()
        ctx.tl.mark("sort_private")
    else:
        # P-MPSM: histogram + public bounds queued, then the private input
        # sorted as one run while the host computes the splitters from them;
        # the run is cut at the partition bounds.  With one worker the
        # partition is the identity (the splitter search returns [0, 2^B]) and
        # the histogram is not needed.
        if ctx.t > 1:
            ctx.queue_histogram()
        ctx.tl.mark("hist_queued")
        ctx.sort_private_whole()
        ctx.tl.mark("sorted_private")
        if ctx.t == 1:
            effective_radix_bits(ctx.dom, cfg.radix_bits)
            for ph in ("histogram", "scatter"):
                ctx._hook(0, ph)
            ctx.stats[0].tuples_scattered = ctx.n_priv
            ctx.tl.mark("partitioned")
            ctx.cut_partitions([0, ctx.n_priv])
        else:
            run_base = ctx.partition()
            ctx.tl.mark("partitioned")
            ctx.cut_partitions(run_base)
        ctx.tl.mark("sort_private")
    ctx.join()
    ctx.tl.mark("join")
    ctx.fetch_status()
    if ctx.packed_overflowed():
        # a payload needs more than 64 - w bits: redo on (key, payload) pairs
        ctx.check_domain()
        return _run(variant, r, s, cfg, phase_hook, packed=False)
    tl = ctx.tl
    if variant == "p-mpsm":
        timings = {"sort_public": tl.seconds("t0", "public"),
                   "partition": tl.seconds("public", "hist_queued") + tl.seconds("sorted_private", "partitioned"),
                   "sort_private": tl.seconds("hist_queued", "sorted_private"),
                   "join": tl.seconds("sort_private", "join"), "total": tl.seconds("t0", "join")}
    else:
        timings = {"sort_public": tl.seconds("t0", "public"), "partition": 0.0,
                   "sort_private": tl.seconds("partitioned", "sort_private"), "join": tl.seconds("sort_private", "join"),
                   "total": tl.seconds("t0", "join")}
    return ctx.finalize(timings)


def run_bmpsm(r: Relation, s: Relation, cfg: JoinConfig, *, phase_hook: PhaseHook = None) -> JoinResult:
    """Basic variant: sort both inputs chunk-wise, join every private run
    against every public run (engine.py:279-334)."""
    return _run("b-mpsm", r, s, cfg, phase_hook)


def run_pmpsm(r: Relation, s: Relation, cfg: JoinConfig, *, phase_hook: PhaseHook = None) -> JoinResult:
    """Range-partitioned variant (engine.py:337-433)."""
    return _run("p-mpsm", r, s, cfg, phase_hook)


def _payloads_below_2_63(rel: Relation) -> bool:
    if rel.cardinality == 0:
        return True
    p = rel.payloads
    if isinstance(p, torch.Tensor) and p.is_cuda:
        return D.domain_report(p, 0, (1 << 63) - 1)[0] == 0
    return int(np.asarray(rel.host_payloads()).max()) < 1 << 63


def run_hash_oracle(r: Relation, s: Relation, cfg: JoinConfig) -> JoinResult:
    """algorithm="hash-oracle" (engine.py:462-465 -> datagen.hash_join_oracle,
    datagen.py:121-200) served on the GPU: the reference's ground-truth join
    over the full 64-bit key space (no key domain), build side = the smaller
    input, with its result shape -- phase_timings build / join / total,
    worker_stats [], aggregate_max only in aggregate-max mode with matches,
    materialized (r, s) rows (MaterializeCapExceeded past the cap), payloads
    >= 2^63 rejected with ValueError.  The build and probe sides are sorted
    by the run sort over all 64 key bits and joined by the merge kernel (the
    same COUNT / MAX / checksum; pair order is key order, not probe order)."""
    if isinstance(r, PackedRelation) or isinstance(s, PackedRelation):
        raise ConfigurationError("algorithm 'hash-oracle' joins Relations (keys and payloads), not PackedRelations")
    for name, rel in (("r", r), ("s", s)):
        if not _payloads_below_2_63(rel):
            raise ValueError(f"relation {name} has payloads >= 2^63; aggregate undefined")
    dev = D.ensure_device()
    build_is_r = r.cardinality <= s.cardinality
    build, probe = (r, s) if build_is_r else (s, r)
    tl = _Timeline()
    tl.mark("t0")
    full = (1 << 64) - 1

    def sorted_run(rel):
        k, p = D.to_device(rel.keys, dev), D.to_device(rel.payloads, dev)
        n = int(k.numel())
        ok, op = torch.empty_like(k), torch.empty_like(p)
        if n:
            tk, tp = torch.empty_like(k), torch.empty_like(p)
            D.sort_pairs(k, p, 0, full, 64, ok, op, tk, tp, None)
        return ok, op

    b_run = sorted_run(build)
    p_run = sorted_run(probe)
    tl.mark("build")
    if b_run[0].numel() == 0 or p_run[0].numel() == 0:
        rec = None
    else:
        rec = D.join_pairs([b_run], [p_run], not build_is_r, _lib.MODE_COUNT)
    tl.mark("join")
    count, best, csum = 0, None, 0
    if rec is not None:
        row = rec.cpu().numpy()[0]
        count = int(row[_lib.PAIR_COUNT])
        best = int(row[_lib.PAIR_BEST]) if count else None
        csum = int(row[_lib.PAIR_CHECKSUM])
        if int(row[_lib.PAIR_FLAGS]) & _lib.FLAG_UNSORTED:
            raise InternalConsistencyError("run keys are not sorted ascending (found by the merge-join walk)")
    materialized = None
    if cfg.query_mode == "materialize":
        if count > cfg.materialize_cap:
            raise MaterializeCapExceeded(f"oracle output exceeds cap {cfg.materialize_cap}")
        if count:
            out = torch.empty(2 * count, dtype=torch.uint64, device=dev)
            D.join_pairs([b_run], [p_run], not build_is_r, _lib.MODE_MATERIALIZE, out, count)
            materialized = out.view(count, 2).cpu().numpy()
        else:
            materialized = np.empty((0, 2), np.uint64)
    torch.cuda.current_stream().synchronize()
    t_build, t_join = tl.seconds("t0", "build"), tl.seconds("build", "join")
    return JoinResult(match_count=count, aggregate_max=best if cfg.query_mode == "aggregate-max" else None,
                      materialized=materialized,
                      phase_timings={"build": t_build, "join": t_join, "total": t_build + t_join},
                      worker_stats=[], checksum=csum)


def hash_join_oracle(r: Relation, s: Relation, query_mode: str = "aggregate-max",
                     cap: Optional[int] = None) -> JoinResult:
    """The reference's ground-truth join as a function (datagen.py:121-200):
    build on the smaller input, result shape of run_hash_oracle; cap None =
    no materialize cap."""
    cfg = JoinConfig(algorithm="hash-oracle", query_mode=query_mode,
                     materialize_cap=(1 << 62) if cap is None else int(cap))
    return run_hash_oracle(r, s, cfg)


def run_join(r: Relation, s: Relation, cfg: JoinConfig, *, phase_hook: PhaseHook = None) -> JoinResult:
    """Dispatch on cfg.algorithm (engine.py:456-466)."""
    if cfg.algorithm == "b-mpsm":
        return run_bmpsm(r, s, cfg, phase_hook=phase_hook)
    if cfg.algorithm == "p-mpsm":
        return run_pmpsm(r, s, cfg, phase_hook=phase_hook)
    if cfg.algorithm == "hash-oracle":
        return run_hash_oracle(r, s, cfg)
    raise ConfigurationError(f"unknown algorithm {cfg.algorithm!r}")
