"""Multi-GPU MPSM join: one process per GPU, torch.distributed (NCCL) plumbing.

The paper's T workers become the G ranks of the process group (SURVEY.md
8(e)); rank i holds position-shard i of R and S (the chunk rule,
core.py:263-279) and plays worker i of P-MPSM (engine.py:337-433):

  1. sort its public shard into public run i                    (local, HBM)
  2. histogram its private shard; all-gather the histograms and
     the f*G equi-height bounds of every public run             (tiny collective)
  3. every rank computes the same splitters (skew.py:287-315)
  4. stable partition scatter of the private shard into G send
     segments (the reference's arena layout, partition.py:233)
  5. ONE all-to-all(v) of the private tuples over NVLink         (NCCL)
  6. sort the received partition into private run i
  7. merge-join private run i against every public run; the
     G-1 remote runs are read in place through NVLink peer loads
     (CUDA IPC mappings, the paper's remote-NUMA reads,
     engine.py:249-260)
  8. all-gather the G x G pair records and fold them exactly like
     the single-GPU engine (_finalize, engine.py:195-225)

Device work goes through a backend object.  The product backend is
CudaBackend (libmpsm_b200.so); tests/test_distributed.py runs the same
protocol under gloo with a CPU backend built on the test oracle, which is how
the multi-rank host logic is covered without several GPUs.
"""

from __future__ import annotations

import json
import math
import os
import time
from typing import Optional

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from . import device as D
from .core import (
    ConfigurationError,
    DomainError,
    InternalConsistencyError,
    JoinConfig,
    JoinResult,
    MaterializeCapExceeded,
    Relation,
    WorkerStats,
)
from .engine import HOST_PACK, MASK64, PACK_RECORDS, choose_roles
from .partition import combine_counts, effective_radix_bits
from .skew import LocalBounds, bound_positions, build_cdf, compute_splitters


class PeerRun:
    """A run in a peer rank's HBM, mapped into this process (read by the
    merge kernel with NVLink peer loads): exposes what device.join_* read."""

    __slots__ = ("ptr", "n", "device")

    def __init__(self, ptr: int, n: int, device):
        self.ptr, self.n, self.device = ptr, n, device

    def data_ptr(self) -> int:
        return self.ptr

    def numel(self) -> int:
        return self.n


# mappings of peer ranks' public runs: (device, peer) -> (handle bytes, base).
# A peer names its public run by the cudaMalloc block holding it; it keeps
# that block alive (CudaBackend's persistent public store) and only retires
# it after the final collective of a join in which every importer has seen
# the new handle -- an importer closes the old mapping the moment a peer's
# handle changes, so no block is freed while mapped (CUDA IPC forbids that).
_IPC_PEERS: dict = {}


def ipc_share(t: torch.Tensor) -> tuple:
    """(handle bytes, byte offset, numel) naming a device tensor for peers"""
    import ctypes

    h = (ctypes.c_char * 64)()
    off = ctypes.c_int64(0)
    _lib.check(_lib.load().mpsm_ipc_get_handle(t.data_ptr(), h, ctypes.byref(off)), "mpsm_ipc_get_handle")
    return bytes(h), int(off.value), int(t.numel())


def ipc_open(shared: tuple, device, peer: int = -1) -> PeerRun:
    """map a peer's tensor into the current device; one mapping per peer,
    replaced (old one closed) when the peer's block changes"""
    import ctypes

    handle, off, n = shared
    key = (torch.cuda.current_device(), peer if peer >= 0 else handle)
    cached = _IPC_PEERS.get(key)
    if cached is None or cached[0] != handle:
        if cached is not None:
            _lib.check(_lib.load().mpsm_ipc_close_handle(ctypes.c_void_p(cached[1])), "mpsm_ipc_close_handle")
            del _IPC_PEERS[key]
        p = ctypes.c_void_p()
        buf = (ctypes.c_char * 64).from_buffer_copy(handle)
        _lib.check(_lib.load().mpsm_ipc_open_handle(buf, ctypes.byref(p)), "mpsm_ipc_open_handle")
        _IPC_PEERS[key] = (handle, int(p.value))
    return PeerRun(_IPC_PEERS[key][1] + off, n, device)


def ipc_close_all() -> None:
    """close every peer mapping of this process (after the last join of a
    process group, before it is destroyed)"""
    import ctypes

    torch.cuda.synchronize()
    for key, (_, base) in list(_IPC_PEERS.items()):
        _lib.check(_lib.load().mpsm_ipc_close_handle(ctypes.c_void_p(base)), "mpsm_ipc_close_handle")
        del _IPC_PEERS[key]


class CudaBackend:
    """Device operations of one rank on its own GPU."""

    def __init__(self, device: Optional[torch.device] = None, packed: Optional[bool] = None,
                 comm_device: Optional[torch.device] = None):
        self.dev = D.ensure_device(device)
        self.packed_pref = PACK_RECORDS if packed is None else packed
        # where the all-to-all buffers live: the GPU (NCCL), or the host for a
        # CPU process group (gloo; tests run several ranks on one GPU)
        self.comm_device = comm_device if comm_device is not None else self.dev
        # the public run lives in a grow-only store the backend owns: peers map
        # its block (CUDA IPC), so it must outlive their mappings (see _IPC_PEERS)
        self._pub = None
        self._retired = []

    def unpacked(self):
        return type(self)(device=self.dev, packed=False, comm_device=self.comm_device)

    def _public_out(self, n: int) -> torch.Tensor:
        if self._pub is None or self._pub.numel() < n:
            if self._pub is not None:
                self._retired.append(self._pub)  # released after this join's last collective
            self._pub = torch.empty(max(n, 1), dtype=torch.uint64, device=self.dev)
        return self._pub[:n]

    def release(self) -> None:
        """after a join's final collective: every importer has switched to the
        current public store, the retired ones can go"""
        self._retired.clear()

    def upload(self, rel):
        """host columns of a packed join -> 8-B records on the device (half the
        PCIe bytes, device.upload_records); None for device columns or pairs"""
        if not (self.packed and HOST_PACK):
            return None
        hk, hp = D.host_columns(rel.keys), D.host_columns(rel.payloads)
        if hk is None or hp is None:
            return None
        rec = self.empty(int(hk[0].shape[0]))
        bad, ovf = D.upload_records(hk[0], hp[0], self.dom.lower, self.span_m1, self.wbits, rec)
        if bad >= 0:
            self.bad.fill_(bad)
        if ovf:
            self.overflow.fill_(1)
        return rec

    def setup(self, dom):
        self.dom = dom
        self.wbits = dom.width_bits
        self.packed = self.packed_pref and 1 <= self.wbits <= 63
        self.pw = 64 - self.wbits
        self.span_m1 = dom.upper - dom.lower - 1
        self.bad = D.new_bad_flag(self.dev)
        self.overflow = torch.zeros(1, dtype=torch.int32, device=self.dev)

    def to_device(self, a) -> torch.Tensor:
        return D.to_device(a, self.dev)

    def empty(self, n: int) -> torch.Tensor:
        return torch.empty(n, dtype=torch.uint64, device=self.dev)

    def sort(self, k, p, public: bool = False):
        n = int(k.numel())
        if self.packed:
            out = self._public_out(n) if public else self.empty(n)
            D.sort_packed(k, p, self.dom.lower, self.span_m1, self.wbits, out, self.empty(n), self.bad, self.overflow)
            return (out, None)
        if public:  # pairs: keys and payloads in one store block
            st = self._public_out(2 * n)
            ok, op = st[:n], st[n:]
        else:
            ok, op = self.empty(n), self.empty(n)
        D.sort_pairs(k, p, self.dom.lower, self.span_m1, self.wbits, ok, op, self.empty(n), self.empty(n), self.bad)
        return (ok, op)

    def histogram_async(self, keys, shift: int, nb: int) -> torch.Tensor:
        """Queue the private histogram; read it with .cpu() later."""
        counts = torch.zeros(nb, dtype=torch.int64, device=self.dev)
        D.radix_histogram(keys, self.dom.lower, self.span_m1, shift, nb, counts, self.bad)
        return counts

    def histogram(self, keys, shift: int, nb: int) -> np.ndarray:
        return self.histogram_async(keys, shift, nb).cpu().numpy()

    def bound_keys(self, run, f: int, t: int) -> np.ndarray:
        n = int(run[0].numel())
        if n == 0:
            return np.empty(0, np.uint64)
        pos = torch.from_numpy(bound_positions(n, f, t)).to(self.dev)
        vals = run[0].view(torch.int64)[pos].cpu().numpy().view(np.uint64)
        if self.packed:
            vals = (vals >> np.uint64(self.pw)) + np.uint64(self.dom.lower)
        return vals

    def partition(self, k, p, shift: int, sp: np.ndarray, npart: int, starts: np.ndarray):
        n = int(k.numel())
        sk, spay = self.empty(n), self.empty(n)
        written = torch.zeros(npart, dtype=torch.int64, device=self.dev)
        D.scatter_chunk(k, p, self.dom.lower, shift, torch.from_numpy(sp.astype(np.int32)).to(self.dev), sp.shape[0],
                        npart, torch.from_numpy(starts.astype(np.int64)).to(self.dev), sk, spay, written)
        return sk, spay

    def partition_records(self, k, p, shift: int, sp: np.ndarray, npart: int):
        """packed join: the private shard straight into records grouped by
        destination rank (one pass), or None for pair joins"""
        if not self.packed:
            return None
        rec = self.empty(int(k.numel()))
        spd = torch.from_numpy(sp.astype(np.int32)).to(self.dev)
        D.partition_records(k, p, self.dom.lower, self.span_m1, self.wbits, shift, spd, npart, rec, self.bad,
                            self.overflow)
        return rec

    def sort_records(self, rec, public: bool = False):
        n = int(rec.numel())
        out = self._public_out(n) if public else self.empty(n)
        D.sort_records(rec, self.wbits, out, self.empty(n))
        return (out, None)

    def bad_index(self) -> int:
        return int(self.bad.item())

    def overflowed(self) -> bool:
        return self.packed and int(self.overflow.item()) != 0

    def share(self, run):
        """CUDA IPC description of a run, for peer ranks (mpsm_ipc_get_handle)."""
        return [None if t is None else ((b"", 0, 0) if t.numel() == 0 else ipc_share(t)) for t in run]

    def open(self, shared, peer: int = -1):
        """a peer's run mapped into this rank's device (lazy NVLink peer access)"""
        return tuple(None if s is None else (PeerRun(0, 0, self.dev) if s[2] == 0 else ipc_open(s, self.dev, peer))
                     for s in shared)

    def join(self, priv_runs, pub_runs, swap: bool, mode: int, out=None, cap: int = 0) -> torch.Tensor:
        if self.packed:
            return D.join_pairs_packed([r[0] for r in priv_runs], [r[0] for r in pub_runs], self.wbits,
                                       self.dom.lower, swap, mode, out, cap)
        return D.join_pairs(priv_runs, pub_runs, swap, mode, out, cap)

    def materialize(self, priv_runs, pub_runs, swap: bool, total: int) -> np.ndarray:
        if total == 0:
            return np.empty((0, 2), np.uint64)
        out = self.empty(2 * total)
        self.join(priv_runs, pub_runs, swap, _lib.MODE_MATERIALIZE, out, total)
        return out.view(total, 2).cpu().numpy()

    def records(self, rec) -> np.ndarray:
        return rec.cpu().numpy()

    def sync(self):
        torch.cuda.current_stream().synchronize()


def _gather_u64(vec, group, device) -> np.ndarray:
    """all-gather of one fixed-length u64 vector per rank -> [G, L].  One
    tensor collective (NCCL on the GPU, gloo on the host) instead of the
    pickling two-step all_gather_object: the protocol's host round trips are
    on the critical path between the public sort and the partition."""
    vec = np.ascontiguousarray(vec, dtype=np.uint64)
    G = dist.get_world_size(group)
    if G == 1:
        return vec[None, :].copy()
    t = torch.from_numpy(vec.view(np.int64).copy()).to(device)
    outs = [torch.empty_like(t) for _ in range(G)]
    dist.all_gather(outs, t, group=group)
    return torch.stack(outs).cpu().numpy().view(np.uint64)


def _enc_share(shared) -> np.ndarray:
    """CudaBackend.share() of a run -> fixed u64 layout (per slot: present,
    numel, offset, 64-B handle)"""
    out = np.zeros(2 * 11, np.uint64)
    for i, sh in enumerate(shared):
        if sh is None:
            continue
        h, off, n = sh
        out[11 * i:11 * i + 3] = (1, n, off)
        if n:
            out[11 * i + 3:11 * i + 11] = np.frombuffer(h, np.uint64)
    return out


def _dec_share(v: np.ndarray) -> list:
    slots = []
    for i in range(2):
        if v[11 * i] == 0:
            slots.append(None)
            continue
        n, off = int(v[11 * i + 1]), int(v[11 * i + 2])
        slots.append((v[11 * i + 3:11 * i + 11].tobytes() if n else b"", off, n))
    return slots


def _gather_obj(obj, group):
    if dist.get_world_size(group) == 1:
        return [obj]
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, obj, group=group)
    return out


class _Guard:
    """Failure protocol between the collectives of one join.

    A rank whose local work raises does not skip ahead: it enters the next
    collective of the protocol with a failure flag (appended to the vector
    every rank gathers there, or a one-word MAX all-reduce before the
    variable-size all-to-all), and then every rank raises at that same point
    -- the failing rank its own exception, the root cause, the others a
    RuntimeError naming it (the reference prefers the root cause over the
    broken-barrier noise of its worker threads, engine.py:440-453).  No rank
    blocks on a peer that has already given up; a peer that dies outright is
    caught by the process group's timeout (init_process_group(timeout=...))."""

    def __init__(self, group, cdev):
        self.group, self.cdev = group, cdev
        self.err: Optional[BaseException] = None

    def call(self, fn, *args, **kw):
        if self.err is not None:
            return None
        try:
            return fn(*args, **kw)
        except Exception as exc:  # noqa: BLE001 - re-raised at the next collective
            self.err = exc
            return None

    def _raise(self, flags) -> None:
        bad = [int(i) for i in np.flatnonzero(np.asarray(flags))]
        if bad:
            if self.err is not None:
                raise self.err
            raise RuntimeError(f"distributed join: rank(s) {bad} failed before this collective "
                               "(their own exception is the root cause)")
        if self.err is not None:  # world of one, no collective
            raise self.err

    def gather(self, vec, length: int) -> np.ndarray:
        """_gather_u64 of a fixed-length vector plus this rank's status -> [G, length]"""
        v = np.zeros(length + 1, np.uint64)
        if self.err is None and vec is not None:
            v[:length] = np.asarray(vec, np.uint64)
        v[length] = 0 if self.err is None else 1
        allv = _gather_u64(v, self.group, self.cdev)
        self._raise(allv[:, length])
        return allv[:, :length]

    def gather_obj(self, obj) -> list:
        out = _gather_obj((self.err is not None, None if self.err is not None else obj), self.group)
        self._raise([x[0] for x in out])
        return [x[1] for x in out]

    def check(self) -> None:
        """a status-only collective (MAX all-reduce of one word)"""
        if dist.get_world_size(self.group) == 1:
            self._raise([0])
            return
        t = torch.tensor([0 if self.err is None else 1], dtype=torch.int64, device=self.cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        if int(t.item()):
            if self.err is not None:
                raise self.err
            raise RuntimeError("distributed join: a peer rank failed before the all-to-all "
                               "(its own exception is the root cause)")


def _alltoall(be, k, p, send_counts, recv_counts, group):
    """all-to-all(v) of the private tuples; received in source-rank order."""
    n_recv = int(recv_counts.sum())
    rk = torch.empty(n_recv, dtype=torch.int64, device=be.comm_device)
    rp = torch.empty(n_recv, dtype=torch.int64, device=be.comm_device)
    sc = [int(x) for x in send_counts]
    rc = [int(x) for x in recv_counts]
    dist.all_to_all_single(rk, k.view(torch.int64).to(be.comm_device), rc, sc, group=group)
    dist.all_to_all_single(rp, p.view(torch.int64).to(be.comm_device), rc, sc, group=group)
    return rk.view(torch.uint64).to(k.device), rp.view(torch.uint64).to(k.device)


def _alltoall_one(be, x, send_counts, recv_counts, group):
    """all-to-all(v) of one u64 column (packed records); source-rank order."""
    out = torch.empty(int(recv_counts.sum()), dtype=torch.int64, device=be.comm_device)
    dist.all_to_all_single(out, x.view(torch.int64).to(be.comm_device), [int(v) for v in recv_counts],
                           [int(v) for v in send_counts], group=group)
    return out.view(torch.uint64).to(x.device)


def run_join_distributed(r: Relation, s: Relation, cfg: JoinConfig, *, group=None, backend=None,
                         timings: Optional[dict] = None) -> JoinResult:
    """P-MPSM over the ranks of `group`; r and s are this rank's shards.

    Every rank returns the same JoinResult (worker i = rank i).  cfg.threads is
    ignored: the worker count is the group size.  Local failures follow the
    _Guard protocol (every rank raises at the same collective).
    """
    if cfg.algorithm != "p-mpsm":
        raise ConfigurationError("the distributed engine runs p-mpsm")
    G = dist.get_world_size(group)
    me = dist.get_rank(group)
    be = backend or CudaBackend()
    dom = cfg.key_domain
    t0 = time.perf_counter()
    trace = [] if (timings is not None and os.environ.get("MPSM_DIST_TRACE") == "1") else None

    def _tr(what):  # host timeline (tools/dist_phase_timing.py)
        if trace is not None:
            trace.append((what, 1e3 * (time.perf_counter() - t0)))

    cdev = getattr(be, "comm_device", torch.device("cpu"))
    gd = _Guard(group, cdev)
    gd.call(be.setup, dom)
    sizes = gd.gather([r.cardinality, s.cardinality], 2).astype(np.int64)
    _tr("sizes gathered")
    n_r, n_s = int(sizes[:, 0].sum()), int(sizes[:, 1].sum())
    roles = choose_roles(n_r, n_s, cfg.role_policy)
    private, public = (r, s) if roles.private == "r" else (s, r)
    bits = effective_radix_bits(dom, cfg.radix_bits)
    if (1 << bits) < G:
        raise ConfigurationError(f"effective radix bits {bits} give fewer buckets than {G} workers")
    nb = 1 << bits
    shift = dom.width_bits - bits
    f = cfg.cdf_fanout
    kb = f * G
    stats = [WorkerStats(i) for i in range(G)]

    # 1-2: private histogram (queued first: it needs only the private
    # shard), public run, bounds
    def local_public():
        # host-resident public shards of a packed join cross PCIe as 8-B records
        pub_rec = be.upload(public) if hasattr(be, "upload") else None
        pk, pp = be.to_device(private.keys), be.to_device(private.payloads)
        h_dev = be.histogram_async(pk, shift, nb) if hasattr(be, "histogram_async") else None
        if pub_rec is not None:
            pub_run = be.sort_records(pub_rec, public=True)
        else:
            pub_run = be.sort(be.to_device(public.keys), be.to_device(public.payloads), public=True)
        hist = h_dev.cpu().numpy() if h_dev is not None else be.histogram(pk, shift, nb)
        bk = np.asarray(be.bound_keys(pub_run, f, G), np.uint64)
        # per rank: [hist (nb) | public cardinality | bad index | #bounds | f*G bounds]
        vec = np.zeros(nb + 3 + kb, np.uint64)
        vec[:nb] = np.asarray(hist, np.int64).view(np.uint64)
        vec[nb:nb + 3] = np.array([int(public.cardinality), be.bad_index(), bk.shape[0]], np.int64).view(np.uint64)
        vec[nb + 3:nb + 3 + bk.shape[0]] = bk
        return pk, pp, pub_run, vec

    loc = gd.call(local_public)
    pk, pp, pub_run, vec = loc if loc is not None else (None, None, None, None)
    _tr("public sorted, hist + bounds on host")
    allv = gd.gather(vec, nb + 3 + kb)
    info = []
    for v in allv:
        card, bad, nbk = (int(x) for x in v[nb:nb + 3].view(np.int64))
        info.append((v[:nb].view(np.int64).copy(), v[nb + 3:nb + 3 + nbk].copy(), card, bad))
    _tr("gathered")
    if any(x[3] != -1 for x in info):
        raise DomainError("a relation shard has out-of-domain keys")
    t_pub = time.perf_counter()
    # 3: identical splitters on every rank
    cdf = build_cdf([LocalBounds(x[1], x[2]) for x in info], anchor_key=dom.lower)
    hists = [x[0] for x in info]
    ss = compute_splitters(np.sum(hists, axis=0), cdf, G, dom, bits)
    cursors = combine_counts(hists, ss.vector.sp, G)
    cursors.verify_disjoint()
    send_counts = cursors.counts[me]
    recv_counts = cursors.counts[:, me]
    send_starts = np.zeros(G, np.int64)
    np.cumsum(send_counts[:-1], out=send_starts[1:])
    _tr("splitters")

    # 4-5: scatter into send segments, one all-to-all
    def local_partition():
        rec = be.partition_records(pk, pp, shift, ss.vector.sp, G) if hasattr(be, "partition_records") else None
        if rec is not None:
            return rec, None, None
        sk, sp = be.partition(pk, pp, shift, ss.vector.sp, G, send_starts)
        return None, sk, sp

    part = gd.call(local_partition)
    gd.check()
    rec, sk, sp = part
    packed_xchg = rec is not None
    if packed_xchg:  # packed join: one all-to-all of 8-B records
        rr = _alltoall_one(be, rec, send_counts, recv_counts, group)
        rk = rp = None
        n_recv_priv = int(rr.numel())
    else:
        rk, rp = _alltoall(be, sk, sp, send_counts, recv_counts, group)
        rr = None
        n_recv_priv = int(rk.numel())
    del pk, pp, rec, sk, sp
    t_part = time.perf_counter()
    _tr("partition + all-to-all issued")

    # 6: private run; this rank's public run named for the peers
    def local_private():
        run = be.sort_records(rr) if packed_xchg else be.sort(rk, rp)
        be.sync()
        return run, (be.share(pub_run) if G > 1 else None)

    got = gd.call(local_private)
    priv_run, my_share = got if got is not None else (None, None)
    t_sort = time.perf_counter()
    _tr("private sorted")
    # 7: join against every public run (remote ones through peer mappings)
    # rank-rotated order, own run first (engine.py:251: (i + k) % T): at any
    # moment each rank reads a different peer, so no peer's NVLink serves
    # all readers at once
    order = [(me + k) % G for k in range(G)]
    if G > 1:
        if isinstance(be, CudaBackend):  # IPC handles: fixed layout, one tensor gather
            enc = _enc_share(my_share) if my_share is not None else None
            shared = [_dec_share(v) for v in gd.gather(enc, 22)]
        else:
            shared = gd.gather_obj(my_share)
    mode = {"aggregate-max": _lib.MODE_AGGREGATE_MAX, "count": _lib.MODE_COUNT,
            "materialize": _lib.MODE_COUNT}[cfg.query_mode]

    def local_join():
        if G > 1:
            pub_runs = [pub_run if j == me else be.open(shared[j], j) for j in order]
        else:
            pub_runs = [pub_run]
        rec_rot = np.asarray(be.records(be.join([priv_run], pub_runs, roles.swapped, mode))).reshape(
            G, _lib.PAIR_FIELDS)
        rec_h = np.empty_like(rec_rot)
        rec_h[order] = rec_rot  # back to public-run (rank) order
        if any(int(x) & _lib.FLAG_UNSORTED for x in rec_h[:, _lib.PAIR_FLAGS]):
            raise InternalConsistencyError("run keys are not sorted ascending (found by the merge-join walk)")
        fin = np.concatenate([np.asarray(rec_h, np.uint64).ravel(),
                              np.array([n_recv_priv, int(be.overflowed())], np.uint64)])
        return pub_runs, rec_h, fin

    got = gd.call(local_join)
    pub_runs, rec_h, fin = got if got is not None else (None, None, None)
    gathered = [(v[:-2].reshape(G, _lib.PAIR_FIELDS), int(v[-2]), bool(v[-1]))
                for v in gd.gather(fin, G * _lib.PAIR_FIELDS + 2)]
    if any(g[2] for g in gathered):
        # a payload is wider than a packed record allows: redo on pairs
        if hasattr(be, "release"):
            be.release()
        return run_join_distributed(r, s, cfg, group=group, backend=be.unpacked(), timings=timings)
    t_join = time.perf_counter()
    # 8: fold, as engine.finalize with worker i = rank i
    pub_sizes = [x[2] for x in info]
    count, agg, csum = 0, None, 0
    for i in range(G):
        rec_i = gathered[i][0].reshape(G, _lib.PAIR_FIELDS).astype(object)
        st = stats[i]
        st.tuples_sorted_public = pub_sizes[i]
        st.tuples_sorted_private = gathered[i][1]
        st.tuples_scattered = int(cursors.counts[i].sum())
        ci, bi = 0, 0
        for j in range(G):
            if gathered[i][1] == 0 or pub_sizes[j] == 0:
                continue
            c = int(rec_i[j, _lib.PAIR_COUNT])
            st.probe_tuples_examined += int(rec_i[j, _lib.PAIR_PROBES])
            st.public_tuples_examined += int(rec_i[j, _lib.PAIR_PROBES]) + int(rec_i[j, _lib.PAIR_EXAMINED])
            if c > 0:
                st.s_runs_with_matches += 1
                b = int(rec_i[j, _lib.PAIR_BEST])
                if ci == 0 or b > bi:
                    bi = b
                ci += c
                csum = (csum + int(rec_i[j, _lib.PAIR_CHECKSUM])) & MASK64
        count += ci
        if ci > 0 and cfg.query_mode == "aggregate-max":
            agg = bi if agg is None or bi > agg else agg
    materialized = None
    if cfg.query_mode == "materialize":
        if count > cfg.materialize_cap:
            raise MaterializeCapExceeded(f"join produced {count} pairs, cap is {cfg.materialize_cap}")
        mine = int(sum(int(x) for x in rec_h.reshape(G, _lib.PAIR_FIELDS)[:, _lib.PAIR_COUNT]))
        local = gd.call(be.materialize, [priv_run], pub_runs, roles.swapped, mine)
        parts = gd.gather_obj(local)
        materialized = np.concatenate(parts, axis=0) if parts else np.empty((0, 2), np.uint64)
    if hasattr(be, "release"):
        be.release()  # every importer is past its mapping step of this join
    tm = {"sort_public": t_pub - t0, "partition": t_part - t_pub, "sort_private": t_sort - t_part,
          "join": t_join - t_sort, "total": t_join - t0}
    if timings is not None:
        timings.update(tm)
        if trace is not None:
            _tr("folded")
            timings["trace"] = trace
    return JoinResult(match_count=int(count), aggregate_max=agg, materialized=materialized, phase_timings=tm,
                      worker_stats=stats, checksum=int(csum))


# ------------------------------------------------------------------ bench
def fk_shard_device(n_r: int, n_s: int, rank: int, world: int, seed: int, device) -> tuple:
    """Position-shard `rank` of a world-wide FK workload generated on the GPU
    (datagen.fk_range_device): a rank builds only its shard."""
    from .core import chunk_bounds
    from .datagen import fk_range_device

    return fk_range_device(n_r, n_s, chunk_bounds(n_r, world)[rank], chunk_bounds(n_s, world)[rank], seed, device)


# BASELINE.json configs the multi-GPU bench runs: (n_r, n_s, kind, scaling)
DIST_CONFIGS = {
    "cfg5": (1_600_000_000, 6_400_000_000, "fk", "strong"),   # configs[4]: whole-box scale-out
    "cfg4": (400_000_000, 1_600_000_000, "negcorr", "strong"),  # configs[3] on 8 B200
    "cfg2": (100_000_000, 400_000_000, "fk", "weak"),          # configs[1] per GPU (weak scaling)
}


def dist_workload(name: str, G: int) -> tuple:
    """(config dict, KeyDomain, n_r, n_s, kind, scaling) of a DIST_CONFIGS
    workload over G GPUs -- the description both bench arms print (ours and
    the --impl reference arm's bounded sample of the same workload)."""
    from .core import KeyDomain

    n_r, n_s, kind, scaling = DIST_CONFIGS[name]
    if scaling == "weak":
        n_r, n_s = n_r * G, n_s * G
    dom = KeyDomain(1, n_r + 1) if kind == "fk" else KeyDomain(1, 1 << 32)
    config = {"workload": f"{name}: |R|={n_r:,} |S|={n_s:,} "
                          + ("FK join" if kind == "fk" else "negatively correlated 80-20 skew join")
                          + f" sharded by position over {G} GPUs",
              "algorithm": "p-mpsm", "key_domain": [dom.lower, dom.upper],
              "l2": "inputs >> L2 (no flush needed)"}
    return config, dom, n_r, n_s, kind, scaling


def _dist_inputs(name: str, G: int, me: int, dev):
    """this rank's position shards of a DIST_CONFIGS workload (counter-based,
    generated on the device chunk by chunk) -> (R, S, KeyDomain, n_r, n_s)"""
    from .core import KeyDomain, chunk_bounds
    from .datagen import fk_shard_chunked, skewed_8020_range_device

    n_r, n_s, kind, scaling = DIST_CONFIGS[name]
    if scaling == "weak":
        n_r, n_s = n_r * G, n_s * G
    if kind == "fk":
        r, s = fk_shard_chunked(n_r, n_s, me, G, 0, dev)
        return r, s, KeyDomain(1, n_r + 1), n_r, n_s
    dom = KeyDomain(1, 1 << 32)
    r = skewed_8020_range_device(n_r, dom, "low", chunk_bounds(n_r, G)[me], 0, dev)
    s = skewed_8020_range_device(n_s, dom, "high", chunk_bounds(n_s, G)[me], 1, dev)
    return r, s, dom, n_r, n_s


def bench_main(args, metric, Clocks):
    """bench.py under torchrun: BASELINE configs[4] (cfg5, 1.6B x 6.4B, strong
    scaling over the ranks) by default, --dist-config cfg4 / cfg2 (cfg2-sized
    shards per GPU, weak scaling).  Every rank generates its position shards
    on its GPU; the join result is checked (COUNT, MAX, checksum) against the
    sharded torch checker (tests/torch_check.py) computed before the timed
    region."""
    import datetime

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    timeout = datetime.timedelta(seconds=int(os.environ.get("MPSM_DIST_TIMEOUT", "600")))
    dist.init_process_group("nccl", device_id=dev, timeout=timeout)
    G, me = dist.get_world_size(), dist.get_rank()
    name = getattr(args, "dist_config", None) or "cfg5"
    n_r0, n_s0, kind, scaling = DIST_CONFIGS[name]
    r, s, dom, n_r, n_s = _dist_inputs(name, G, me, dev)
    # the expected result, before any join buffer exists (the checker
    # rebuilds all of R on every rank)
    from tests import torch_check as tc

    want = tc.fk_join_dist(r, s, n_r) if kind == "fk" else tc.general_join_dist(r, s)
    torch.cuda.empty_cache()
    cfg = JoinConfig(threads=G, key_domain=dom)
    be = CudaBackend()
    for _ in range(args.warmup):
        res = run_join_distributed(r, s, cfg, backend=be)
    got = (res.match_count, res.aggregate_max, res.checksum)
    clocks = Clocks(local)
    clocks.start()
    dist.barrier()
    torch.cuda.synchronize()
    w0 = time.time()
    _lib.profile_enable(True)
    l0 = _lib.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        res = run_join_distributed(r, s, cfg, backend=be)
    e1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / args.steps], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    dist.barrier()
    clocks.mark(w0, time.time())
    clk = clocks.stop()
    launches = _lib.launch_count() - l0
    sc_ms, sc_n = _lib.profile_read("seg_scatter")
    mg_ms, _ = _lib.profile_read("merge")
    _lib.profile_enable(False)
    ms = float(ms.item())
    timed_ok = (res.match_count, res.aggregate_max, res.checksum) == got

    # roofline of the radix scatter on this rank: public sort (packing pass +
    # record passes) and the record sort of the received private tuples
    passes = _lib.load().mpsm_sort_pass_count(dom.width_bits)
    n_recv = res.worker_stats[me].tuples_sorted_private
    sc_bytes = args.steps * (s.cardinality * (24 + 16 * (passes - 1)) + n_recv * 16 * passes)
    achieved = sc_bytes / (sc_ms / 1e3) / 1e9 if sc_ms > 0 else None
    peak = 6548.2
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                               "MEASURED_PEAKS.json")) as fh:
            peak = json.load(fh).get("hbm_gbs", peak)
    except OSError:
        pass
    roof = {"bound": "hbm", "kernel": "seg::k_scatter (radix scatter pass), rank 0", "achieved": achieved,
            "peak": peak, "unit": "GB/s", "frac": (achieved / peak) if achieved else None, "traffic": None,
            "launches": sc_n, "merge_ms_per_step_rank0": mg_ms / args.steps}

    # end to end: every rank's shard from pinned host memory through the same
    # call, when the host has the RAM for all ranks' shards
    e2e = None
    need = 16 * (r.cardinality + s.cardinality) * int(os.environ.get("LOCAL_WORLD_SIZE", G))
    try:
        import psutil

        room = psutil.virtual_memory().available > 1.5 * need
    except ImportError:
        room = False
    if not getattr(args, "no_e2e", False) and room:
        def pinned(t):  # device -> pinned host directly (no pageable copy: N ranks share the host RAM)
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            h.copy_(t)
            return h

        rh = Relation(pinned(r.keys), pinned(r.payloads))
        sh = Relation(pinned(s.keys), pinned(s.payloads))
        k = max(1, min(args.steps, getattr(args, "e2e_steps", 3)))
        run_join_distributed(rh, sh, cfg, backend=be)
        _lib.load().mpsm_upload_bytes(1)
        dist.barrier()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(k):
            res_e = run_join_distributed(rh, sh, cfg, backend=be)
        e1.record()
        torch.cuda.synchronize()
        e_ms = torch.tensor([e0.elapsed_time(e1) / k], device="cuda")
        dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        up = torch.tensor([int(_lib.load().mpsm_upload_bytes(1)) // k], dtype=torch.int64, device="cuda")
        dist.all_reduce(up, op=dist.ReduceOp.SUM)
        e_ms = float(e_ms.item())
        up = int(up.item())
        e2e = {"value": (n_r + n_s) / (e_ms / 1e3), "unit": "tuples/s", "ms_per_step": e_ms, "steps": k,
               "h2d_bytes_per_step": up + 16 * (n_r if up else n_r + n_s),
               "d2h_bytes_per_step": 8 * _lib.PAIR_FIELDS * G * G,
               "result_ok": (res_e.match_count, res_e.aggregate_max, res_e.checksum) == got,
               "input_path": "pinned host shards; public side as packed 8-B records (CudaBackend.upload), "
                             "private side as columns"}
        del rh, sh
    elif not room:
        e2e = {"value": None, "skipped": f"host RAM below 1.5 x the {need / 1e9:.0f} GB of pinned shards"}
    if me == 0:
        line = {
            "metric": metric, "value": (n_r + n_s) / (ms / 1e3), "unit": "tuples/s", "n_gpus": G,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (counter-based generators on device, seed 0)",
            "config": dist_workload(name, G)[0],
            "engine": {"impl": "paper_1207_0145_b200.distributed (NCCL all-to-all of R, NVLink peer reads of "
                               "S runs)", "threads": G, "parallelism": f"dp{G}"},
            "result": {"match_count": got[0], "aggregate_max": got[1], "checksum": hex(got[2]),
                       "expected": [want[0], want[1], hex(want[2])],
                       "verified_by": "sharded torch checker (tests/torch_check.py)", "matches": got == want,
                       "timed_steps_match": timed_ok},
            "gpu_launches": launches, "clocks": clk, "e2e": e2e, "roofline": roof, "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    ipc_close_all()
    dist.destroy_process_group()
