"""CPU backend for the distributed join protocol -- TEST INFRASTRUCTURE.

Implements paper_1207_0145_b200.distributed's backend interface with the CPU
oracle (oracle/), so tests/test_distributed.py can run the multi-rank host
protocol (gathers, splitters, all-to-all, folding) under gloo on CPU.  The
product never uses it; its device work is CudaBackend.
"""

import numpy as np
import torch

from oracle import oracle as orc
from paper_1207_0145_b200 import _lib


class OracleBackend:
    comm_device = torch.device("cpu")

    def __init__(self, packed=None):
        pass

    def unpacked(self):
        return self

    def setup(self, dom):
        self.dom = dom
        self.bad = -1

    def _flag(self, idx):
        if idx >= 0 and (self.bad == -1 or idx < self.bad):
            self.bad = idx

    def to_device(self, a):
        if isinstance(a, torch.Tensor):
            return a.cpu()
        return torch.from_numpy(np.ascontiguousarray(a, np.uint64).copy())

    def sort(self, k, p, public=False):
        kk = k.numpy().copy()
        pp = p.numpy().copy()
        if orc.three_phase_sort(kk, pp, self.dom.lower, self.dom.width_bits) < 0:
            self._flag(0)
        return (torch.from_numpy(kk), torch.from_numpy(pp))

    def histogram(self, keys, shift, nb):
        c = np.zeros(nb, np.int64)
        kk = np.ascontiguousarray(keys.numpy())
        if kk.shape[0]:
            self._flag(orc.radix_histogram(kk, self.dom.lower, shift, c))
        return c

    def bound_keys(self, run, f, t):
        keys = run[0].numpy()
        return orc.local_equiheight_bounds(keys, f, t)[0]

    def partition(self, k, p, shift, sp, npart, starts):
        kk, pp = np.ascontiguousarray(k.numpy()), np.ascontiguousarray(p.numpy())
        n = kk.shape[0]
        out_k, out_p = np.empty(n, np.uint64), np.empty(n, np.uint64)
        if n:
            buckets = ((kk - np.uint64(self.dom.lower)) >> np.uint64(shift)).astype(np.int64)
            cnt = np.bincount(sp[np.minimum(buckets, sp.shape[0] - 1)], minlength=npart)
            cur = starts.astype(np.int64).copy()
            ends = cur + cnt
            orc.scatter_chunk(kk, pp, self.dom.lower, shift, sp.astype(np.int64), cur, ends, out_k, out_p)
        return torch.from_numpy(out_k), torch.from_numpy(out_p)

    def bad_index(self):
        return self.bad

    def overflowed(self):
        return False

    def share(self, run):
        return (run[0].numpy().copy(), run[1].numpy().copy())

    def open(self, shared, peer=-1):
        return (torch.from_numpy(shared[0]), torch.from_numpy(shared[1]))

    def join(self, priv_runs, pub_runs, swap, mode, out=None, cap=0):
        rec = np.zeros((len(priv_runs) * len(pub_runs), _lib.PAIR_FIELDS), np.uint64)
        for i, (rk, rp) in enumerate(priv_runs):
            rk, rp = rk.numpy(), rp.numpy()
            for j, (sk, sp) in enumerate(pub_runs):
                sk, sp = sk.numpy(), sp.numpy()
                row = rec[i * len(pub_runs) + j]
                if rk.shape[0] == 0 or sk.shape[0] == 0:
                    continue
                start, probes = orc.interp_lower_bound(sk, int(rk[0]))
                c, b, ex, _, cs = orc.merge_join_run(rk, rp, sk, sp, start, swap=swap)
                row[_lib.PAIR_COUNT] = c
                row[_lib.PAIR_BEST] = b
                row[_lib.PAIR_CHECKSUM] = cs
                row[_lib.PAIR_START] = start
                row[_lib.PAIR_PROBES] = probes
                row[_lib.PAIR_EXAMINED] = ex
        return rec

    def materialize(self, priv_runs, pub_runs, swap, total):
        pieces = []
        for rk, rp in priv_runs:
            for sk, sp in pub_runs:
                a, b, c, d = rk.numpy(), rp.numpy(), sk.numpy(), sp.numpy()
                if a.shape[0] == 0 or c.shape[0] == 0:
                    continue
                start, _ = orc.interp_lower_bound(c, int(a[0]))
                o_r = np.empty(max(total, 1), np.uint64)
                o_s = np.empty(max(total, 1), np.uint64)
                cnt, _, _, em, _ = orc.merge_join_run(a, b, c, d, start, True, o_r, o_s, swap)
                pieces.append(np.stack([o_r[:em], o_s[:em]], axis=1))
        return np.concatenate(pieces, axis=0) if pieces else np.empty((0, 2), np.uint64)

    def records(self, rec):
        return rec

    def sync(self):
        pass
