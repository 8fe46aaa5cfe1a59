"""Independent plain-PyTorch checker of the three join outputs at full size.

Test infrastructure, not product code: the CPU oracle (oracle/) cannot join
billions of tuples in test time, so at BASELINE.json's full sizes the GPU
join is checked against COUNT, MAX(r.payload + s.payload) and the splitmix64
checksum of SURVEY.md 8(a) a13 computed here with torch gathers / sorts /
searchsorted on the same device -- none of this package's kernels.
``tests/test_gpu_fullsize.py::test_torch_checksum_matches_the_oracle_definition``
pins this restatement to the CPU oracle on small inputs.

* ``fk_join``: R keys unique (a permutation, BASELINE configs 1-3, 5), so the
  match of every S tuple is lookup[s.key] (the oracle's FK gather).
* ``general_join``: duplicates on both sides (config 4): R sorted by
  torch.sort, every S tuple's equal-key R range by searchsorted, the pairs
  enumerated with repeat_interleave.
"""

from __future__ import annotations

import torch

M64 = (1 << 64) - 1


def _s64(c: int) -> int:
    return c - (1 << 64) if c >= 1 << 63 else c


C0, C1, C2 = _s64(0x9E3779B97F4A7C15), _s64(0xBF58476D1CE4E5B9), _s64(0x94D049BB133111EB)


def _lsr(z, k):
    """logical right shift of int64 tensors"""
    return torch.bitwise_and(torch.bitwise_right_shift(z, k), (1 << (64 - k)) - 1)


def pair_hash(rp, sp):
    """splitmix64(r ^ rotl64(s, 17)) in wrapping int64 arithmetic"""
    x = torch.bitwise_xor(rp, torch.bitwise_or(torch.bitwise_left_shift(sp, 17), _lsr(sp, 47)))
    z = x + C0
    z = torch.bitwise_xor(z, _lsr(z, 30)) * C1
    z = torch.bitwise_xor(z, _lsr(z, 27)) * C2
    return torch.bitwise_xor(z, _lsr(z, 31))


class Acc:
    """(count, max, checksum) accumulated over pair batches; payloads < 2^32"""

    def __init__(self):
        self.count, self.best, self.csum = 0, None, 0

    def add(self, rp, sp):
        if rp.numel() == 0:
            return
        self.count += int(rp.numel())
        b = int((rp + sp).max().item())  # payloads < 2^32: the sum fits int64
        self.best = b if self.best is None or b > self.best else self.best
        self.csum = (self.csum + int(pair_hash(rp, sp).sum().item())) & M64

    def result(self):
        return self.count, self.best, self.csum


def fk_lookup(r_keys, r_pays):
    """lookup[key] = payload of the (unique) R tuple with that key"""
    rk, rp = r_keys.view(torch.int64), r_pays.view(torch.int64)
    lookup = torch.zeros(int(rk.max().item()) + 1, dtype=torch.int64, device=rk.device)
    lookup[rk] = rp
    return lookup


def fk_add(acc: Acc, lookup, s_keys, s_pays, chunk: int = 1 << 28) -> None:
    sk, sp = s_keys.view(torch.int64), s_pays.view(torch.int64)
    for a in range(0, sk.numel(), chunk):
        acc.add(lookup[sk[a:a + chunk]], sp[a:a + chunk])


def fk_join(r, s, chunk: int = 1 << 28):
    """FK join (R keys unique, every S key present): -> (count, max, checksum)"""
    lookup = fk_lookup(r.keys, r.payloads)
    acc = Acc()
    fk_add(acc, lookup, s.keys, s.payloads, chunk)
    return acc.result()


def _general_add(acc: Acc, r_keys, r_pays, s, chunk: int) -> None:
    """every (R, S) pair with equal keys into acc: R sorted by torch.sort,
    each S tuple's equal-key R range by searchsorted, the pairs enumerated
    with repeat_interleave"""
    dev = r_keys.device
    rk, order = torch.sort(r_keys.view(torch.int64))
    rp = r_pays.view(torch.int64)[order]
    del order
    sk_all, sp_all = s.keys.view(torch.int64), s.payloads.view(torch.int64)
    for a in range(0, sk_all.numel(), chunk):
        sk, sp = sk_all[a:a + chunk], sp_all[a:a + chunk]
        lo = torch.searchsorted(rk, sk, right=False)
        cnt = torch.searchsorted(rk, sk, right=True) - lo
        hit = cnt > 0
        lo, cnt, spm = lo[hit], cnt[hit], sp[hit]
        if cnt.numel() == 0:
            continue
        total = int(cnt.sum().item())
        start = torch.cumsum(cnt, 0) - cnt  # first pair of each S tuple
        s_of = torch.repeat_interleave(torch.arange(cnt.numel(), device=dev), cnt, output_size=total)
        r_idx = lo[s_of] + (torch.arange(total, device=dev) - start[s_of])
        acc.add(rp[r_idx], spm[s_of])


def general_join(r, s, chunk: int = 1 << 27):
    """general equi-join (duplicates on both sides) by sort + searchsorted"""
    acc = Acc()
    _general_add(acc, r.keys, r.payloads, s, chunk)
    return acc.result()


# ------------------------------------------------ sharded (torch.distributed)
def _reduce(acc: Acc, group, device):
    """(count, max, checksum) over the ranks: sum / max / sum mod 2^64"""
    import torch.distributed as dist

    cs = acc.csum - (1 << 64) if acc.csum >= 1 << 63 else acc.csum
    t = torch.tensor([acc.count, cs], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    b = torch.tensor([-1 if acc.best is None else acc.best], dtype=torch.int64, device=device)
    dist.all_reduce(b, op=dist.ReduceOp.MAX, group=group)
    count, best = int(t[0].item()), int(b[0].item())
    return count, (None if best < 0 else best), int(t[1].item()) & M64


def _gather_padded(x, group, chunk: int):
    """all_gather of this rank's x[c:c+chunk] for every chunk c, padded with
    zeros (yields the gathered chunk tensors, [G * chunk] each)"""
    import torch.distributed as dist

    G = dist.get_world_size(group)
    n = torch.tensor([x.numel()], dtype=torch.int64, device=x.device)
    sizes = [torch.empty_like(n) for _ in range(G)]
    dist.all_gather(sizes, n, group=group)
    top = max(int(v.item()) for v in sizes)
    for c in range(0, top, chunk):
        piece = torch.zeros(chunk, dtype=torch.int64, device=x.device)
        part = x.view(torch.int64)[c:c + chunk]
        piece[:part.numel()] = part
        outs = [torch.empty_like(piece) for _ in range(G)]
        dist.all_gather(outs, piece, group=group)
        yield outs, [max(0, min(chunk, int(v.item()) - c)) for v in sizes]


def fk_join_dist(r, s, n_r: int, group=None, chunk: int = 1 << 26):
    """FK join over position shards (every rank holds one R and one S shard):
    the full lookup is rebuilt on every rank from gathered R chunks, each rank
    gathers its S shard, the partials are reduced."""
    dev = r.keys.device
    lookup = torch.zeros(n_r + 1, dtype=torch.int64, device=dev)
    for (ks, ns), (ps, _) in zip(_gather_padded(r.keys, group, chunk), _gather_padded(r.payloads, group, chunk)):
        for k, p, m in zip(ks, ps, ns):
            lookup[k[:m]] = p[:m]
    acc = Acc()
    fk_add(acc, lookup, s.keys, s.payloads)
    del lookup
    return _reduce(acc, group, dev)


def general_join_dist(r, s, group=None, chunk: int = 1 << 26):
    """general equi-join over position shards: every rank gathers all of R,
    joins its S shard against it, the partials are reduced."""
    ks, ps = [], []
    for (kc, ns), (pc, _) in zip(_gather_padded(r.keys, group, chunk), _gather_padded(r.payloads, group, chunk)):
        for k, p, m in zip(kc, pc, ns):
            ks.append(k[:m].clone())
            ps.append(p[:m].clone())
    rk, rp = torch.cat(ks), torch.cat(ps)
    del ks, ps
    acc = Acc()
    _general_add(acc, rk, rp, s, chunk)
    return _reduce(acc, group, r.keys.device)
