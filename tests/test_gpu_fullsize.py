"""Parity at BASELINE.json's full sizes (opt-in: MPSM_FULLSIZE=1; minutes and up
to ~120 GB of HBM).

The CPU oracle cannot join billions of tuples in test time, so at full size
the GPU join is checked against an independent plain-PyTorch computation of
the same three outputs on the same device (COUNT, MAX(r.payload + s.payload)
and the splitmix64 checksum of SURVEY.md 8(a) a13), written with torch
gathers / sorts / searchsorted -- none of this package's kernels:

* FK configs (2 and 3 at multiplicity 16): R keys are a permutation, so the
  match of every S tuple is lookup[s.key] (the oracle's FK gather, done on the
  GPU); cfg2 also against the committed golden (the reference's count/max).
* config 4 (negatively correlated skew, duplicates on both sides): R sorted by
  torch.sort, every S tuple's equal-key R range by searchsorted, the pairs
  enumerated with repeat_interleave.

``tools/fullsize_parity.sh`` runs this module on the GPU box; its log is kept
under profiles/.
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - collected on CPU boxes too
    pytest.skip("needs a CUDA device", allow_module_level=True)
if os.environ.get("MPSM_FULLSIZE") != "1":
    pytest.skip("full BASELINE sizes: set MPSM_FULLSIZE=1 (minutes, up to ~120 GB of HBM)", allow_module_level=True)

import paper_1207_0145_b200 as P  # noqa: E402
from paper_1207_0145_b200 import datagen  # noqa: E402
from paper_1207_0145_b200.core import JoinConfig, KeyDomain, Relation  # noqa: E402

DEV = torch.device("cuda", 0)
M64 = (1 << 64) - 1


def _s64(c: int) -> int:
    return c - (1 << 64) if c >= 1 << 63 else c


C0, C1, C2 = _s64(0x9E3779B97F4A7C15), _s64(0xBF58476D1CE4E5B9), _s64(0x94D049BB133111EB)


def _lsr(z, k):
    """logical right shift of int64 tensors"""
    return torch.bitwise_and(torch.bitwise_right_shift(z, k), (1 << (64 - k)) - 1)


def _pair_hash(rp, sp):
    """splitmix64(r ^ rotl64(s, 17)) in wrapping int64 arithmetic"""
    x = torch.bitwise_xor(rp, torch.bitwise_or(torch.bitwise_left_shift(sp, 17), _lsr(sp, 47)))
    z = x + C0
    z = torch.bitwise_xor(z, _lsr(z, 30)) * C1
    z = torch.bitwise_xor(z, _lsr(z, 27)) * C2
    return torch.bitwise_xor(z, _lsr(z, 31))


class _Acc:
    def __init__(self):
        self.count, self.best, self.csum = 0, None, 0

    def add(self, rp, sp):
        if rp.numel() == 0:
            return
        self.count += int(rp.numel())
        b = int((rp + sp).max().item())  # payloads < 2^32: the sum fits int64
        self.best = b if self.best is None or b > self.best else self.best
        self.csum = (self.csum + int(_pair_hash(rp, sp).sum().item())) & M64

    def result(self):
        return self.count, self.best, self.csum


def _torch_fk(r, s, chunk=1 << 28):
    rk, rp = r.keys.view(torch.int64), r.payloads.view(torch.int64)
    lookup = torch.zeros(int(rk.max().item()) + 1, dtype=torch.int64, device=DEV)
    lookup[rk] = rp
    acc = _Acc()
    sk, sp = s.keys.view(torch.int64), s.payloads.view(torch.int64)
    for a in range(0, sk.numel(), chunk):
        acc.add(lookup[sk[a:a + chunk]], sp[a:a + chunk])
    return acc.result()


def _torch_join(r, s, chunk=1 << 27):
    """general equi-join (duplicates on both sides) by sort + searchsorted"""
    rk, order = torch.sort(r.keys.view(torch.int64))
    rp = r.payloads.view(torch.int64)[order]
    del order
    acc = _Acc()
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
        s_of = torch.repeat_interleave(torch.arange(cnt.numel(), device=DEV), cnt, output_size=total)
        r_idx = lo[s_of] + (torch.arange(total, device=DEV) - start[s_of])
        acc.add(rp[r_idx], spm[s_of])
    return acc.result()


def _ours(r, s, dom):
    res = P.run_join(r, s, JoinConfig(threads=1, algorithm="p-mpsm", key_domain=dom))
    out = (res.match_count, res.aggregate_max, res.checksum)
    torch.cuda.empty_cache()
    return out


def _to_dev(rel):
    return Relation(torch.from_numpy(rel.keys).to(DEV), torch.from_numpy(rel.payloads).to(DEV))


def test_cfg2_full_size_vs_torch_and_golden():
    r, s, dom = datagen.gen_fk(100_000_000, 400_000_000, 0)
    rd, sd = _to_dev(r), _to_dev(s)
    del r, s
    ours = _ours(rd, sd, dom)
    assert ours == (400_000_000, 8_589_753_492, 0xAA48801BE88FA31B)  # tests/golden/golden.json cfg2
    assert ours == _torch_fk(rd, sd)


def test_cfg3_multiplicity16_full_size_vs_torch():
    # |R| = 200M, |S| = 3.2B (54 GB of input); counter-based generator on the device
    r, s, dom = datagen.gen_fk_device(200_000_000, 3_200_000_000, seed=3, device=DEV)
    ours = _ours(r, s, dom)
    want = _torch_fk(r, s)
    assert want[0] == 3_200_000_000
    assert ours == want


def test_cfg4_negcorr_skew_full_size_vs_torch():
    dom = KeyDomain(1, 1 << 32)
    r, s = datagen.gen_negcorr(400_000_000, 1_600_000_000, dom, 0)
    rd, sd = _to_dev(r), _to_dev(s)
    del r, s
    ours = _ours(rd, sd, dom)
    want = _torch_join(rd, sd)
    # E[matches] = 0.35 |R||S| / (0.8 (2^32 - 1)) ~ 6.52e7
    assert 6.0e7 < want[0] < 7.0e7
    assert ours == want


def test_torch_checksum_matches_the_oracle_definition():
    """the torch restatement of the checksum equals the CPU oracle's on small inputs"""
    from oracle import oracle as orc

    rng = np.random.default_rng(7)
    n = 10_000
    rk = (rng.permutation(n) + 1).astype(np.uint64)
    rp = rng.integers(0, 1 << 32, n, dtype=np.uint64)
    sk = rng.integers(1, n + 1, 4 * n, dtype=np.uint64)
    sp = rng.integers(0, 1 << 32, 4 * n, dtype=np.uint64)
    want = orc.join(rk, rp, sk, sp, threads=1, lower=1, upper=n + 1)
    r = Relation(torch.from_numpy(rk).to(DEV), torch.from_numpy(rp).to(DEV))
    s = Relation(torch.from_numpy(sk).to(DEV), torch.from_numpy(sp).to(DEV))
    assert _torch_fk(r, s) == (want.match_count, want.aggregate_max, want.checksum)
    assert _torch_join(r, s) == (want.match_count, want.aggregate_max, want.checksum)
