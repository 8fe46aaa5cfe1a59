"""Parity at BASELINE.json's full sizes, every config (part of ``-m gpu``).

The CPU oracle cannot join billions of tuples in test time, so at full size
the GPU join is checked against the independent plain-PyTorch computation of
the same three outputs in tests/torch_check.py (COUNT, MAX(r.payload +
s.payload), the splitmix64 checksum of SURVEY.md 8(a) a13 -- torch gathers /
sorts / searchsorted, none of this package's kernels), itself pinned to the
CPU oracle by ``test_torch_checksum_matches_the_oracle_definition``:

* config 2 (100M x 400M FK, numpy PCG64 seed 0): also the committed golden
  (the reference's own count / max);
* config 3 (|R| = 200M, |S| = 1x, 4x, 8x, 16x |R|, up to 3.4G tuples / 54 GB):
  the counter-based FK generator on the device;
* config 4 (400M x 1.6B, negatively correlated 80-20 skew, 32-bit keys,
  duplicates on both sides; numpy generator of the reference's datagen);
* config 5 (1.6B x 6.4B FK, 8G tuples): its 16-B columns (128 GB) plus runs
  do not fit one B200, so the relations are generated chunk by chunk
  straight into packed 8-B records (PackedRelation, 64 GB) and joined on one
  GPU; the checker sees the same chunks.  The multi-GPU engine runs this
  config sharded over 2-8 GPUs (distributed.py); the join result does not
  depend on the GPU count.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - collected on CPU boxes too
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1207_0145_b200 as P  # noqa: E402
from paper_1207_0145_b200 import datagen  # noqa: E402
from paper_1207_0145_b200 import device as D  # noqa: E402
from paper_1207_0145_b200.core import JoinConfig, KeyDomain, PackedRelation, Relation  # noqa: E402
from tests import torch_check as tc  # noqa: E402

DEV = torch.device("cuda", 0)


@pytest.fixture(autouse=True)
def _free_hbm():
    torch.cuda.empty_cache()
    yield
    torch.cuda.empty_cache()


def _ours(r, s, dom, threads=1):
    res = P.run_join(r, s, JoinConfig(threads=threads, algorithm="p-mpsm", key_domain=dom))
    return res.match_count, res.aggregate_max, res.checksum


def _to_dev(rel):
    return Relation(torch.from_numpy(rel.keys).to(DEV), torch.from_numpy(rel.payloads).to(DEV))


def test_cfg2_full_size_vs_torch_and_golden():
    r, s, dom = datagen.gen_fk(100_000_000, 400_000_000, 0)
    rd, sd = _to_dev(r), _to_dev(s)
    del r, s
    ours = _ours(rd, sd, dom)
    assert ours == (400_000_000, 8_589_753_492, 0xAA48801BE88FA31B)  # tests/golden/golden.json cfg2
    assert ours == tc.fk_join(rd, sd)


@pytest.mark.parametrize("mult", [1, 4, 8, 16])
def test_cfg3_multiplicity_full_size_vs_torch(mult):
    # |R| = 200M, |S| = mult x |R| (16: 3.2B, 54 GB of input); counter-based generator on the device
    n_r = 200_000_000
    r, s, dom = datagen.gen_fk_device(n_r, mult * n_r, seed=3, device=DEV)
    ours = _ours(r, s, dom)
    want = tc.fk_join(r, s)
    assert want[0] == mult * n_r
    assert ours == want


def test_cfg4_negcorr_skew_full_size_vs_torch():
    dom = KeyDomain(1, 1 << 32)
    r, s = datagen.gen_negcorr(400_000_000, 1_600_000_000, dom, 0)
    rd, sd = _to_dev(r), _to_dev(s)
    del r, s
    ours = _ours(rd, sd, dom)
    want = tc.general_join(rd, sd)
    # E[matches] = 0.35 |R||S| / (0.8 (2^32 - 1)) ~ 6.52e7
    assert 6.0e7 < want[0] < 7.0e7
    assert ours == want


def _packed_fk(n_r, n_s, seed, chunk=1 << 28):
    """cfg5-sized FK relations generated chunk-wise into packed records, with
    the torch checker fed the same chunks: -> (R, S PackedRelations, dom, want)"""
    dom = KeyDomain(1, n_r + 1)
    w = dom.width_bits
    span_m1 = dom.upper - dom.lower - 1
    bad = D.new_bad_flag(DEV)
    ovf = torch.zeros(1, dtype=torch.int32, device=DEV)
    r_rec = torch.empty(n_r, dtype=torch.uint64, device=DEV)
    lookup = torch.zeros(n_r + 1, dtype=torch.int64, device=DEV)
    for a in range(0, n_r, chunk):
        b = min(n_r, a + chunk)
        r, _ = datagen.fk_range_device(n_r, n_s, (a, b), (0, 0), seed, DEV)
        lookup[r.keys.view(torch.int64)] = r.payloads.view(torch.int64)
        D.pack_records(r.keys, r.payloads, dom.lower, span_m1, w, r_rec[a:b], bad, ovf)
        del r
    s_rec = torch.empty(n_s, dtype=torch.uint64, device=DEV)
    acc = tc.Acc()
    for a in range(0, n_s, chunk):
        b = min(n_s, a + chunk)
        _, s = datagen.fk_range_device(n_r, n_s, (0, 0), (a, b), seed, DEV)
        tc.fk_add(acc, lookup, s.keys, s.payloads)
        D.pack_records(s.keys, s.payloads, dom.lower, span_m1, w, s_rec[a:b], bad, ovf)
        del s
    del lookup
    assert int(bad.item()) == -1 and int(ovf.item()) == 0
    return PackedRelation(r_rec, dom), PackedRelation(s_rec, dom), dom, acc.result()


def test_cfg5_full_size_one_gpu_packed_vs_torch():
    # BASELINE configs[4]: |R| = 1.6B, |S| = 6.4B (8G tuples); 64 GB of packed records
    r, s, dom, want = _packed_fk(1_600_000_000, 6_400_000_000, seed=5)
    assert want[0] == 6_400_000_000
    ours = _ours(r, s, dom)
    assert ours == want


def test_packed_relation_matches_columns():
    """PackedRelation inputs give the column path's results and statistics
    (T = 1 and T = 3, both engines)"""
    r, s, dom, want = _packed_fk(3_000_000, 12_000_000, seed=9, chunk=1 << 20)
    pw = 64 - dom.width_bits

    def unpack(rec):
        v = rec.view(torch.int64)
        return Relation((tc._lsr(v, pw) + dom.lower).view(torch.uint64), (v & ((1 << pw) - 1)).view(torch.uint64))

    cols = (unpack(r.records), unpack(s.records))
    for algo in ("p-mpsm", "b-mpsm"):
        for t in (1, 3):
            cfg = JoinConfig(threads=t, algorithm=algo, key_domain=dom)
            a = P.run_join(*cols, cfg)
            pr = PackedRelation(r.records.clone(), dom)
            ps = PackedRelation(s.records.clone(), dom)
            b = P.run_join(pr, ps, cfg)
            assert (a.match_count, a.aggregate_max, a.checksum) == want
            assert (b.match_count, b.aggregate_max, b.checksum) == want
            def stats(res):
                return [{k: v for k, v in vars(x).items() if not k.endswith("_seconds")} for x in res.worker_stats]

            assert stats(a) == stats(b)


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
    assert tc.fk_join(r, s) == (want.match_count, want.aggregate_max, want.checksum)
    assert tc.general_join(r, s) == (want.match_count, want.aggregate_max, want.checksum)
