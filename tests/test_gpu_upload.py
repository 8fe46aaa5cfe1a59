"""The packed upload path (host threads pack (key, payload) columns into 8-B
records while earlier chunks copy; mpsm_upload_records) and the record sort
(mpsm_sort_records), checked against numpy."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CHUNK = 1 << 20


def _pack_np(k, p, lower, w):
    return ((k - np.uint64(lower)) << np.uint64(64 - w)) | p


@pytest.mark.parametrize("n", [1, 7, CHUNK - 1, CHUNK, CHUNK + 1, 3 * CHUNK + 5, 40 * CHUNK + 3])
def test_upload_matches_numpy(n):
    import torch

    from paper_1207_0145_b200 import device as D

    rng = np.random.default_rng(n)
    w, lower = 27, 5
    k = rng.integers(lower, lower + (1 << w), n, dtype=np.uint64)
    p = rng.integers(0, 1 << 32, n, dtype=np.uint64)
    if n > CHUNK:  # pinned columns: every 4th chunk is packed by the GPU from mapped host memory
        kt, pt = torch.from_numpy(k).pin_memory(), torch.from_numpy(p).pin_memory()
    else:
        kt, pt = torch.from_numpy(k), p
    rec = torch.empty(n, dtype=torch.uint64, device="cuda")
    bad, ovf = D.upload_records(kt, pt, lower, (1 << w) - 1, w, rec)
    assert bad == -1 and not ovf
    assert np.array_equal(rec.cpu().numpy(), _pack_np(k, p, lower, w))


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("where", [5, 2 * CHUNK + 9, 3 * CHUNK + 2, 7 * CHUNK + 1])
def test_upload_reports_domain_and_overflow(pinned, where):
    """host-packed chunks and (pinned input) GPU-packed chunks report the
    first out-of-domain index and payload overflow alike"""
    import torch

    from paper_1207_0145_b200 import device as D

    n = 8 * CHUNK + 11
    w = 20
    k = torch.full((n,), 3, dtype=torch.int64)
    p = torch.zeros(n, dtype=torch.int64)
    if pinned:
        k, p = k.pin_memory(), p.pin_memory()
    k[where] = 1 << 21  # out of [0, 2^20)
    k[n - 1] = 1 << 22
    rec = torch.empty(n, dtype=torch.uint64, device="cuda")
    bad, ovf = D.upload_records(k, p, 0, (1 << w) - 1, w, rec)
    assert bad == where and not ovf
    k.fill_(3)
    p[where] = 1 << (64 - w)  # one payload too wide
    bad, ovf = D.upload_records(k, p, 0, (1 << w) - 1, w, rec)
    assert bad == -1 and ovf


@pytest.mark.parametrize("n,w", [(1, 9), (4095, 27), (8193, 27), (1_000_003, 20), (3_000_001, 33)])
def test_sort_records_matches_numpy(n, w):
    import torch

    from paper_1207_0145_b200 import device as D

    rng = np.random.default_rng(w + n)
    rec = rng.integers(0, np.iinfo(np.uint64).max, n, dtype=np.uint64, endpoint=True)
    d_in = torch.from_numpy(rec).cuda()
    out = torch.empty_like(d_in)
    tmp = torch.empty_like(d_in)
    D.sort_records(d_in, w, out, tmp)
    got = out.cpu().numpy()
    keys = rec >> np.uint64(64 - w)
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(got >> np.uint64(64 - w), keys[order])
    assert np.array_equal(got, rec[order])  # the sort is stable


def test_join_host_inputs_all_paths(monkeypatch):
    """numpy inputs through host packing, device packing and pairs agree;
    a too-wide payload falls back to pairs; an out-of-domain key raises."""
    import paper_1207_0145_b200 as P
    from paper_1207_0145_b200 import engine
    from paper_1207_0145_b200.core import DomainError

    r, s, dom = P.gen_fk(300_000, 1_200_000, seed=9)
    outs = []
    for pack, host in ((True, True), (True, False), (False, False)):
        monkeypatch.setattr(engine, "PACK_RECORDS", pack)
        monkeypatch.setattr(engine, "HOST_PACK", host)
        for t in (1, 4):
            for algo in ("p-mpsm", "b-mpsm"):
                res = P.run_join(r, s, P.JoinConfig(threads=t, algorithm=algo, key_domain=dom))
                outs.append((res.match_count, res.aggregate_max, res.checksum,
                             [w.public_tuples_examined for w in res.worker_stats]))
    for i in range(4):  # the same (T, algorithm) through the three paths
        assert outs[i] == outs[i + 4] == outs[i + 8], i
    assert outs[0][0] == 1_200_000
    monkeypatch.setattr(engine, "PACK_RECORDS", True)
    monkeypatch.setattr(engine, "HOST_PACK", True)
    wide = P.Relation(np.asarray(s.keys), np.asarray(s.payloads) | np.uint64(1 << 40))
    a = P.run_join(r, wide, P.JoinConfig(threads=1, key_domain=dom))
    monkeypatch.setattr(engine, "PACK_RECORDS", False)
    b = P.run_join(r, wide, P.JoinConfig(threads=1, key_domain=dom))
    assert (a.match_count, a.aggregate_max, a.checksum) == (b.match_count, b.aggregate_max, b.checksum)
    monkeypatch.setattr(engine, "PACK_RECORDS", True)
    badk = np.asarray(s.keys).copy()
    badk[12345] = dom.upper + 7
    with pytest.raises(DomainError, match="12345"):
        P.run_join(r, P.Relation(badk, np.asarray(s.payloads)), P.JoinConfig(threads=1, key_domain=dom))


@pytest.mark.parametrize("n", [8191, 8192, 8193, 2 * 8192 + 1, 5 * 8192 - 3, 123_457])
@pytest.mark.parametrize("w", [10, 18, 27])
def test_sort_packed_tile_edges(n, w):
    """the packing pass (4096-tuple tiles) and record passes (8192-tuple
    tiles) at tile-boundary sizes; stable"""
    import torch

    from paper_1207_0145_b200 import device as D

    rng = np.random.default_rng(n + 7 * w)
    lower = 3
    k = rng.integers(lower, lower + (1 << w), n, dtype=np.uint64)
    p = np.arange(n, dtype=np.uint64)
    dk, dp = torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda()
    out = torch.empty_like(dk)
    tmp = torch.empty_like(dk)
    ovf = torch.zeros(1, dtype=torch.int32, device="cuda")
    D.sort_packed(dk, dp, lower, (1 << w) - 1, w, out, tmp, None, ovf)
    got = out.cpu().numpy()
    order = np.argsort(k, kind="stable")
    want = ((k[order] - np.uint64(lower)) << np.uint64(64 - w)) | p[order]
    assert int(ovf.item()) == 0
    assert np.array_equal(got, want)


def test_pack_records_and_partition_records_match_numpy():
    """mpsm_pack_records (device columns -> records) and
    mpsm_partition_records (records grouped by partition id, stable)."""
    import torch

    from paper_1207_0145_b200 import device as D

    rng = np.random.default_rng(77)
    n, w, lower = 1_000_003, 24, 9
    k = rng.integers(lower, lower + (1 << w), n, dtype=np.uint64)
    p = rng.integers(0, 1 << 32, n, dtype=np.uint64)
    dk, dp = torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda()
    bad = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    ovf = torch.zeros(1, dtype=torch.int32, device="cuda")
    rec = torch.empty_like(dk)
    D.pack_records(dk, dp, lower, (1 << w) - 1, w, rec, bad, ovf)
    want = _pack_np(k, p, lower, w)
    assert np.array_equal(rec.cpu().numpy(), want) and int(bad.item()) == -1 and int(ovf.item()) == 0
    # partition: 2^10 buckets of the top 10 key bits -> 5 partitions
    shift = w - 10
    cuts = np.sort(rng.choice(np.arange(1, 1 << 10), 4, replace=False))
    sp = np.searchsorted(cuts, np.arange(1 << 10), side="right").astype(np.int32)
    part = sp[((k - np.uint64(lower)) >> np.uint64(shift)).astype(np.int64)]
    out = torch.empty_like(dk)
    D.partition_records(dk, dp, lower, (1 << w) - 1, w, shift, torch.from_numpy(sp).cuda(), 5, out, bad, ovf)
    order = np.argsort(part, kind="stable")
    assert np.array_equal(out.cpu().numpy(), want[order])
