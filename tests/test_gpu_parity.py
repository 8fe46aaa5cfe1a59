"""GPU parity: the CUDA path (through the C ABI) vs the reference's golden
outputs and the CPU oracle on identical seeded inputs.  Integer results must
be bit-exact.  Run with ``pytest -m gpu`` on a B200."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - collected on CPU boxes too
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1207_0145_b200 as P  # noqa: E402
from paper_1207_0145_b200 import _lib  # noqa: E402
from paper_1207_0145_b200 import device as D  # noqa: E402
from paper_1207_0145_b200.core import DomainError, JoinConfig, KeyDomain, MaterializeCapExceeded, Relation  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from tests.golden_inputs import dataset, make_inputs, reference_totals  # noqa: E402

DEV = torch.device("cuda", 0)


def _cfg(case, **kw):
    d = dataset(case["dataset"])
    rk, rp, sk, sp, lo, up = make_inputs(d)
    cfg = JoinConfig(threads=case["threads"], algorithm=case["algorithm"], key_domain=KeyDomain(lo, up),
                     radix_bits=case["radix_bits"], query_mode=case["query_mode"], role_policy=case["role_policy"],
                     materialize_cap=1 << 26, **kw)
    return Relation(rk, rp), Relation(sk, sp), cfg


# --------------------------------------------------------------- engine parity

@pytest.fixture(params=["host", "device", "pairs"], ids=["packed-host", "packed-device", "pairs"])
def pack_mode(request, monkeypatch):
    """run with packed 8-B records packed on the host during the upload
    (default for host inputs), packed by the first sort pass on the device,
    and with (key, payload) pairs"""
    from paper_1207_0145_b200 import engine

    monkeypatch.setattr(engine, "PACK_RECORDS", request.param != "pairs")
    monkeypatch.setattr(engine, "HOST_PACK", request.param == "host")
    return request.param != "pairs"


def test_engine_cases_match_reference(golden, pack_mode):
    import warnings

    checked = 0
    for case in golden["engine_cases"]:
        r, s, cfg = _cfg(case)
        tag = (case["dataset"], case["algorithm"], case["threads"], case["query_mode"], case["role_policy"])
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            res = P.run_join(r, s, cfg)
        if "error" in case:
            # the reference fails on a float artifact in its CDF (skew.py:150);
            # we clamp the span and must return the T-independent totals
            count, mx, cs = reference_totals(case["dataset"])
            assert (res.match_count, res.checksum) == (count, cs), tag
            continue
        assert res.match_count == case["match_count"], tag
        assert res.aggregate_max == case["aggregate_max"], tag
        count, mx, cs = reference_totals(case["dataset"])
        assert res.checksum == cs, tag
        if case["query_mode"] == "materialize":
            assert res.materialized.shape == (case["match_count"], 2)
            assert orc.pairs_checksum(res.materialized[:, 0].copy(), res.materialized[:, 1].copy()) == case["checksum"]
        for got, want in zip(res.worker_stats, case["worker_stats"]):
            for k in ("tuples_sorted_public", "tuples_sorted_private", "tuples_scattered",
                      "public_tuples_examined", "probe_tuples_examined", "s_runs_with_matches"):
                assert getattr(got, k) == want[k], (tag, k, getattr(got, k), want[k])
        assert len(res.worker_stats) == case["threads"]
        checked += 1
    assert checked > 100


def test_materialized_multiset_matches_oracle(pack_mode):
    d = dataset("dup_heavy")
    rk, rp, sk, sp, lo, up = make_inputs(d)
    want = orc.join(rk, rp, sk, sp, threads=1, lower=lo, upper=up, query_mode="materialize", materialize_cap=1 << 24)
    for algo in ("b-mpsm", "p-mpsm"):
        for role in ("auto", "s-private"):
            res = P.run_join(Relation(rk, rp), Relation(sk, sp),
                             JoinConfig(threads=3, algorithm=algo, key_domain=KeyDomain(lo, up),
                                        query_mode="materialize", role_policy=role, materialize_cap=1 << 24))
            got = sorted(map(tuple, res.materialized.tolist()))
            assert got == sorted(map(tuple, want.materialized.tolist()))


def test_config1_golden(golden, pack_mode):
    g = golden["config1"]
    r, s, dom = P.gen_fk(g["n_r"], g["n_s"], g["seed"])
    for t in (1, 8):
        res = P.run_join(r, s, JoinConfig(threads=t, key_domain=dom))
        assert res.match_count == g["match_count"]
        assert res.aggregate_max == g["aggregate_max"]
        assert res.checksum == g["checksum"] == 0x7CDED1377072045D
        if t == 8:
            for got, want in zip(res.worker_stats, g["worker_stats"]):
                assert got.public_tuples_examined == want["public_tuples_examined"]
                assert got.probe_tuples_examined == want["probe_tuples_examined"]
                assert got.s_runs_with_matches == want["s_runs_with_matches"]
    # device-resident inputs take the same path without a host round trip
    rd = Relation(torch.from_numpy(r.keys).to(DEV), torch.from_numpy(r.payloads).to(DEV))
    sd = Relation(torch.from_numpy(s.keys).to(DEV), torch.from_numpy(s.payloads).to(DEV))
    res = P.run_join(rd, sd, JoinConfig(threads=1, key_domain=dom))
    assert (res.match_count, res.aggregate_max, res.checksum) == (g["match_count"], g["aggregate_max"], g["checksum"])


@pytest.mark.parametrize("n_r,n_s,seed", [(3_000_000, 12_000_000, 5), (10_000_000, 40_000_000, 0)])
def test_fk_vs_oracle_gather(n_r, n_s, seed):
    r, s, dom = P.gen_fk(n_r, n_s, seed)
    res = P.run_join(r, s, JoinConfig(threads=1, key_domain=dom))
    assert (res.match_count, res.aggregate_max, res.checksum) == orc.fk_gather(r.keys, r.payloads, s.keys,
                                                                              s.payloads, 1)


@pytest.mark.parametrize("threads,algorithm", [(2, "p-mpsm"), (16, "p-mpsm"), (64, "p-mpsm"), (100, "p-mpsm"),
                                                (7, "b-mpsm"), (64, "b-mpsm")])
def test_fk_many_workers_vs_oracle_gather(threads, algorithm):
    """T x T dense pairs through the streamed join (k_dense_flat up to 64 x 64
    = 4096 pairs; beyond 64 runs a side the merge walk), both variants"""
    r, s, dom = P.gen_fk(2_000_000, 8_000_000, 11)
    res = P.run_join(r, s, JoinConfig(threads=threads, algorithm=algorithm, key_domain=dom))
    assert (res.match_count, res.aggregate_max, res.checksum) == orc.fk_gather(r.keys, r.payloads, s.keys,
                                                                              s.payloads, 1)
    assert len(res.worker_stats) == threads


def test_negcorr_skew_vs_oracle(pack_mode):
    dom = KeyDomain(1, 1 << 32)
    r, s = P.gen_negcorr(400_000, 1_600_000, dom, seed=0)
    want = orc.join(r.keys, r.payloads, s.keys, s.payloads, threads=4, lower=dom.lower, upper=dom.upper,
                    parallel=True)
    for t in (1, 4):
        res = P.run_join(r, s, JoinConfig(threads=t, key_domain=dom))
        assert (res.match_count, res.aggregate_max, res.checksum) == (want.match_count, want.aggregate_max,
                                                                     want.checksum)


def test_heavy_duplicates_cross_product(pack_mode):
    # 200 x 200 pairs on one key plus a sprinkle of other keys
    rng = np.random.default_rng(3)
    rk = np.concatenate([np.full(200, 3, np.uint64), rng.integers(0, 8, 50, dtype=np.uint64)])
    sk = np.concatenate([np.full(200, 3, np.uint64), rng.integers(0, 8, 70, dtype=np.uint64)])
    rp = rng.integers(0, 1 << 32, rk.shape[0], dtype=np.uint64)
    sp = rng.integers(0, 1 << 32, sk.shape[0], dtype=np.uint64)
    want = orc.join(rk, rp, sk, sp, threads=1, lower=0, upper=8)
    for t in (1, 2, 5):
        res = P.run_pmpsm(Relation(rk, rp), Relation(sk, sp), JoinConfig(threads=t, key_domain=KeyDomain(0, 8)))
        assert (res.match_count, res.aggregate_max, res.checksum) == (want.match_count, want.aggregate_max,
                                                                     want.checksum)


def test_materialize_cap_and_domain_errors():
    keys = np.full(200, 3, np.uint64)
    rel = Relation(keys, keys.copy())
    with pytest.raises(MaterializeCapExceeded):
        P.run_pmpsm(rel, rel, JoinConfig(threads=1, key_domain=KeyDomain(0, 8), query_mode="materialize",
                                         materialize_cap=100))
    bad = Relation.from_tuples([(300, 1)])
    ok = Relation.from_tuples([(3, 1)])
    with pytest.raises(DomainError):
        P.run_pmpsm(bad, ok, JoinConfig(key_domain=KeyDomain(0, 256)))
    with pytest.raises(DomainError):
        P.run_bmpsm(ok, bad, JoinConfig(key_domain=KeyDomain(0, 256)))
    with pytest.raises(DomainError):
        P.run_pmpsm(bad, Relation(np.arange(10), np.arange(10)), JoinConfig(threads=2, key_domain=KeyDomain(0, 256)))


def test_role_swap_orientation():
    r = Relation.from_tuples([(1, 100), (2, 101), (3, 102), (2, 103)])
    s = Relation.from_tuples([(2, 900)])
    res = P.run_pmpsm(r, s, JoinConfig(threads=1, key_domain=KeyDomain(0, 8), query_mode="materialize"))
    assert sorted(map(tuple, res.materialized.tolist())) == [(101, 900), (103, 900)]
    assert res.checksum == (orc.pair_hash(101, 900) + orc.pair_hash(103, 900)) % (1 << 64)


def test_empty_and_tiny_inputs():
    dom = KeyDomain(0, 256)
    res = P.run_bmpsm(Relation.empty(), Relation(np.arange(50), np.arange(50)), JoinConfig(key_domain=dom))
    assert res.match_count == 0 and res.aggregate_max is None and res.checksum == 0
    rel = Relation.from_tuples([(1, 10), (1, 20)])
    res = P.run_pmpsm(rel, rel, JoinConfig(threads=8, key_domain=dom))
    assert res.match_count == 4 and res.aggregate_max == 40
    res = P.run_pmpsm(rel, rel, JoinConfig(threads=2, key_domain=dom, query_mode="count"))
    assert res.match_count == 4 and res.aggregate_max is None


def test_phase_hook_and_timings():
    calls = []
    r = Relation(np.arange(1000, dtype=np.uint64) % 512, np.arange(1000, dtype=np.uint64))
    s = Relation(np.arange(3000, dtype=np.uint64) % 512, np.arange(3000, dtype=np.uint64))
    res = P.run_pmpsm(r, s, JoinConfig(threads=2, key_domain=KeyDomain(0, 512)),
                      phase_hook=lambda w, ph: calls.append((w, ph)))
    for w in range(2):
        assert [p for ww, p in calls if ww == w] == ["sort_public", "histogram", "scatter", "sort_private", "join"]
    pt = res.phase_timings
    assert set(pt) == {"sort_public", "partition", "sort_private", "join", "total"}
    assert pt["sort_public"] + pt["partition"] + pt["sort_private"] + pt["join"] <= pt["total"] * 1.05 + 1e-9


# ---------------------------------------------------------------- operator level

@pytest.mark.parametrize("n", [0, 1, 2, 17, 4095, 4096, 4097, 3 * 4096 + 5, 200_003])
@pytest.mark.parametrize("upper_bits", [1, 5, 9, 20, 27, 32, 64])
def test_sort_pairs_vs_numpy(n, upper_bits):
    rng = np.random.default_rng(n * 131 + upper_bits)
    hi = (1 << upper_bits) if upper_bits < 64 else None
    keys = rng.integers(0, hi, n, dtype=np.uint64) if hi else rng.integers(0, 1 << 63, n, dtype=np.uint64) * np.uint64(2)
    pays = np.arange(n, dtype=np.uint64)
    rel = Relation(keys.copy(), pays.copy())
    P.sort_run(rel, KeyDomain(0, 1 << upper_bits))
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(rel.keys, keys[order])
    # payload order among equal keys is unspecified (sorter.py:6-7): compare
    # the (key, payload) multisets
    got = np.lexsort((rel.payloads, rel.keys))
    want = np.lexsort((pays, keys))
    assert np.array_equal(rel.payloads[got], pays[want])


def test_sort_shifted_domain_and_errors():
    rng = np.random.default_rng(9)
    keys = rng.integers(1000, 1512, 40_000, dtype=np.uint64)
    rel = Relation(keys.copy(), keys.copy())
    P.sort_run(rel, KeyDomain(1000, 1512))
    assert np.array_equal(rel.keys, np.sort(keys))
    with pytest.raises(DomainError):
        P.sort_run(Relation.from_tuples([(40, 1)]), KeyDomain(0, 32))


def test_histogram_and_scatter_kats():
    from paper_1207_0145_b200.partition import (SplitterVector, allocate_partition_arena, build_radix_histogram,
                                                combine_prefix_cursors, scatter)

    A = Relation.from_tuples([(13, 0), (1, 1), (9, 2), (27, 3), (5, 4), (30, 5), (19, 6)])
    B = Relation.from_tuples([(2, 10), (17, 11), (6, 12), (22, 13), (31, 14), (11, 15), (25, 16)])
    C = Relation.from_tuples([(0, 0), (3, 1), (9, 2), (1, 3), (16, 4), (7, 5), (21, 6)])
    Dd = Relation.from_tuples([(4, 10), (12, 11), (8, 12), (5, 13), (26, 14), (18, 15), (6, 16)])
    dom = KeyDomain(0, 32)
    assert build_radix_histogram(A, dom, 1).counts.tolist() == [4, 3]
    assert build_radix_histogram(B, dom, 1).counts.tolist() == [3, 4]
    assert build_radix_histogram(C, dom, 2).counts.tolist() == [4, 1, 2, 0]
    assert build_radix_histogram(Dd, dom, 2).counts.tolist() == [3, 2, 1, 1]
    hists = [build_radix_histogram(A, dom, 1), build_radix_histogram(B, dom, 1)]
    sp = SplitterVector.identity(2)
    cur = combine_prefix_cursors(hists, sp)
    arena = allocate_partition_arena(cur)
    scatter(A, 0, cur, sp, dom, arena)
    scatter(B, 1, cur, sp, dom, arena)
    r0, r1 = arena.run_view(0), arena.run_view(1)
    assert r0.keys.tolist() == [13, 1, 9, 5, 2, 6, 11]  # exact reference layout (host view, as the reference's)
    assert r0.payloads.tolist() == [0, 1, 2, 4, 10, 12, 15]
    assert r1.keys.tolist() == [27, 30, 19, 17, 22, 31, 25]
    assert arena.device_keys.cpu().tolist() == [13, 1, 9, 5, 2, 6, 11, 27, 30, 19, 17, 22, 31, 25]
    from paper_1207_0145_b200.core import InternalConsistencyError

    hc = [build_radix_histogram(C, dom, 2)]
    cur = combine_prefix_cursors(hc, SplitterVector.identity(4))
    with pytest.raises(InternalConsistencyError):
        scatter(Dd, 0, cur, SplitterVector.identity(4), dom, allocate_partition_arena(cur))


def test_radix_msd_pass():
    rel = Relation.from_tuples([(255, 0), (0, 1), (128, 2)])
    b = P.radix_msd_pass(rel, KeyDomain(0, 256))
    assert rel.keys.tolist() == [0, 128, 255] and b.bucket_count == 256
    rel = Relation.from_tuples([(7, i) for i in range(10)])
    b = P.radix_msd_pass(rel, KeyDomain(0, 256))
    assert b.offsets[8] - b.offsets[7] == 10


def test_interp_search_probes_match_reference(golden):
    for c in golden["interp_search"]:
        keys = torch.from_numpy(np.array(c["keys"], np.uint64)).to(DEV)
        tg = torch.from_numpy(np.array(c["targets"], np.uint64)).to(DEV)
        idx, probes = D.interp_lower_bound(keys, tg)
        got = list(zip(idx.cpu().tolist(), probes.cpu().tolist()))
        assert [list(x) for x in got] == c["results"]
    assert P.interpolation_search(P.Run(np.array([10, 20, 30, 40], np.uint64), np.zeros(4, np.uint64)), 25) == 2


def test_merge_join_kats():
    r = P.Run(np.array([2, 2], np.uint64), np.array([1, 2], np.uint64))
    s = P.Run(np.array([2, 2, 2], np.uint64), np.array([10, 20, 30], np.uint64))
    pairs = []
    assert P.merge_join(r, s, 0, lambda a, b: pairs.append((a, b))) == 6
    assert sorted(pairs) == sorted((a, b) for a in (1, 2) for b in (10, 20, 30))
    r = P.Run(np.array([1, 3], np.uint64), np.array([1, 3], np.uint64))
    s = P.Run(np.array([2, 4], np.uint64), np.array([2, 4], np.uint64))
    assert P.merge_join(r, s, 0, lambda a, b: None) == 0


def test_launch_counter_moves():
    before = _lib.launch_count()
    r, s, dom = P.gen_fk(1000, 4000, 1)
    P.run_join(r, s, JoinConfig(key_domain=dom))
    assert _lib.launch_count() > before


def test_wide_payloads_fall_back_to_pairs():
    # domain [0, 2^32) leaves 32 payload bits in a packed record; 2^40 payloads
    # overflow it, so the engine must redo the join on (key, payload) pairs
    rng = np.random.default_rng(4)
    rk = rng.integers(0, 1 << 32, 50_000, dtype=np.uint64)
    sk = np.concatenate([rk[:30_000], rng.integers(0, 1 << 32, 20_000, dtype=np.uint64)])
    rp = rng.integers(0, 1 << 44, rk.shape[0], dtype=np.uint64)
    sp = rng.integers(0, 1 << 63, sk.shape[0], dtype=np.uint64)
    want = orc.join(rk, rp, sk, sp, threads=2, lower=0, upper=1 << 32)
    for t in (1, 2):
        res = P.run_join(Relation(rk, rp), Relation(sk, sp), JoinConfig(threads=t, key_domain=KeyDomain(0, 1 << 32)))
        assert (res.match_count, res.aggregate_max, res.checksum) == (want.match_count, want.aggregate_max,
                                                                     want.checksum)


@pytest.mark.parametrize("width", [1, 7, 27, 33, 63])
def test_packed_sort_round_trip(width):
    n = 300_001
    rng = np.random.default_rng(width)
    lower = 5
    keys = rng.integers(lower, lower + (1 << width), n, dtype=np.uint64)
    pw = 64 - width
    pays = rng.integers(0, 1 << min(pw, 63), n, dtype=np.uint64)
    kd, pd = torch.from_numpy(keys).to(DEV), torch.from_numpy(pays).to(DEV)
    out, tmp = torch.empty_like(kd), torch.empty_like(kd)
    ovf = torch.zeros(1, dtype=torch.int32, device=DEV)
    D.sort_packed(kd, pd, lower, (1 << width) - 1, width, out, tmp, None, ovf)
    rec = out.cpu().numpy()
    assert int(ovf.item()) == 0
    got_k = (rec >> np.uint64(pw)) + np.uint64(lower)
    got_p = rec & np.uint64((1 << pw) - 1) if pw < 64 else rec
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(got_k, keys[order])
    a, b = np.lexsort((got_p, got_k)), np.lexsort((pays, keys))
    assert np.array_equal(got_p[a], pays[b])


_STABLE_CHILD = r'''
import sys
import numpy as np
import torch
sys.path.insert(0, sys.argv[1])
from paper_1207_0145_b200 import device as D
dev = torch.device("cuda", 0)
D.ensure_device()
for n, width in ((1, 9), (4097, 9), (8193, 27), (300_001, 27), (1_000_003, 33), (2_500_000, 20),
                 (5_000_000, 18), (1_300_000, 10), (70_000, 3)):
    rng = np.random.default_rng(n + width)
    keys = rng.integers(0, 1 << width, n, dtype=np.uint64)
    idx = np.arange(n, dtype=np.uint64)  # payload = input position: a stable sort keeps it increasing per key
    order = np.argsort(keys, kind="stable")
    kd, pd = torch.from_numpy(keys).to(dev), torch.from_numpy(idx).to(dev)
    # packed (SP + PP record passes, k_scatter_ws)
    out, tmp = torch.empty_like(kd), torch.empty_like(kd)
    ovf = torch.zeros(1, dtype=torch.int32, device=dev)
    D.sort_packed(kd, pd, 0, (1 << width) - 1, width, out, tmp, None, ovf)
    rec = out.cpu().numpy()
    pw = 64 - width
    assert int(ovf.item()) == 0
    assert np.array_equal(rec >> np.uint64(pw), keys[order]), ("packed keys", n, width)
    assert np.array_equal(rec & np.uint64((1 << pw) - 1), idx[order]), ("packed stability", n, width)
    # records in, records out (PP only)
    rin_np = rec[rng.permutation(n)]
    out2, tmp2 = torch.empty_like(kd), torch.empty_like(kd)
    D.sort_records(torch.from_numpy(rin_np).to(dev), width, out2, tmp2)
    want = rin_np[np.argsort(rin_np >> np.uint64(pw), kind="stable")]
    assert np.array_equal(out2.cpu().numpy(), want), ("records", n, width)
    # pairs (SS passes, k_scatter)
    ok, op, tk, tp = (torch.empty_like(kd) for _ in range(4))
    D.sort_pairs(kd, pd, 0, (1 << width) - 1, width, ok, op, tk, tp, None)
    assert np.array_equal(ok.cpu().numpy(), keys[order]), ("pairs keys", n, width)
    assert np.array_equal(op.cpu().numpy(), idx[order]), ("pairs stability", n, width)
print("STABLE-OK lane_ordered=%d" % D._lib.load().mpsm_dbg_lane_ordered())
'''


@pytest.mark.parametrize("ballot", ["0", "1"], ids=["lane-ordered-atomics", "ballot-fallback"])
def test_sorts_are_stable_on_both_ranking_paths(ballot):
    """Every scatter kernel (pairs, packing, record passes) is a stable
    pass, with the lane-ordered shared-atomic ranking and with the warp-ballot
    fallback the library uses where the start-up probe fails
    (MPSM_SEG_BALLOT_RANK=1 forces it; read once per process)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MPSM_SEG_BALLOT_RANK=ballot)
    r = subprocess.run([sys.executable, "-c", _STABLE_CHILD, root], env=env, capture_output=True, text=True,
                       timeout=600)
    assert "STABLE-OK" in r.stdout, r.stdout + r.stderr
    assert f"lane_ordered={1 - int(ballot)}" in r.stdout or ballot == "0", r.stdout


# ------------------------------------------------------- unaligned buffers

@pytest.mark.parametrize("off_r,off_s", [(1, 0), (0, 1), (1, 3), (3, 1)])
def test_unaligned_device_views_match_oracle(off_r, off_s, pack_mode):
    """Inputs that are views at an 8-B (not 16-B) offset: the sorts' bulk
    tile copies move the aligned body and copy the head/tail elements
    themselves (segsort.cu tile_plain), the merge stages aligned supersets."""
    r, s, dom = P.gen_fk(300_001, 1_200_007, 11)
    want = orc.fk_gather(r.keys, r.payloads, s.keys, s.payloads, 1)

    def view(a, off):
        buf = torch.empty(a.shape[0] + off, dtype=torch.uint64, device=DEV)
        buf[off:] = torch.from_numpy(a).to(DEV)
        return buf[off:]

    rd = Relation(view(r.keys, off_r), view(r.payloads, off_s))
    sd = Relation(view(s.keys, off_s), view(s.payloads, off_r))
    assert rd.keys.data_ptr() % 16 == 8 * (off_r % 2)
    for t in (1, 3):
        res = P.run_join(rd, sd, JoinConfig(threads=t, key_domain=dom))
        assert (res.match_count, res.aggregate_max, res.checksum) == want


@pytest.mark.parametrize("off", [1, 3])
def test_sorts_into_unaligned_outputs(off):
    """every sort entry with input, output and scratch buffers at 8-B offsets"""
    n, width = 70_001, 27
    rng = np.random.default_rng(off)
    keys = rng.integers(0, 1 << width, n, dtype=np.uint64)
    idx = np.arange(n, dtype=np.uint64)
    order = np.argsort(keys, kind="stable")

    def buf(src=None):
        b = torch.empty(n + off, dtype=torch.uint64, device=DEV)[off:]
        if src is not None:
            b.copy_(torch.from_numpy(src).to(DEV))
        return b

    kd, pd = buf(keys), buf(idx)
    out, tmp = buf(), buf()
    ovf = torch.zeros(1, dtype=torch.int32, device=DEV)
    D.sort_packed(kd, pd, 0, (1 << width) - 1, width, out, tmp, None, ovf)
    rec = out.cpu().numpy()
    pw = 64 - width
    assert np.array_equal(rec >> np.uint64(pw), keys[order])
    assert np.array_equal(rec & np.uint64((1 << pw) - 1), idx[order])
    out2, tmp2 = buf(), buf()
    shuffled = rec[rng.permutation(n)]
    D.sort_records(buf(shuffled), width, out2, tmp2)
    assert np.array_equal(out2.cpu().numpy(), shuffled[np.argsort(shuffled >> np.uint64(pw), kind="stable")])
    ok, op, tk, tp = buf(), buf(), buf(), buf()
    D.sort_pairs(kd, pd, 0, (1 << width) - 1, width, ok, op, tk, tp, None)
    assert np.array_equal(ok.cpu().numpy(), keys[order])
    assert np.array_equal(op.cpu().numpy(), idx[order])


@pytest.mark.parametrize("frac_wide", [0.0, 0.001, 1.0])
def test_payloads_above_32_bits_in_packed_records(frac_wide, pack_mode):
    """w = 27 leaves 37 payload bits in a packed record: payloads of 33-37
    bits stay on the packed path; merge tiles holding one switch from the
    low-word match phase to the full-record one (k_merge's per-tile flag)."""
    n_r, n_s = 200_000, 800_000
    r, s, _ = P.gen_fk(n_r, n_s, 3)
    dom = KeyDomain(1, (1 << 27) + 1)  # w = 27
    rng = np.random.default_rng(4)
    for rel in (r, s):
        n = rel.payloads.shape[0]
        big = rng.random(n) < frac_wide
        rel.payloads[big] = rng.integers(1 << 32, 1 << 37, int(big.sum()), dtype=np.uint64)
    want = orc.fk_gather(r.keys, r.payloads, s.keys, s.payloads, 1)
    for t in (1, 2):
        res = P.run_join(r, s, JoinConfig(threads=t, key_domain=dom))
        assert (res.match_count, res.aggregate_max, res.checksum) == want


@pytest.mark.parametrize("layout", ["packed", "records", "pairs"])
@pytest.mark.parametrize("sizes", [[5, 0, 8193, 1, 4095, 4097, 3], [100_003] * 7, [0, 0, 1], [12345]])
def test_segmented_sort_sorts_every_segment(layout, sizes):
    """mpsm_sort_*_segments: each segment sorted in place of position, stable
    (odd segment offsets, empty and one-element segments, tile edges)"""
    import torch

    from paper_1207_0145_b200 import device as D

    w = 23
    rng = np.random.default_rng(sum(sizes) + len(sizes))
    n = sum(sizes)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    keys = rng.integers(0, 1 << w, n, dtype=np.uint64)
    keys[::7] = keys[0]  # repeated keys: stability matters
    pays = np.arange(n, dtype=np.uint64)
    dk, dp = torch.from_numpy(keys).cuda(), torch.from_numpy(pays).cuda()
    out, tmp = torch.empty_like(dk), torch.empty_like(dk)
    bad = D.new_bad_flag(dk.device)
    ovf = torch.zeros(1, dtype=torch.int32, device=dk.device)
    pw = 64 - w
    if layout == "packed":
        D.sort_packed_segments(dk, dp, off, 0, (1 << w) - 1, w, out, tmp, bad, ovf)
        got_k = (out.cpu().numpy() >> np.uint64(pw))
        got_p = out.cpu().numpy() & np.uint64((1 << pw) - 1)
    elif layout == "records":
        rec = torch.from_numpy((keys << np.uint64(pw)) | pays).cuda()
        D.sort_records_segments(rec, off, w, out, tmp)
        got_k = (out.cpu().numpy() >> np.uint64(pw))
        got_p = out.cpu().numpy() & np.uint64((1 << pw) - 1)
    else:
        op, tp = torch.empty_like(dp), torch.empty_like(dp)
        D.sort_pairs_segments(dk, dp, off, 0, (1 << w) - 1, w, out, op, tmp, tp, bad)
        got_k, got_p = out.cpu().numpy(), op.cpu().numpy()
    assert int(bad.item()) == -1
    for s in range(len(sizes)):
        a, b = off[s], off[s + 1]
        order = np.argsort(keys[a:b], kind="stable")
        assert np.array_equal(got_k[a:b], keys[a:b][order]), s
        assert np.array_equal(got_p[a:b], pays[a:b][order]), s
