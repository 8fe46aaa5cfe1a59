"""Pin the CPU oracle (oracle/) to the reference's own outputs.

The fixtures in tests/golden/golden.json were produced by running the
reference package (tests/golden/make_golden.py).  If the oracle reproduces
every one of them, it is a trustworthy checker for the CUDA path.
"""

import numpy as np
import pytest

from oracle import oracle as orc
from tests.golden_inputs import dataset, fingerprint, make_inputs

pytestmark = []


def test_inputs_reproduce_reference_generators(golden):
    for d in golden["datasets"]:
        rk, rp, sk, sp, lo, up = make_inputs(d)
        fp = golden["input_fingerprints"][d["name"]]
        assert fingerprint(rk) == fp["r_keys"], d["name"]
        assert fingerprint(rp) == fp["r_pays"], d["name"]
        assert fingerprint(sk) == fp["s_keys"], d["name"]
        assert fingerprint(sp) == fp["s_pays"], d["name"]
        assert (lo, up) == (fp["lower"], fp["upper"])


def _run(case):
    d = dataset(case["dataset"])
    rk, rp, sk, sp, lo, up = make_inputs(d)
    return orc.join(rk, rp, sk, sp, threads=case["threads"], lower=lo, upper=up, radix_bits=case["radix_bits"],
                    algorithm=case["algorithm"], role_policy=case["role_policy"], query_mode=case["query_mode"],
                    materialize_cap=1 << 26)


def test_engine_cases_match_reference(golden):
    n_checked = 0
    for case in golden["engine_cases"]:
        if "error" in case:
            with pytest.raises(ValueError):
                _run(case)
            continue
        res = _run(case)
        tag = (case["dataset"], case["algorithm"], case["threads"], case["query_mode"], case["role_policy"])
        assert res.match_count == case["match_count"], tag
        assert res.aggregate_max == case["aggregate_max"], tag
        if "checksum" in case:
            assert res.checksum == case["checksum"], tag
            assert orc.pairs_checksum(res.materialized[:, 0].copy(), res.materialized[:, 1].copy()) == case["checksum"]
        for got, want in zip(res.worker_stats, case["worker_stats"]):
            for k in ("tuples_sorted_public", "tuples_sorted_private", "tuples_scattered",
                      "public_tuples_examined", "probe_tuples_examined", "s_runs_with_matches"):
                assert getattr(got, k) == want[k], (tag, k)
        n_checked += 1
    assert n_checked > 100


def test_config1_golden(golden):
    g = golden["config1"]
    rk, rp, sk, sp = orc.gen_fk(g["n_r"], g["n_s"], g["seed"])
    assert fingerprint(sk) == g["s_keys"] and fingerprint(rk) == g["r_keys"]
    res = orc.join(rk, rp, sk, sp, threads=8, lower=g["lower"], upper=g["upper"], parallel=True)
    assert res.match_count == g["match_count"] == 4_000_000
    assert res.aggregate_max == g["aggregate_max"] == 8_587_739_465
    assert res.checksum == g["checksum"] == 0x7CDED1377072045D
    for got, want in zip(res.worker_stats, g["worker_stats"]):
        assert got.public_tuples_examined == want["public_tuples_examined"]
        assert got.probe_tuples_examined == want["probe_tuples_examined"]
        assert got.s_runs_with_matches == want["s_runs_with_matches"]
    # independent FK gather agrees
    assert orc.fk_gather(rk, rp, sk, sp, 1) == (g["match_count"], g["aggregate_max"], g["checksum"])


def test_splitters_match_reference(golden):
    for c in golden["splitters"]:
        runs = [np.array(k, np.uint64) for k in c["runs"]]
        cdf = orc.build_cdf([orc.local_equiheight_bounds(k, c["f"], c["t"]) for k in runs], anchor_key=c["lower"])
        wb = orc.width_bits(c["lower"], c["upper"])
        bounds = orc.compute_splitters(np.array(c["hist"], np.int64), cdf, c["t"], c["lower"], wb, c["bits"])
        assert bounds == c["bucket_bounds"], c["bits"]


def test_interp_search_matches_reference(golden):
    for c in golden["interp_search"]:
        keys = np.array(c["keys"], np.uint64)
        for tgt, want in zip(c["targets"], c["results"]):
            assert list(orc.interp_lower_bound(keys, tgt)) == want


# known answers from the reference's tests (paper Fig. 6 / Fig. 10 chunks,
# test_partition.py:27-43, 88-95, 177-184)
CHUNK_A = [(13, 0), (1, 1), (9, 2), (27, 3), (5, 4), (30, 5), (19, 6)]
CHUNK_B = [(2, 10), (17, 11), (6, 12), (22, 13), (31, 14), (11, 15), (25, 16)]
CHUNK_C = [(0, 0), (3, 1), (9, 2), (1, 3), (16, 4), (7, 5), (21, 6)]
CHUNK_D = [(4, 10), (12, 11), (8, 12), (5, 13), (26, 14), (18, 15), (6, 16)]


def _keys(ch):
    return np.array([k for k, _ in ch], np.uint64), np.array([p for _, p in ch], np.uint64)


def test_histogram_kats():
    for ch, bits, want in ((CHUNK_A, 1, [4, 3]), (CHUNK_B, 1, [3, 4]), (CHUNK_C, 2, [4, 1, 2, 0]),
                           (CHUNK_D, 2, [3, 2, 1, 1])):
        c = np.zeros(1 << bits, np.int64)
        assert orc.radix_histogram(_keys(ch)[0], 0, 5 - bits, c) == -1
        assert c.tolist() == want


def test_scatter_layout_kat():
    # two workers, identity splitter vector over 1-bit buckets -> exact arena layout
    sp = np.array([0, 1], np.int64)
    ak = np.zeros(14, np.uint64)
    ap = np.zeros(14, np.uint64)
    starts = [[0, 7], [4, 10]]
    ends = [[4, 10], [7, 14]]
    for w, ch in enumerate((CHUNK_A, CHUNK_B)):
        k, p = _keys(ch)
        cur = np.array(starts[w], np.int64)
        assert orc.scatter_chunk(k, p, 0, 4, sp, cur, np.array(ends[w], np.int64), ak, ap) == -1
        assert cur.tolist() == ends[w]
    assert ak[:7].tolist() == [13, 1, 9, 5, 2, 6, 11]
    assert ap[:7].tolist() == [0, 1, 2, 4, 10, 12, 15]
    assert ak[7:].tolist() == [27, 30, 19, 17, 22, 31, 25]


def test_interp_kats():
    k = np.array([10, 20, 30, 40], np.uint64)
    assert orc.interp_lower_bound(k, 10)[0] == 0
    assert orc.interp_lower_bound(k, 45)[0] == 4
    assert orc.interp_lower_bound(k, 25)[0] == 2
    assert orc.interp_lower_bound(np.array([7, 7, 7, 7], np.uint64), 7)[0] == 0
    assert orc.interp_lower_bound(np.array([7, 7], np.uint64), 8)[0] == 2
    assert orc.interp_lower_bound(np.array([3, 9], np.uint64), 9)[0] == 1


def test_merge_kats():
    rk = np.array([2, 2], np.uint64)
    rp = np.array([1, 2], np.uint64)
    sk = np.array([2, 2, 2], np.uint64)
    sp = np.array([10, 20, 30], np.uint64)
    c, b, ex, _, cs = orc.merge_join_run(rk, rp, sk, sp, 0)
    assert c == 6 and b == 32
    assert cs == sum(orc.pair_hash(a, x) for a in (1, 2) for x in (10, 20, 30)) % (1 << 64)
    # scan stops at the private maximum (test_engine.py:157-166)
    r = np.array([5, 6], np.uint64)
    s = np.arange(1000, dtype=np.uint64)
    c, _, ex, _, _ = orc.merge_join_run(r, r.copy(), s, s.copy(), 0)
    assert c == 2 and ex <= 8


def test_sort_matches_numpy():
    rng = np.random.default_rng(7)
    for n, upper in ((0, 8), (1, 8), (15, 8), (1000, 64), (100_000, 1 << 32)):
        k = rng.integers(0, upper, n, dtype=np.uint64)
        p = rng.integers(0, 1 << 32, n, dtype=np.uint64)
        want = sorted(zip(k.tolist(), p.tolist()))
        kk, pp = k.copy(), p.copy()
        assert orc.three_phase_sort(kk, pp, 0, (upper - 1).bit_length()) >= 0
        assert np.all(kk[:-1] <= kk[1:])
        assert sorted(zip(kk.tolist(), pp.tolist())) == want
