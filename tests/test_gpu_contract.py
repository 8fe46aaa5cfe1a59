"""Boundary contract on the GPU against fixtures the REFERENCE produced
(tests/golden/contract.json, tests/golden/make_contract_golden.py):

* DomainError wording: r checked before s, violation count, first index
  (engine.py:181-190), for device and host inputs, both engines, T in {1, 3};
* algorithm="hash-oracle" (engine.py:462-465, datagen.py:121-200): counts,
  MAX, materialized rows, result shape, its ValueError / MaterializeCapExceeded;
* the Run order invariant (core.py:153-154): device Runs are checked, and the
  merge-join flags an unsorted run (InternalConsistencyError from run_join);
* materialize storage stops at the cap at the C ABI (_kernels.py:382-390).
"""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - collected on CPU boxes too
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1207_0145_b200 as P  # noqa: E402
from paper_1207_0145_b200 import _lib, engine  # noqa: E402
from paper_1207_0145_b200 import device as D  # noqa: E402
from paper_1207_0145_b200.core import (  # noqa: E402
    DomainError,
    InternalConsistencyError,
    JoinConfig,
    KeyDomain,
    MaterializeCapExceeded,
    Relation,
)
from oracle import oracle as orc  # noqa: E402  (checker only)

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "contract.json")) as fh:
    CONTRACT = json.load(fh)
DEV = torch.device("cuda", 0)


def _rel(keys, pays, device: bool):
    k, p = np.asarray(keys, np.uint64), np.asarray(pays, np.uint64)
    if device:
        return Relation(torch.from_numpy(k).to(DEV), torch.from_numpy(p).to(DEV))
    return Relation(k, p)


@pytest.mark.parametrize("device", [True, False], ids=["device", "host"])
@pytest.mark.parametrize("case", range(len(CONTRACT["domain_errors"])))
def test_domain_error_wording_matches_reference(case, device):
    c = CONTRACT["domain_errors"][case]
    dom = KeyDomain(c["lower"], c["upper"])
    for run in c["runs"]:
        r = _rel(c["r_keys"], c["r_pays"], device)
        s = _rel(c["s_keys"], c["s_pays"], device)
        with pytest.raises(DomainError) as ei:
            P.run_join(r, s, JoinConfig(threads=run["threads"], algorithm=run["algorithm"], key_domain=dom))
        assert str(ei.value) == run["message"], (run, str(ei.value))


@pytest.mark.parametrize("device", [True, False], ids=["device", "host"])
@pytest.mark.parametrize("i", range(len(CONTRACT["hash_oracle"])))
def test_hash_oracle_matches_reference(i, device):
    c = CONTRACT["hash_oracle"][i]
    r = _rel(c["r_keys"], c["r_pays"], device)
    s = _rel(c["s_keys"], c["s_pays"], device)
    res = P.run_join(r, s, JoinConfig(algorithm="hash-oracle", query_mode=c["mode"], materialize_cap=1 << 22))
    assert res.match_count == c["match_count"]
    assert res.aggregate_max == c["aggregate_max"]
    assert sorted(res.phase_timings) == c["phase_timing_keys"]
    assert len(res.worker_stats) == c["worker_stats"]
    if c["materialized_rows"] is None:
        assert res.materialized is None
    else:
        m = res.materialized
        assert m.shape == (c["materialized_rows"], 2)
        got = int(np.sum(orc.pair_hash_np(m[:, 0], m[:, 1]), dtype=np.uint64)) if m.shape[0] else 0
        assert got == c["materialized_checksum"]
    # the checksum of every mode equals the reference's materialized pairs'
    mat = [x for x in CONTRACT["hash_oracle"] if x["case"] == c["case"] and x["mode"] == "materialize"][0]
    assert res.checksum == mat["materialized_checksum"]


@pytest.mark.parametrize("i", range(len(CONTRACT["hash_oracle_errors"])))
def test_hash_oracle_errors_match_reference(i):
    c = CONTRACT["hash_oracle_errors"][i]
    r = _rel(c["r_keys"], c["r_pays"], True)
    s = _rel(c["s_keys"], c["s_pays"], True)
    exc = {"ValueError": ValueError, "MaterializeCapExceeded": MaterializeCapExceeded}[c["error"][0]]
    with pytest.raises(exc) as ei:
        P.run_join(r, s, JoinConfig(algorithm="hash-oracle", query_mode="materialize", materialize_cap=c["cap"]))
    assert str(ei.value) == c["error"][1]


def test_device_run_order_check():
    k = torch.arange(1000, dtype=torch.int64, device=DEV).view(torch.uint64)
    P.Run(k, k)  # sorted: fine
    bad = k.clone()
    bad.view(torch.int64)[500] = 7
    with pytest.raises(ValueError, match="not sorted"):
        P.Run(bad, k)


@pytest.mark.parametrize("packed", [True, False])
def test_merge_flags_unsorted_runs(packed):
    rng = np.random.default_rng(5)
    w = 20
    rk = np.sort(rng.integers(0, 1 << w, 50_000, dtype=np.uint64))
    sk = np.sort(rng.integers(0, 1 << w, 200_000, dtype=np.uint64))
    for which in ("none", "r", "s"):
        r2, s2 = rk.copy(), sk.copy()
        if which == "r":
            r2[30_000], r2[30_001] = r2[30_001] + 1, r2[30_000]
        if which == "s":
            s2[123_456] = s2[123_456] + 5000  # one key far out of place
        if packed:
            rr = torch.from_numpy(r2 << np.uint64(64 - w)).to(DEV)
            ss = torch.from_numpy(s2 << np.uint64(64 - w)).to(DEV)
            rec = D.join_pairs_packed([rr], [ss], w, 0, False, _lib.MODE_COUNT)
        else:
            rr = torch.from_numpy(r2).to(DEV)
            ss = torch.from_numpy(s2).to(DEV)
            rec = D.join_pairs([(rr, rr)], [(ss, ss)], False, _lib.MODE_COUNT)
        flags = int(rec[0, _lib.PAIR_FLAGS].item())
        assert bool(flags & _lib.FLAG_UNSORTED) == (which != "none"), which


def test_engine_raises_on_unsorted_run(monkeypatch):
    """a broken run sort (simulated: two records swapped after the sort) is
    caught by the merge walk instead of silently losing matches"""
    r, s, dom = P.gen_fk(200_000, 800_000, seed=4)
    real = D.sort_records

    def broken(in_rec, width_bits, out_rec, tmp_rec, dense=None):
        # the density probe (if asked for) describes the sort's own output;
        # the swap below happens after it -- the dense join's check of every
        # gathered R key must still catch the corrupted private run
        real(in_rec, width_bits, out_rec, tmp_rec, dense)
        n = out_rec.numel()
        if n > 1000:
            o = out_rec.view(torch.int64)
            a = o[n // 2].clone()
            o[n // 2] = o[n // 2 + 7]
            o[n // 2 + 7] = a

    monkeypatch.setattr(D, "sort_records", broken)
    with pytest.raises(InternalConsistencyError, match="not sorted"):
        P.run_join(r, s, JoinConfig(threads=1, key_domain=dom))  # host inputs: record sorts


@pytest.mark.parametrize("packed", [True, False])
def test_materialize_stops_at_cap(packed):
    rng = np.random.default_rng(11)
    w = 12
    rk = np.sort(rng.integers(0, 1 << w, 5_000, dtype=np.uint64))
    sk = np.sort(rng.integers(0, 1 << w, 20_000, dtype=np.uint64))
    rp = rng.integers(0, 1 << 20, rk.shape[0], dtype=np.uint64)
    sp = rng.integers(0, 1 << 20, sk.shape[0], dtype=np.uint64)
    want = orc.join(rk, rp, sk, sp, threads=1, lower=0, upper=1 << w)
    total = want.match_count
    assert total > 1000
    cap = total // 3
    if packed:
        rr = torch.from_numpy((rk << np.uint64(64 - w)) | rp).to(DEV)
        ss = torch.from_numpy((sk << np.uint64(64 - w)) | sp).to(DEV)
        run = lambda mode, out=None, c=0: D.join_pairs_packed([rr], [ss], w, 0, False, mode, out, c)  # noqa: E731
    else:
        rr = (torch.from_numpy(rk).to(DEV), torch.from_numpy(rp).to(DEV))
        ss = (torch.from_numpy(sk).to(DEV), torch.from_numpy(sp).to(DEV))
        run = lambda mode, out=None, c=0: D.join_pairs([rr], [ss], False, mode, out, c)  # noqa: E731
    guard = 1000
    out = torch.full((2 * (cap + guard),), 0xABCD, dtype=torch.int64, device=DEV).view(torch.uint64)
    rec = run(_lib.MODE_MATERIALIZE, out, cap)
    assert int(rec[0, _lib.PAIR_COUNT].item()) == total
    assert int(rec[0, _lib.PAIR_EMITTED].item()) == cap
    o = out.view(torch.int64).cpu().numpy()
    assert np.all(o[2 * cap:] == 0xABCD)  # nothing written past the cap
    # the stored rows are genuine pairs: a prefix of the full emission
    full = torch.empty(2 * total, dtype=torch.uint64, device=DEV)
    run(_lib.MODE_MATERIALIZE, full, total)
    assert np.array_equal(o[:2 * cap], full.view(torch.int64).cpu().numpy()[:2 * cap])


def test_threads_above_partition_scatter_limit():
    """JoinConfig accepts T <= 2^radix_bits (1024 with the defaults) like the
    reference; the one-GPU engine's partition is a cut of the sorted private
    run, so T = 600 works (the scatter held T to 512)"""
    r, s, dom = P.gen_fk(50_000, 200_000, seed=8)
    want = orc.fk_gather(r.keys, r.payloads, s.keys, s.payloads, dom.lower)
    res = P.run_join(r, s, JoinConfig(threads=600, key_domain=dom))
    assert (res.match_count, res.aggregate_max, res.checksum) == want
    assert sum(w.tuples_sorted_private for w in res.worker_stats) == r.cardinality


@pytest.mark.parametrize("pay_bits", [32, 33, 40])
@pytest.mark.parametrize("dense", [True, False])
def test_packed_payloads_above_32_bits(pay_bits, dense):
    """packed records whose payloads use bits above 31 (kept in the record's
    high word, w + pay_bits <= 64) take the merge's 64-bit payload path; every
    other tile the 32-bit one -- both against the oracle (FK dense keys and
    sparse keys)"""
    rng = np.random.default_rng(pay_bits + 100 * dense)
    w = 20
    n_r, n_s = 200_000, 800_000
    if dense:
        rk = (rng.permutation(n_r) + 1).astype(np.uint64)
        sk = rng.integers(1, n_r + 1, n_s, dtype=np.uint64)
    else:
        rk = rng.integers(1, 1 << w, n_r, dtype=np.uint64)
        sk = rng.integers(1, 1 << w, n_s, dtype=np.uint64)
    rp = rng.integers(0, 1 << 32, n_r, dtype=np.uint64)
    sp = rng.integers(0, 1 << 32, n_s, dtype=np.uint64)
    # a few payloads with high bits (one per ~1000 tuples: most tiles stay narrow)
    hi = np.uint64((1 << pay_bits) - 1)
    rp[::997] = rng.integers(0, 1 << 62, rp[::997].shape[0], dtype=np.uint64) & hi
    sp[::1009] = rng.integers(0, 1 << 62, sp[::1009].shape[0], dtype=np.uint64) & hi
    dom = KeyDomain(1, 1 << w)
    want = orc.join(rk, rp, sk, sp, threads=1, lower=1, upper=1 << w)
    for device in (True, False):
        res = P.run_join(_rel(rk, rp, device), _rel(sk, sp, device), JoinConfig(threads=1, key_domain=dom))
        assert (res.match_count, res.aggregate_max, res.checksum) == (want.match_count, want.aggregate_max,
                                                                     want.checksum)
