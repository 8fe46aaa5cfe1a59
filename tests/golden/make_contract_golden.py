"""Generate tests/golden/contract.json by running the REFERENCE package itself:
the exact error messages and result shapes of the boundary that the engine
fixtures (make_golden.py) do not cover.

    python tests/golden/make_contract_golden.py   # build container only

* domain errors: run_join over small relations with out-of-domain keys in r
  and / or s -> the reference's DomainError text (engine.py:181-190: r checked
  before s, violation count, first index);
* hash-oracle: run_join(algorithm="hash-oracle") (engine.py:462-465 ->
  datagen.hash_join_oracle, datagen.py:121-200) in every query mode ->
  match_count, aggregate_max, the checksum of its materialized pairs,
  phase_timings keys, worker_stats length; its ValueError for payloads >=
  2^63 and its MaterializeCapExceeded.
The inputs are small and stored in the JSON itself.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF_SRC)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import mpsm  # noqa: E402  (the reference)

from oracle.oracle import pair_hash_np  # noqa: E402


def checksum_pairs(mat) -> int:
    if mat is None or mat.shape[0] == 0:
        return 0
    return int(np.sum(pair_hash_np(mat[:, 0], mat[:, 1]), dtype=np.uint64))


def rel(keys, pays):
    return mpsm.Relation(np.asarray(keys, np.uint64), np.asarray(pays, np.uint64))


def main():
    rng = np.random.default_rng(20261020)
    out = {"reference": REF_SRC, "domain_errors": [], "hash_oracle": [], "hash_oracle_errors": []}

    # ---- domain errors
    lower, upper = 10, 1010
    for case, (n_r, bad_r, n_s, bad_s) in enumerate([
        (500, [17], 2000, []), (500, [], 2000, [5, 1999]), (500, [0, 3, 499], 2000, [7]),
        (3, [], 7000, [6999]), (9000, [8999, 4], 300, [0]),
    ]):
        rk = rng.integers(lower, upper, n_r, dtype=np.uint64)
        sk = rng.integers(lower, upper, n_s, dtype=np.uint64)
        for j, i in enumerate(bad_r):
            rk[i] = np.uint64(upper + j) if j % 2 == 0 else np.uint64(lower - 1 - j)
        for j, i in enumerate(bad_s):
            sk[i] = np.uint64(upper + 100 + j)
        rp = rng.integers(0, 1 << 32, n_r, dtype=np.uint64)
        sp = rng.integers(0, 1 << 32, n_s, dtype=np.uint64)
        runs = []
        for algo in ("p-mpsm", "b-mpsm"):
            for t in (1, 3):
                cfg = mpsm.JoinConfig(threads=t, algorithm=algo, key_domain=mpsm.KeyDomain(lower, upper))
                try:
                    mpsm.run_join(rel(rk, rp), rel(sk, sp), cfg)
                    msg = None
                except mpsm.DomainError as e:
                    msg = str(e)
                runs.append(dict(algorithm=algo, threads=t, message=msg))
        out["domain_errors"].append(dict(case=case, lower=lower, upper=upper, r_keys=rk.tolist(), r_pays=rp.tolist(),
                                         s_keys=sk.tolist(), s_pays=sp.tolist(), runs=runs))

    # ---- hash oracle
    for case, (n_r, n_s, upper_k, wide) in enumerate([
        (300, 1200, 400, False), (1500, 200, 60, False), (0, 50, 10, False), (200, 800, 1 << 64, False),
        (100, 100, 5, True),
    ]):
        if upper_k == 1 << 64:
            rk = rng.integers(0, 1 << 63, n_r, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
            h = min(n_r, n_s // 2)
            sk = np.concatenate([rk[:h], rng.integers(0, 1 << 63, n_s - h, dtype=np.uint64)])
        else:
            rk = rng.integers(0, upper_k, n_r, dtype=np.uint64)
            sk = rng.integers(0, upper_k, n_s, dtype=np.uint64)
        hi = (1 << 62) if wide else (1 << 32)
        rp = rng.integers(0, hi, n_r, dtype=np.uint64)
        sp = rng.integers(0, hi, n_s, dtype=np.uint64)
        for mode in ("aggregate-max", "count", "materialize"):
            cfg = mpsm.JoinConfig(algorithm="hash-oracle", query_mode=mode, materialize_cap=1 << 22)
            res = mpsm.run_join(rel(rk, rp), rel(sk, sp), cfg)
            out["hash_oracle"].append(dict(
                case=case, mode=mode, r_keys=rk.tolist(), r_pays=rp.tolist(), s_keys=sk.tolist(), s_pays=sp.tolist(),
                match_count=res.match_count, aggregate_max=res.aggregate_max,
                materialized_rows=None if res.materialized is None else int(res.materialized.shape[0]),
                materialized_checksum=None if res.materialized is None else checksum_pairs(res.materialized),
                phase_timing_keys=sorted(res.phase_timings), worker_stats=len(res.worker_stats)))

    # ---- hash oracle errors
    keys = np.arange(20, dtype=np.uint64) % 4
    pays = np.arange(20, dtype=np.uint64)
    big = pays.copy()
    big[3] = np.uint64(1 << 63)
    for name, (r_, s_, cap) in {"wide_payload_s": ((keys, pays), (keys, big), 1 << 20),
                                "wide_payload_r": ((keys, big), (keys, big), 1 << 20),
                                "cap": ((keys, pays), (keys, pays), 50)}.items():
        cfg = mpsm.JoinConfig(algorithm="hash-oracle", query_mode="materialize", materialize_cap=cap)
        try:
            mpsm.run_join(rel(*r_), rel(*s_), cfg)
            err = None
        except Exception as e:  # noqa: BLE001 - recorded
            err = [type(e).__name__, str(e)]
        out["hash_oracle_errors"].append(dict(name=name, r_keys=r_[0].tolist(), r_pays=r_[1].tolist(),
                                              s_keys=s_[0].tolist(), s_pays=s_[1].tolist(), cap=cap, error=err))

    path = os.path.join(HERE, "contract.json")
    with open(path, "w") as f:
        json.dump(out, f)
    print("wrote", path, {k: len(v) for k, v in out.items() if isinstance(v, list)})


if __name__ == "__main__":
    main()
