"""Generate tests/golden/golden.json by running the REFERENCE package itself.

Run in the build container (the reference lives at /root/reference and is
read-only; it does not exist on the GPU box, which only reads the committed
JSON):

    python tests/golden/make_golden.py

What it records (all from /root/reference/pkg/src/mpsm, unmodified):
* engine cases: run_join over seeded inputs (aggregate-max and materialize
  modes) for b-mpsm / p-mpsm and several T -> match_count, aggregate_max,
  checksum of the reference's materialized (r_pay, s_pay) pairs (the
  reference has no checksum; SURVEY.md finding 3), per-worker statistics;
* config 1 of BASELINE.json (FK 1M x 4M, seed 0): count, max, checksum from
  the reference's materialized pairs;
* splitter cases: skew.compute_splitters bucket bounds (exact-search and
  float-bisection paths);
* interpolation search: (index, probes) of _kernels.interp_lower_bound;
* input fingerprints of datagen.gen_skewed_8020 so our restated generator
  can be checked to reproduce the reference's arrays.
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
from mpsm import _kernels  # noqa: E402

from oracle.oracle import gen_fk, pair_hash_np  # noqa: E402


def checksum_pairs(mat: np.ndarray) -> int:
    if mat is None or mat.shape[0] == 0:
        return 0
    return int(np.sum(pair_hash_np(mat[:, 0], mat[:, 1]), dtype=np.uint64))


def fingerprint(a: np.ndarray) -> list:
    a = np.ascontiguousarray(a, np.uint64)
    return [int(a.shape[0]), int(np.sum(a, dtype=np.uint64)), int(np.sum(pair_hash_np(a, np.arange(a.shape[0], dtype=np.uint64)), dtype=np.uint64))]


def rel_random(n, seed, upper):
    rng = np.random.default_rng(seed)
    return (rng.integers(0, upper, n, dtype=np.uint64), rng.integers(0, 1 << 32, n, dtype=np.uint64))


# dataset recipes understood by tests/golden_inputs.py (kept in sync)
DATASETS = [
    dict(name="uniform_small", kind="random", n_r=1000, n_s=4000, upper=1 << 10, seed_r=50, seed_s=150),
    dict(name="uniform_mid", kind="random", n_r=10000, n_s=40000, upper=1 << 14, seed_r=51, seed_s=151),
    dict(name="sparse_wide", kind="random", n_r=5000, n_s=5000, upper=1 << 30, seed_r=52, seed_s=152),
    dict(name="empty_r", kind="random", n_r=0, n_s=100, upper=256, seed_r=53, seed_s=153),
    dict(name="empty_s", kind="random", n_r=100, n_s=0, upper=256, seed_r=54, seed_s=154),
    dict(name="dup_heavy", kind="random", n_r=800, n_s=1600, upper=64, seed_r=91, seed_s=92),
    dict(name="r_bigger", kind="random", n_r=9000, n_s=3000, upper=1 << 12, seed_r=61, seed_s=62),
    dict(name="fk_small", kind="fk", n_r=20000, n_s=80000, seed=3),
    dict(name="negcorr", kind="skew", n_r=20000, n_s=80000, upper=1 << 16, seed_r=7, seed_s=8),
    dict(name="self_join", kind="self", n=500, upper=64, seed=33),
]


def make_inputs(d):
    if d["kind"] == "random":
        rk, rp = rel_random(d["n_r"], d["seed_r"], d["upper"])
        sk, sp = rel_random(d["n_s"], d["seed_s"], d["upper"])
        return rk, rp, sk, sp, 0, d["upper"]
    if d["kind"] == "fk":
        rk, rp, sk, sp = gen_fk(d["n_r"], d["n_s"], d["seed"])
        return rk, rp, sk, sp, 1, d["n_r"] + 1
    if d["kind"] == "skew":
        dom = mpsm.KeyDomain(0, d["upper"])
        r = mpsm.generate(mpsm.GenSpec(d["n_r"], dom, "skew-80-20-high", seed=d["seed_r"]))
        s = mpsm.generate(mpsm.GenSpec(d["n_s"], dom, "skew-80-20-low", seed=d["seed_s"]))
        return r.keys, r.payloads, s.keys, s.payloads, 0, d["upper"]
    if d["kind"] == "self":
        rng = np.random.default_rng(d["seed"])
        k = rng.integers(0, d["upper"], d["n"], dtype=np.uint64)
        return k, k.copy(), k.copy(), k.copy(), 0, d["upper"]
    raise ValueError(d)


def run_case(d, algo, t, mode="aggregate-max", role="auto", radix_bits=10):
    rk, rp, sk, sp, lo, up = make_inputs(d)
    cfg = mpsm.JoinConfig(threads=t, algorithm=algo, key_domain=mpsm.KeyDomain(lo, up), radix_bits=radix_bits,
                          query_mode=mode, role_policy=role, materialize_cap=1 << 26)
    import warnings

    out = dict(dataset=d["name"], algorithm=algo, threads=t, query_mode=mode, role_policy=role,
               radix_bits=radix_bits)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        try:
            res = mpsm.run_join(mpsm.Relation(rk, rp), mpsm.Relation(sk, sp), cfg)
        except Exception as exc:  # the reference's own failure is part of its behaviour
            out["error"] = type(exc).__name__
            out["error_message"] = str(exc)
            return out
    out.update(match_count=res.match_count, aggregate_max=res.aggregate_max)
    if mode == "materialize":
        out["checksum"] = checksum_pairs(res.materialized)
    out["worker_stats"] = [
        dict(worker=w.worker, tuples_sorted_public=w.tuples_sorted_public,
             tuples_sorted_private=w.tuples_sorted_private, tuples_scattered=w.tuples_scattered,
             public_tuples_examined=w.public_tuples_examined, probe_tuples_examined=w.probe_tuples_examined,
             s_runs_with_matches=w.s_runs_with_matches)
        for w in res.worker_stats
    ]
    return out


def main():
    mpsm.warmup()
    golden = dict(generator="tests/golden/make_golden.py", reference="/root/reference/pkg/src/mpsm",
                  numpy=np.__version__)
    golden["datasets"] = DATASETS
    fps = {}
    for d in DATASETS:
        rk, rp, sk, sp, lo, up = make_inputs(d)
        fps[d["name"]] = dict(r_keys=fingerprint(rk), r_pays=fingerprint(rp), s_keys=fingerprint(sk),
                              s_pays=fingerprint(sp), lower=lo, upper=up)
    golden["input_fingerprints"] = fps

    cases = []
    for d in DATASETS:
        for algo in ("b-mpsm", "p-mpsm"):
            for t in (1, 2, 3, 4, 8):
                cases.append(run_case(d, algo, t))
        # materialize (checksum source) at two worker counts
        for algo in ("b-mpsm", "p-mpsm"):
            for t in (1, 4):
                cases.append(run_case(d, algo, t, mode="materialize"))
        cases.append(run_case(d, "p-mpsm", 2, mode="count"))
        for role in ("r-private", "s-private"):
            cases.append(run_case(d, "p-mpsm", 2, mode="materialize", role=role))
    # narrow radix grids (exact-search splitter path in the engine)
    for d in DATASETS[:3]:
        cases.append(run_case(d, "p-mpsm", 4, radix_bits=6))
    golden["engine_cases"] = cases

    # config 1 of BASELINE.json
    rk, rp, sk, sp = gen_fk(1_000_000, 4_000_000, 0)
    cfg = mpsm.JoinConfig(threads=8, algorithm="p-mpsm", key_domain=mpsm.KeyDomain(1, 1_000_001),
                          query_mode="materialize", materialize_cap=1 << 23)
    res = mpsm.run_join(mpsm.Relation(rk, rp), mpsm.Relation(sk, sp), cfg)
    cfg_agg = mpsm.JoinConfig(threads=8, algorithm="p-mpsm", key_domain=mpsm.KeyDomain(1, 1_000_001))
    res_agg = mpsm.run_join(mpsm.Relation(rk, rp), mpsm.Relation(sk, sp), cfg_agg)
    golden["config1"] = dict(n_r=1_000_000, n_s=4_000_000, seed=0, lower=1, upper=1_000_001,
                             match_count=res_agg.match_count, aggregate_max=res_agg.aggregate_max,
                             checksum=checksum_pairs(res.materialized),
                             r_keys=fingerprint(rk), r_pays=fingerprint(rp), s_keys=fingerprint(sk),
                             s_pays=fingerprint(sp),
                             worker_stats=[dict(worker=w.worker, public_tuples_examined=w.public_tuples_examined,
                                                probe_tuples_examined=w.probe_tuples_examined,
                                                s_runs_with_matches=w.s_runs_with_matches,
                                                tuples_sorted_private=w.tuples_sorted_private)
                                           for w in res_agg.worker_stats])

    # splitters: exact (n<=256) and float-bisection (n>256) paths
    spl = []
    rng = np.random.default_rng(1234)
    for case in range(40):
        bits = [2, 4, 6, 8, 9, 10, 10, 12][case % 8]
        t = [1, 2, 3, 4, 8, 8, 16, 5][case % 8]
        if (1 << bits) < t:
            continue
        lo = int(rng.integers(0, 1000))
        width = 1 << int(rng.integers(bits, 33))
        dom = mpsm.KeyDomain(lo, lo + width)
        skew = case % 3
        if skew == 0:
            hist = rng.integers(0, 1000, 1 << bits).astype(np.int64)
        elif skew == 1:
            hist = (rng.pareto(1.5, 1 << bits) * 100).astype(np.int64)
        else:
            hist = np.zeros(1 << bits, np.int64)
            hist[rng.integers(0, 1 << bits, 5)] = rng.integers(1, 10000, 5)
        runs = []
        for _ in range(t):
            n = int(rng.integers(0, 300))
            keys = np.sort(rng.integers(lo, lo + width, n, dtype=np.uint64))
            runs.append(keys)
        f = 4
        bounds = [mpsm.local_equiheight_bounds(mpsm.Run(k, k.copy()), f, t) for k in runs]
        cdf = mpsm.build_cdf(bounds, anchor_key=lo)
        ss = mpsm.compute_splitters(hist, cdf, t, dom, bits)
        spl.append(dict(bits=bits, t=t, lower=lo, upper=lo + width, f=f, hist=hist.tolist(),
                        runs=[k.tolist() for k in runs], bucket_bounds=ss.bucket_bounds.tolist(),
                        splitter_keys=ss.splitter_keys.tolist(), partition_sizes=ss.partition_sizes.tolist()))
    golden["splitters"] = spl

    # interpolation search probes
    isr = []
    for case in range(30):
        n = int(rng.integers(0, 2000))
        kind = case % 3
        if kind == 0:
            keys = np.sort(rng.integers(0, 1 << 32, n, dtype=np.uint64))
        elif kind == 1:
            keys = np.cumsum(rng.integers(1, 1000, n, dtype=np.uint64) ** np.uint64(3))
        else:
            keys = np.sort(rng.integers(0, 16, n, dtype=np.uint64))
        top = int(keys[-1]) + 2 if n else 100
        targets = rng.integers(0, top, 16, dtype=np.uint64).tolist()
        res = [list(map(int, _kernels.interp_lower_bound(keys, np.uint64(x)))) for x in targets]
        isr.append(dict(keys=keys.tolist(), targets=targets, results=res))
    golden["interp_search"] = isr

    path = os.path.join(HERE, "golden.json")
    with open(path, "w") as fh:
        json.dump(golden, fh, separators=(",", ":"))
    print("wrote", path, os.path.getsize(path), "bytes;", len(cases), "engine cases")


if __name__ == "__main__":
    main()
