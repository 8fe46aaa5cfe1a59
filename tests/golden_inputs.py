"""Rebuild the seeded inputs named in tests/golden/golden.json.

The recipes mirror tests/golden/make_golden.py but depend only on numpy and
this repo (the reference is not present on the GPU box).  Skewed inputs come
from the product's restated generator; test_oracle_golden checks its arrays'
fingerprints against the reference's.
"""

from __future__ import annotations

import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_GOLDEN = None


def load_golden() -> dict:
    global _GOLDEN
    if _GOLDEN is None:
        with open(os.path.join(HERE, "golden", "golden.json")) as fh:
            _GOLDEN = json.load(fh)
    return _GOLDEN


def rel_random(n, seed, upper):
    rng = np.random.default_rng(seed)
    return rng.integers(0, upper, n, dtype=np.uint64), rng.integers(0, 1 << 32, n, dtype=np.uint64)


def make_inputs(d: dict):
    """-> (r_keys, r_pays, s_keys, s_pays, lower, upper)"""
    from paper_1207_0145_b200 import datagen
    from paper_1207_0145_b200.core import KeyDomain

    if d["kind"] == "random":
        rk, rp = rel_random(d["n_r"], d["seed_r"], d["upper"])
        sk, sp = rel_random(d["n_s"], d["seed_s"], d["upper"])
        return rk, rp, sk, sp, 0, d["upper"]
    if d["kind"] == "fk":
        r, s, dom = datagen.gen_fk(d["n_r"], d["n_s"], d["seed"])
        return r.keys, r.payloads, s.keys, s.payloads, dom.lower, dom.upper
    if d["kind"] == "skew":
        dom = KeyDomain(0, d["upper"])
        r = datagen.gen_skewed_8020(d["n_r"], dom, "high", seed=d["seed_r"])
        s = datagen.gen_skewed_8020(d["n_s"], dom, "low", seed=d["seed_s"])
        return r.keys, r.payloads, s.keys, s.payloads, 0, d["upper"]
    if d["kind"] == "self":
        rng = np.random.default_rng(d["seed"])
        k = rng.integers(0, d["upper"], d["n"], dtype=np.uint64)
        return k, k.copy(), k.copy(), k.copy(), 0, d["upper"]
    raise ValueError(d)


def fingerprint(a) -> list:
    from oracle.oracle import pair_hash_np

    a = np.ascontiguousarray(a, np.uint64)
    return [int(a.shape[0]), int(np.sum(a, dtype=np.uint64)),
            int(np.sum(pair_hash_np(a, np.arange(a.shape[0], dtype=np.uint64)), dtype=np.uint64))]


def dataset(name: str) -> dict:
    for d in load_golden()["datasets"]:
        if d["name"] == name:
            return d
    raise KeyError(name)


def reference_totals(name: str):
    """(count, max, checksum) of a dataset from the reference (T-independent)."""
    g = load_golden()
    count = mx = cs = None
    for c in g["engine_cases"]:
        if c["dataset"] != name or "error" in c:
            continue
        if c["query_mode"] == "aggregate-max":
            count, mx = c["match_count"], c["aggregate_max"]
        if c["query_mode"] == "materialize" and "checksum" in c:
            cs = c["checksum"]
    return count, mx, cs
