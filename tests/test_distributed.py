"""Multi-rank host protocol of the distributed join under gloo (CPU, 2 ranks).

The ranks run paper_1207_0145_b200.distributed.run_join_distributed with the
oracle-backed CPU backend (tests/dist_backend.py): histogram all-gather,
identical splitters on every rank, stable scatter into send segments, the
all-to-all(v), peer-run exchange and the final fold.  Results must equal the
reference's own T=world_size run (golden fixtures) bit for bit, including the
per-worker statistics.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1207_0145_b200.core import JoinConfig, KeyDomain, Relation, chunk_bounds
        from paper_1207_0145_b200.distributed import run_join_distributed
        from tests.dist_backend import OracleBackend
        from tests.golden_inputs import dataset, make_inputs

        out = []
        for name, mode, role in cases:
            rk, rp, sk, sp, lo, up = make_inputs(dataset(name))
            ra, rb = chunk_bounds(rk.shape[0], world)[rank]
            sa, sb = chunk_bounds(sk.shape[0], world)[rank]
            cfg = JoinConfig(threads=world, key_domain=KeyDomain(lo, up), query_mode=mode, role_policy=role,
                             materialize_cap=1 << 24)
            res = run_join_distributed(Relation(rk[ra:rb], rp[ra:rb]), Relation(sk[sa:sb], sp[sa:sb]), cfg,
                                       backend=OracleBackend())
            mat = None if res.materialized is None else sorted(map(tuple, res.materialized.tolist()))
            out.append((res.match_count, res.aggregate_max, res.checksum, mat,
                        [(w.public_tuples_examined, w.probe_tuples_examined, w.s_runs_with_matches,
                          w.tuples_sorted_private) for w in res.worker_stats]))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


CASES = [("fk_small", "aggregate-max", "auto"), ("uniform_mid", "aggregate-max", "auto"),
         ("negcorr", "aggregate-max", "auto"), ("dup_heavy", "materialize", "auto"),
         ("r_bigger", "aggregate-max", "auto"), ("uniform_small", "count", "s-private")]


def test_two_ranks_gloo_match_reference(golden):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, CASES, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert results[0] == results[1]  # every rank folds the same result
    from oracle import oracle as orc
    from tests.golden_inputs import dataset, make_inputs, reference_totals

    for (name, mode, role), got in zip(CASES, results[0]):
        want = None
        for c in golden["engine_cases"]:
            if (c["dataset"], c["algorithm"], c["threads"], c["query_mode"], c["role_policy"]) == \
                    (name, "p-mpsm", 2, "aggregate-max", role) and "error" not in c:
                want = c
        count, mx, cs = reference_totals(name)
        assert got[0] == count and got[2] == cs, name
        if mode == "aggregate-max":
            assert got[1] == mx, name
        if want is not None:
            stats = [(w["public_tuples_examined"], w["probe_tuples_examined"], w["s_runs_with_matches"],
                      w["tuples_sorted_private"]) for w in want["worker_stats"]]
            assert got[4] == stats, name
        if mode == "materialize":
            rk, rp, sk, sp, lo, up = make_inputs(dataset(name))
            ref = orc.join(rk, rp, sk, sp, threads=1, lower=lo, upper=up, query_mode="materialize",
                           materialize_cap=1 << 24)
            assert got[3] == sorted(map(tuple, ref.materialized.tolist()))


def test_counter_based_fk_shards_form_a_permutation():
    from paper_1207_0145_b200.distributed import fk_shard_device

    n_r, n_s, world = 100_003, 400_011, 3
    parts = [fk_shard_device(n_r, n_s, r, world, 0, torch.device("cpu")) for r in range(world)]
    rk = np.concatenate([p[0].keys.numpy() for p in parts])
    sk = np.concatenate([p[1].keys.numpy() for p in parts])
    assert np.array_equal(np.sort(rk), np.arange(1, n_r + 1, dtype=np.uint64))  # FK: R keys unique, dense
    assert sk.shape[0] == n_s and sk.min() >= 1 and sk.max() <= n_r
    assert np.unique(sk).shape[0] > 0.9 * (1 - np.exp(-4)) * n_r
    pays = np.concatenate([p[0].payloads.numpy() for p in parts])
    assert pays.max() < (1 << 32) and np.unique(pays).shape[0] > 0.99 * n_r


def _fault_worker(rank, world, port, where, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import datetime

    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=60))
    try:
        from paper_1207_0145_b200.core import JoinConfig, KeyDomain, Relation, chunk_bounds
        from paper_1207_0145_b200.distributed import run_join_distributed
        from tests.dist_backend import OracleBackend
        from tests.golden_inputs import dataset, make_inputs

        class Faulty(OracleBackend):
            def sort(self, k, p, public=False):
                if where == "public" and public:
                    raise ValueError("boom in the public sort")
                if where == "private" and not public:
                    raise ValueError("boom in the private sort")
                return super().sort(k, p, public)

            def partition(self, *a):
                if where == "partition":
                    raise ValueError("boom in the partition")
                return super().partition(*a)

        rk, rp, sk, sp, lo, up = make_inputs(dataset("fk_small"))
        ra, rb = chunk_bounds(rk.shape[0], world)[rank]
        sa, sb = chunk_bounds(sk.shape[0], world)[rank]
        be = Faulty() if rank == 1 else OracleBackend()
        try:
            run_join_distributed(Relation(rk[ra:rb], rp[ra:rb]), Relation(sk[sa:sb], sp[sa:sb]),
                                 JoinConfig(threads=world, key_domain=KeyDomain(lo, up)), backend=be)
            q.put((rank, "ok", ""))
        except Exception as exc:  # noqa: BLE001 - reported to the test
            q.put((rank, type(exc).__name__, str(exc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("where", ["public", "partition", "private"])
def test_failing_rank_raises_everywhere_without_hanging(where):
    """a rank whose local work raises enters the next collective with a
    failure flag: it raises its own exception (the root cause), its peers a
    RuntimeError naming it, and nobody blocks (engine.py:440-453)"""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fault_worker, args=(r, 2, port, where, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict((r, (kind, msg)) for r, kind, msg in (q.get(timeout=120) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert results[1][0] == "ValueError" and "boom" in results[1][1]
    kind, msg = results[0]
    assert kind == "RuntimeError" and ("rank(s) [1]" in msg or "peer rank failed" in msg), (kind, msg)
