"""The distributed engine's CUDA backend on one GPU (NCCL, world size 1).

With one rank the protocol still runs every device step (sort, histogram,
partition scatter into send segments, NCCL all-to-all, join, fold)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402

from paper_1207_0145_b200.core import JoinConfig, KeyDomain, Relation  # noqa: E402
from paper_1207_0145_b200.distributed import run_join_distributed  # noqa: E402
import paper_1207_0145_b200 as P  # noqa: E402


@pytest.fixture(scope="module")
def nccl_group():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def test_world_of_one_matches_golden(golden, nccl_group):
    g = golden["config1"]
    r, s, dom = P.gen_fk(g["n_r"], g["n_s"], g["seed"])
    res = run_join_distributed(r, s, JoinConfig(threads=1, key_domain=dom))
    assert (res.match_count, res.aggregate_max, res.checksum) == (g["match_count"], g["aggregate_max"],
                                                                 g["checksum"])
    # pairs layout and a skewed domain
    from paper_1207_0145_b200.distributed import CudaBackend
    from oracle import oracle as orc

    d2 = KeyDomain(1, 1 << 32)
    r2, s2 = P.gen_negcorr(200_000, 800_000, d2)
    want = orc.join(r2.keys, r2.payloads, s2.keys, s2.payloads, threads=1, lower=1, upper=1 << 32)
    for packed in (True, False):
        res = run_join_distributed(r2, s2, JoinConfig(key_domain=d2), backend=CudaBackend(packed=packed))
        assert (res.match_count, res.aggregate_max, res.checksum) == (want.match_count, want.aggregate_max,
                                                                     want.checksum)


def test_device_fk_shard_join(nccl_group):
    from paper_1207_0145_b200.distributed import fk_shard_device

    n_r, n_s = 2_000_000, 8_000_000
    r, s = fk_shard_device(n_r, n_s, 0, 1, 0, torch.device("cuda", 0))
    res = run_join_distributed(r, s, JoinConfig(key_domain=KeyDomain(1, n_r + 1)))
    assert res.match_count == n_s
    rk, rp = r.keys.cpu().numpy(), r.payloads.cpu().numpy()
    sk, sp = s.keys.cpu().numpy(), s.payloads.cpu().numpy()
    from oracle import oracle as orc

    assert (res.match_count, res.aggregate_max, res.checksum) == orc.fk_gather(rk, rp, sk, sp, 1)


@pytest.mark.gpu
def test_ipc_handle_offset_roundtrip_in_child_process():
    """mpsm_ipc_get_handle names the cudaMalloc block of a sub-allocated
    tensor plus its byte offset; a second process maps it (lazy peer access)
    and reads exactly the tensor's elements (what a peer rank's merge reads)."""
    import subprocess
    import sys

    import torch

    from paper_1207_0145_b200.distributed import ipc_share

    big = torch.arange(1 << 20, dtype=torch.int64, device="cuda") * 7 + 3
    x = big[12345:12345 + 5000]  # inside a caching-allocator block
    torch.cuda.synchronize()
    handle, off, n = ipc_share(x)
    assert n == 5000 and off >= 12345 * 8
    child = r"""
import sys, torch
sys.path.insert(0, sys.argv[1])
from paper_1207_0145_b200.distributed import ipc_open
torch.cuda.set_device(0)
run = ipc_open((bytes.fromhex(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])), torch.device("cuda", 0))
class A:
    __cuda_array_interface__ = {"shape": (run.numel(),), "typestr": "<i8", "data": (run.data_ptr(), False), "version": 3}
t = torch.as_tensor(A(), device="cuda")
want = torch.arange(12345, 12345 + 5000, dtype=torch.int64, device="cuda") * 7 + 3
print("OK" if bool((t == want).all()) else "MISMATCH")
"""
    root = __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", child, root, handle.hex(), str(off), str(n)], capture_output=True,
                       text=True, timeout=300)
    assert "OK" in r.stdout, r.stdout + r.stderr
    del big, x


def _gloo_cuda_worker(rank, world, port, cases, packed, q, per_rank_device=False):
    import os as _os

    _os.environ["MASTER_ADDR"] = "127.0.0.1"
    _os.environ["MASTER_PORT"] = str(port)
    import torch as _t
    import torch.distributed as _dist

    _t.cuda.set_device(rank if per_rank_device else 0)
    _dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1207_0145_b200.core import JoinConfig as _JC, KeyDomain as _KD, Relation as _Rel, chunk_bounds
        from paper_1207_0145_b200.distributed import CudaBackend, run_join_distributed as _rjd
        from tests.golden_inputs import dataset, make_inputs

        out = []
        for name, mode, role in cases:
            rk, rp, sk, sp, lo, up = make_inputs(dataset(name))
            ra, rb = chunk_bounds(rk.shape[0], world)[rank]
            sa, sb = chunk_bounds(sk.shape[0], world)[rank]
            cfg = _JC(threads=world, key_domain=_KD(lo, up), query_mode=mode, role_policy=role,
                      materialize_cap=1 << 24)
            be = CudaBackend(packed=packed, comm_device=_t.device("cpu"))
            res = _rjd(_Rel(rk[ra:rb], rp[ra:rb]), _Rel(sk[sa:sb], sp[sa:sb]), cfg, backend=be)
            mat = None if res.materialized is None else sorted(map(tuple, res.materialized.tolist()))
            out.append((res.match_count, res.aggregate_max, res.checksum, mat,
                        [(w.public_tuples_examined, w.probe_tuples_examined, w.s_runs_with_matches,
                          w.tuples_sorted_private) for w in res.worker_stats]))
        q.put((rank, out))
    finally:
        from paper_1207_0145_b200.distributed import ipc_close_all

        ipc_close_all()
        _dist.destroy_process_group()


@pytest.mark.parametrize("packed", [True, False], ids=["packed", "pairs"])
def test_cuda_backend_two_ranks_one_gpu_match_reference(golden, packed):
    """Two ranks of the CUDA engine (gloo for the host collectives, both on
    cuda:0): partition, exchange, public runs mapped by CUDA IPC from the
    other process and read by the merge kernel, rank-rotated order, fold.
    Only correctness: the ranks' kernels never wait on one another."""
    import torch.multiprocessing as mp

    from tests.test_distributed import CASES

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as sck:
        sck.bind(("127.0.0.1", 0))
        port = sck.getsockname()[1]
    procs = [ctx.Process(target=_gloo_cuda_worker, args=(r, 2, port, CASES, packed, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert results[0] == results[1]
    from tests.golden_inputs import reference_totals

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


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs: a peer run on another device")
@pytest.mark.parametrize("packed", [True, False], ids=["packed", "pairs"])
def test_merge_reads_public_run_on_another_gpu(golden, packed):
    """Rank i on cuda:i: each rank's merge kernel TMA-loads the other rank's
    public run from the other GPU's HBM through its CUDA-IPC mapping (NVLink
    peer access) -- the multi-GPU data path, checked against the reference."""
    import torch.multiprocessing as mp

    from tests.test_distributed import CASES

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as sck:
        sck.bind(("127.0.0.1", 0))
        port = sck.getsockname()[1]
    procs = [ctx.Process(target=_gloo_cuda_worker, args=(r, 2, port, CASES, packed, q, True)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert results[0] == results[1]
    from tests.golden_inputs import reference_totals

    for (name, mode, role), got in zip(CASES, results[0]):
        count, mx, cs = reference_totals(name)
        assert got[0] == count and got[2] == cs, name
