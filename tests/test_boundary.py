"""CPU tests of the drop-in boundary: the C-ABI library, host logic, API shape.

No GPU needed: these load libmpsm_b200.so (no CUDA calls), check it exports
every symbol include/mpsm_b200.h declares, run the host-side C++ splitter
search against the reference's golden splitters, and check the product never
routes through the oracle.
"""

import os
import re

import numpy as np
import pytest

import paper_1207_0145_b200 as P
from paper_1207_0145_b200 import _lib
from paper_1207_0145_b200.core import ConfigurationError, JoinConfig, KeyDomain, Relation

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    with open(os.path.join(ROOT, "include", "mpsm_b200.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(mpsm_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    syms = _header_symbols()
    assert len(syms) >= 15
    for name in syms:
        assert hasattr(L, name), name
    assert sorted(_lib.EXPORTS) == syms
    assert L.mpsm_version() == 1


def test_library_built_for_sm100a():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1207_0145_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                with open(os.path.join(dirpath, f)) as fh:
                    src = fh.read()
                assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), f
                assert "liboracle" not in src, f


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    r = Relation.from_tuples([(1, 1)])
    with pytest.raises(RuntimeError):
        P.run_join(r, r, JoinConfig(key_domain=KeyDomain(0, 8)))


def test_cpp_splitters_match_reference(golden):
    from paper_1207_0145_b200.skew import build_cdf, compute_splitters, local_equiheight_bounds

    for c in golden["splitters"]:
        dom = KeyDomain(c["lower"], c["upper"])
        runs = [np.array(k, np.uint64) for k in c["runs"]]
        bounds = [local_equiheight_bounds(P.Run(k, k.copy()), c["f"], c["t"]) for k in runs]
        cdf = build_cdf(bounds, anchor_key=c["lower"])
        ss = compute_splitters(np.array(c["hist"], np.int64), cdf, c["t"], dom, c["bits"])
        assert ss.bucket_bounds.tolist() == c["bucket_bounds"]
        assert ss.splitter_keys.tolist() == c["splitter_keys"]
        assert ss.partition_sizes.tolist() == c["partition_sizes"]


def test_splitter_kats():
    # test_skew.py:197-208 (paper Fig. 10): the lone splitter lands on key 8
    from paper_1207_0145_b200.skew import Cdf, build_cdf, compute_splitters, local_equiheight_bounds

    dom = KeyDomain(0, 32)
    s_keys = np.sort(np.array([0, 3, 9, 1, 16, 7, 21, 4, 12, 8, 5, 26, 18, 6], np.uint64))
    cdf = build_cdf([local_equiheight_bounds(P.Run(s_keys, s_keys.copy()), 4, 2)], anchor_key=0)
    ss = compute_splitters(np.array([7, 3, 3, 1], np.int64), cdf, 2, dom, 2)
    assert ss.splitter_keys.tolist() == [8]
    assert ss.partition_sizes.tolist() == [7, 7]
    assert ss.vector.sp.tolist() == [0, 1, 1, 1]
    cdf = Cdf(np.array([8, 16, 24, 32], np.uint64), np.array([5.0, 10.0, 15.0, 20.0]), 20)
    ss = compute_splitters(np.array([5, 5, 5, 5], np.int64), cdf, 4, dom, 2)
    assert ss.bucket_bounds.tolist() == [0, 1, 2, 3, 4]
    with pytest.raises(ConfigurationError):
        compute_splitters(np.array([1, 1], np.int64), Cdf(np.empty(0, np.uint64), np.empty(0), 0), 4, dom, 1)
    ss = compute_splitters(np.array([10, 0, 0, 0], np.int64), Cdf(np.empty(0, np.uint64), np.empty(0), 0), 3, dom, 2)
    assert np.all(np.diff(ss.bucket_bounds) >= 1)
    assert sorted(ss.partition_sizes.tolist()) == [0, 0, 10]


def test_size_balanced_contrast():
    from paper_1207_0145_b200.skew import Cdf, compute_size_balanced_splitters, compute_splitters

    dom = KeyDomain(0, 32)
    r_hist = np.array([7, 3, 3, 1], np.int64)
    cdf = Cdf(np.array([28, 30, 31], np.uint64), np.array([50.0, 100.0, 150.0]), 150)
    size_ss = compute_size_balanced_splitters(r_hist, cdf, 2, dom, 2)
    assert size_ss.partition_sizes.tolist() == [7, 7]
    assert compute_splitters(r_hist, cdf, 2, dom, 2).max_cost <= size_ss.max_cost


def test_host_types_match_reference_semantics():
    assert P.choose_roles(100, 400).private == "r"
    assert P.choose_roles(400, 100).private == "s"
    assert P.choose_roles(77, 77).private == "r"
    assert P.choose_roles(100, 400, "s-private").swapped
    assert [s.name for s in P.plan_phases("p-mpsm").steps] == ["sort_public", "histogram", "scatter",
                                                               "sort_private", "join"]
    assert [s.name for s in P.plan_phases("b-mpsm").steps] == ["sort_public", "sort_private", "join"]
    with pytest.raises(ConfigurationError):
        JoinConfig(threads=0)
    with pytest.raises(ConfigurationError):
        JoinConfig(threads=8, radix_bits=2)
    with pytest.raises(ConfigurationError):
        KeyDomain(5, 5)
    assert KeyDomain(1, 1_000_001).width_bits == 20
    assert KeyDomain(1, 100_000_001).width_bits == 27
    assert [c.cardinality for c in P.chunk(Relation(np.arange(10), np.arange(10)), 3)] == [4, 3, 3]
    rep = P.validate_relation(Relation.from_tuples([(1, 0), (40, 0)]), KeyDomain(0, 32))
    assert rep.violation_count == 1 and rep.sample_indices == (1,)


def test_partition_host_kats():
    from paper_1207_0145_b200.partition import (PrefixCursors, SplitterVector, bucket_lower_key, combine_counts,
                                                normalize_key)
    from paper_1207_0145_b200.core import DomainError, InternalConsistencyError

    dom = KeyDomain(0, 32)
    assert normalize_key(13, dom, 1) == 0 and normalize_key(27, dom, 1) == 1
    assert normalize_key(8, dom, 2) == 1 and normalize_key(24, dom, 2) == 3
    assert normalize_key(107, KeyDomain(100, 132), 2) == 0
    with pytest.raises(DomainError):
        normalize_key(32, dom, 1)
    with pytest.raises(ConfigurationError):
        normalize_key(3, dom, 6)
    for b in range(4):
        assert normalize_key(bucket_lower_key(b, KeyDomain(100, 132), 2), KeyDomain(100, 132), 2) == b
    cur = combine_counts([np.array([4, 1, 2, 0]), np.array([3, 2, 1, 1])], np.array([0, 1, 1, 1]), 2)
    assert cur.counts[0].tolist() == [4, 3] and cur.counts[1].tolist() == [3, 4]
    assert cur.starts[1, 0] == 4 and cur.run_sizes.tolist() == [7, 7]
    cur.verify_disjoint()
    with pytest.raises(InternalConsistencyError):
        PrefixCursors(np.array([[0], [3]]), np.array([[4], [3]]), np.array([7]), np.array([0, 7])).verify_disjoint()
    assert SplitterVector.from_bucket_bounds([0, 1, 4], 4).sp.tolist() == [0, 1, 1, 1]


# the reference's operator layer (mpsm._kernels, _kernels.py:217-408) as the
# package exposes it over the C ABI: same names and parameter lists
_REF_KERNEL_SIGNATURES = {
    "radix_histogram": ["keys", "lower", "shift", "counts"],
    "scatter_chunk": ["keys", "pays", "lower", "shift", "sp", "cursors", "ends", "out_keys", "out_pays"],
    "interp_lower_bound": ["keys", "target"],
    "merge_join_run": ["r_keys", "r_pays", "s_keys", "s_pays", "s_start", "collect", "out_r", "out_s"],
    "three_phase_sort": ["keys", "pays", "lo", "hi", "lower", "width_bits"],
    "warmup": [],
}


def test_operator_layer_signatures():
    import inspect

    from paper_1207_0145_b200 import _kernels as K

    for name, params in _REF_KERNEL_SIGNATURES.items():
        assert list(inspect.signature(getattr(K, name)).parameters) == params, name
    assert K._EMPTY_U64.dtype == np.uint64 and K._EMPTY_U64.size == 0
    assert P.hash_join_oracle is not None  # datagen.hash_join_oracle's name at the top level, as the reference's


def test_reference_suite_staging(tmp_path):
    """oracle.ref_suite stages the reference's tests with the alias conftest
    (needs /root/reference: this container; the GPU box runs the staged copy)"""
    from oracle import ref_suite

    src = "/root/reference/pkg/tests"
    if not os.path.isdir(src):
        pytest.skip("the reference is not present here")
    conf = ref_suite.CONFTEST
    assert 'sys.modules["mpsm"] = P' in conf and 'sys.modules["mpsm._kernels"] = K' in conf
    assert ref_suite.prepare(src)
    assert os.path.exists(os.path.join(ref_suite.DST, "conftest.py"))
    assert len([f for f in os.listdir(ref_suite.DST) if f.startswith("test_")]) >= 5


def test_reference_arm_under_torchrun_prints_the_distributed_config():
    """bench.py --impl reference with WORLD_SIZE > 1: rank 0 alone joins a
    bounded sample of the distributed workload on the host and prints the
    distributed arm's `config`; the other ranks exit 0 without output."""
    import json
    import subprocess
    import sys

    from paper_1207_0145_b200.distributed import dist_workload

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if not (os.path.isdir(os.path.join(root, "oracle", "_ref", "mpsm")) or
            os.path.exists(os.path.join(root, "oracle", "liboracle.so"))):
        pytest.skip("neither the reference install nor the oracle is built")
    cmd = [sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "1",
           "--warmup", "1"]
    base = dict(os.environ, WORLD_SIZE="2", LOCAL_RANK="0", MPSM_BENCH_REF_SAMPLE="20000,80000")
    out0 = subprocess.run(cmd, env=dict(base, RANK="0"), capture_output=True, text=True, timeout=600)
    assert out0.returncode == 0, out0.stderr[-2000:]
    line = json.loads([x for x in out0.stdout.splitlines() if x.startswith("{")][-1])
    config, _, n_r, n_s, _, scaling = dist_workload("cfg5", 2)
    assert line["impl"] == "reference" and line["config"] == config and line["scaling"] == scaling
    assert line["n_gpus"] == 2 and line["result"]["match_count"] == 80000
    assert "bounded sample" in line["cpu_baseline"]["sample"] and line["e2e"]["h2d_bytes_per_step"] == 0
    out1 = subprocess.run(cmd, env=dict(base, RANK="1", LOCAL_RANK="1"), capture_output=True, text=True, timeout=600)
    assert out1.returncode == 0 and not [x for x in out1.stdout.splitlines() if x.startswith("{")]
