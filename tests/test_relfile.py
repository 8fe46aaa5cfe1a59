"""Relation files and report rows -- the input side of the bench path
(SURVEY.md 8(f) row 4).  CPU tests pin read/write against files written by
the reference itself (tests/golden/make_relfile_golden.py): identical bytes,
identical FormatError messages and byte offsets.  The GPU test loads a file
through pinned memory + mpsm_deinterleave and joins it."""

import csv
import json
import os

import numpy as np
import pytest

from paper_1207_0145_b200 import relfile, report
from paper_1207_0145_b200.core import FormatError, JoinConfig, JoinResult, Relation, WorkerStats

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")


@pytest.fixture(scope="module")
def rgold():
    with open(os.path.join(GOLD, "relfile.json")) as fh:
        return json.load(fh)


def test_read_reference_written_file(rgold):
    rel = relfile.read_relation(os.path.join(GOLD, "rel_small.mpsmrel"))
    assert rel.cardinality == rgold["n"] == 256
    assert np.array_equal(np.asarray(rel.keys), np.array(rgold["keys"], dtype=np.uint64))
    assert np.array_equal(np.asarray(rel.payloads), np.array(rgold["payloads"], dtype=np.uint64))
    assert relfile.read_header(os.path.join(GOLD, "rel_small.mpsmrel")) == 256


def test_write_is_byte_identical_to_reference(rgold, tmp_path):
    rel = Relation(np.array(rgold["keys"], dtype=np.uint64), np.array(rgold["payloads"], dtype=np.uint64))
    p = tmp_path / "w.mpsmrel"
    relfile.write_relation(rel, p)
    with open(os.path.join(GOLD, "rel_small.mpsmrel"), "rb") as fh:
        assert p.read_bytes() == fh.read()
    z = tmp_path / "z.mpsmrel"
    relfile.write_relation(Relation(np.zeros(0, np.uint64), np.zeros(0, np.uint64)), z)
    assert z.read_bytes().hex() == rgold["zero_file_hex"]
    assert relfile.read_relation(z).cardinality == 0


VARIANTS = {
    "bad_magic": lambda b: b"MPSMREL2" + b[8:],
    "short_magic": lambda b: b[:5],
    "truncated_header": lambda b: b[:12],
    "extra_byte": lambda b: b + b"\x00",
    "missing_record": lambda b: b[:-16],
    "missing_byte": lambda b: b[:-1],
    "count_too_large": lambda b: b[:8] + (10**6).to_bytes(8, "little") + b[16:],
    "empty_file": lambda b: b"",
}


@pytest.mark.parametrize("name", sorted(VARIANTS))
def test_format_errors_match_reference(rgold, tmp_path, name):
    with open(os.path.join(GOLD, "rel_small.mpsmrel"), "rb") as fh:
        blob = fh.read()
    p = tmp_path / name
    p.write_bytes(VARIANTS[name](blob))
    want = rgold["errors"][name]
    with pytest.raises(FormatError) as ei:
        relfile.read_relation(p)
    assert ei.value.byte_offset == want["byte_offset"]
    assert str(ei.value) == want["message"].replace("{path}", str(p))


def test_missing_file_is_oserror(tmp_path):
    with pytest.raises(OSError):
        relfile.read_relation(tmp_path / "nope")


def test_report_rows_and_emit(tmp_path):
    cfg = JoinConfig(threads=2)
    res = JoinResult(match_count=12, aggregate_max=99, materialized=None,
                     phase_timings={"sort_public": 0.5, "partition": 0.25, "sort_private": 0.125, "join": 1.0,
                                    "total": 1.875},
                     worker_stats=[WorkerStats(worker=i, tuples_sorted_public=10 + i, tuples_sorted_private=5,
                                               tuples_scattered=3, public_tuples_examined=7 * (i + 1))
                                   for i in range(2)])
    row = report.fill_row(report.base_row(cfg, 100, 400, seed=3), res, expected=(12, 99))
    assert row["t_total"] == "1.875000" and row["t_partition"] == "0.250000"
    assert row["correct"] is True and row["multiplicity"] == 4
    assert row["tuples_sorted"] == 10 + 11 + 10 and row["tuples_scattered"] == 6
    assert row["examined_total"] == 21 and row["examined_max_worker"] == 14 and row["examined_per_worker"] == "7;14"
    report.emit_report([row], "csv", tmp_path / "r.csv")
    with open(tmp_path / "r.csv") as fh:
        rows = list(csv.reader(fh))
    assert rows[0] == report.REPORT_COLUMNS and len(rows) == 2
    report.emit_report([row], "json", tmp_path / "r.json")
    assert list(json.load(open(tmp_path / "r.json"))[0]) == report.REPORT_COLUMNS


@pytest.mark.gpu
def test_load_relation_to_device_and_join(tmp_path):
    import torch

    import paper_1207_0145_b200 as P

    r, s, dom = P.gen_fk(20_000, 80_000, seed=5)
    pr, ps = tmp_path / "r.mpsmrel", tmp_path / "s.mpsmrel"
    relfile.write_relation(r, pr)
    relfile.write_relation(s, ps)
    rd, sd = relfile.load_relation(pr), relfile.load_relation(ps)
    assert rd.keys.is_cuda and sd.payloads.is_cuda
    assert np.array_equal(rd.keys.cpu().numpy(), np.asarray(r.keys))
    assert np.array_equal(sd.payloads.cpu().numpy(), np.asarray(s.payloads))
    cfg = JoinConfig(threads=2, key_domain=dom)
    a = P.run_join(rd, sd, cfg)
    b = P.run_join(r, s, cfg)
    assert (a.match_count, a.aggregate_max, a.checksum) == (b.match_count, b.aggregate_max, b.checksum)
    assert a.match_count == 80_000
    # odd sizes and an empty file through the device path
    for n in (0, 1, 7, 4097):
        q = tmp_path / f"q{n}.mpsmrel"
        rel = Relation(np.arange(n, dtype=np.uint64) * 3, np.arange(n, dtype=np.uint64) ^ 5)
        relfile.write_relation(rel, q)
        got = relfile.load_relation(q)
        assert np.array_equal(got.keys.cpu().numpy(), np.asarray(rel.keys))
        assert np.array_equal(got.payloads.cpu().numpy(), np.asarray(rel.payloads))
    torch.cuda.synchronize()


@pytest.mark.gpu
def test_device_generator_fk_shape():
    import paper_1207_0145_b200 as P

    r, s, dom = P.gen_fk_device(50_000, 200_000, seed=3)
    rk = r.keys.cpu().numpy()
    assert np.array_equal(np.sort(rk), np.arange(1, 50_001, dtype=np.uint64))  # a permutation
    sk = s.keys.cpu().numpy()
    assert sk.min() >= 1 and sk.max() <= 50_000
    res = P.run_join(r, s, P.JoinConfig(threads=1, key_domain=dom))
    assert res.match_count == 200_000
