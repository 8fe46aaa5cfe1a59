"""The reference's benchmark row schema (``mpsm-bench``) for B200 runs.

One flat row per configuration point with phase times, results and
per-worker statistics, in the column order and formatting of
``/root/reference/pkg/src/mpsm/bench.py:40-67`` (``REPORT_COLUMNS``),
``bench.py:169-197`` (``_base_row``), ``bench.py:247-268`` (filling a row
from a ``JoinResult``) and ``bench.py:274-289`` (``emit_report``), so rows
from either engine go into the same CSV / JSON reports.
"""

from __future__ import annotations

import csv
import json
from typing import Optional, Sequence

from .core import ConfigurationError, JoinConfig, JoinResult

REPORT_COLUMNS = [
    "algorithm", "threads", "size_r", "size_s", "multiplicity", "distribution", "seed", "rep", "radix_bits",
    "cdf_fanout", "role_policy", "query_mode", "t_sort_public", "t_partition", "t_sort_private", "t_join",
    "t_total", "match_count", "aggregate_max", "correct", "tuples_sorted", "tuples_scattered", "examined_total",
    "examined_max_worker", "examined_per_worker", "error",
]


def base_row(cfg: JoinConfig, size_r: int, size_s: int, *, distribution: str = "uniform", seed: int = 0,
             rep: int = 0, multiplicity: Optional[int] = None) -> dict:
    """A row with the configuration columns set and the result columns empty."""
    row = {k: "" for k in REPORT_COLUMNS}
    row.update({
        "algorithm": cfg.algorithm, "threads": cfg.threads, "size_r": size_r, "size_s": size_s,
        "multiplicity": multiplicity if multiplicity is not None else (size_s // size_r if size_r else 0),
        "distribution": distribution, "seed": seed, "rep": rep, "radix_bits": cfg.radix_bits,
        "cdf_fanout": cfg.cdf_fanout, "role_policy": cfg.role_policy, "query_mode": cfg.query_mode,
    })
    return row


def fill_row(row: dict, res: JoinResult, expected: Optional[tuple] = None) -> dict:
    """Result columns from a JoinResult (bench.py:247-268 formatting)."""
    pt = res.phase_timings
    row["t_sort_public"] = f"{pt.get('sort_public', 0.0):.6f}"
    row["t_partition"] = f"{pt.get('partition', 0.0):.6f}"
    row["t_sort_private"] = f"{pt.get('sort_private', 0.0):.6f}"
    row["t_join"] = f"{pt.get('join', 0.0):.6f}"
    row["t_total"] = f"{pt['total']:.6f}"
    row["match_count"] = res.match_count
    row["aggregate_max"] = "" if res.aggregate_max is None else res.aggregate_max
    if expected is not None:
        row["correct"] = (res.match_count, res.aggregate_max) == tuple(expected)
    ws = res.worker_stats
    row["tuples_sorted"] = sum(w.tuples_sorted_public + w.tuples_sorted_private for w in ws)
    row["tuples_scattered"] = sum(w.tuples_scattered for w in ws)
    examined = [w.public_tuples_examined for w in ws]
    row["examined_total"] = sum(examined)
    row["examined_max_worker"] = max(examined) if examined else 0
    row["examined_per_worker"] = ";".join(str(e) for e in examined)
    return row


def emit_report(rows: Sequence[dict], fmt: str, path) -> None:
    """Write rows as CSV (fixed header) or JSON (array of flat objects)."""
    if not rows:
        raise ConfigurationError("refusing to emit an empty report")
    if fmt == "csv":
        with open(path, "w", newline="") as fh:
            writer = csv.DictWriter(fh, fieldnames=REPORT_COLUMNS)
            writer.writeheader()
            for row in rows:
                writer.writerow({k: row.get(k, "") for k in REPORT_COLUMNS})
    elif fmt == "json":
        payload = [{k: row.get(k, "") for k in REPORT_COLUMNS} for row in rows]
        with open(path, "w") as fh:
            json.dump(payload, fh, indent=1, default=str)
    else:
        raise ConfigurationError(f"unknown report format {fmt!r}")
