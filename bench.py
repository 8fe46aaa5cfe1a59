#!/usr/bin/env python
"""Benchmark of the B200 MPSM join (BASELINE.json metric: join input tuples/s
(|R|+|S|) and achieved HBM GB/s fraction).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg2] [--no-cpu-baseline] [--no-e2e]

One step = one complete P-MPSM join through the public API ``run_join``
(sort S into runs, partition/sort R, merge-join with fused COUNT / MAX /
checksum, result read back to the host) over the configuration's synthetic
inputs.  At N=1 the workload is BASELINE.json configs[1] (cfg2: |R|=100M,
|S|=400M FK join, 8 GB of 16-B tuples), which fits one B200.  Under torchrun
(N>1) every rank holds a cfg2-sized shard (weak scaling) and the ranks run the
distributed engine (NCCL all-to-all of R + NVLink peer reads of S runs).

Printed JSON line (rank 0):
  value      whole-job tuples/s, inputs resident in HBM, CUDA-event timed, max
             over ranks
  e2e        the same through run_join with pinned HOST buffers: H2D of the
             inputs and D2H of the result inside the timed region
  roofline   the radix scatter pass seg::k_scatter[_ws] (the dominant kernel):
             algorithmic bytes (packing pass 16 + 8, record passes 8 + 8 B per
             tuple) / its summed CUDA-event launch time inside the timed region
             vs MEASURED_PEAKS.json hbm_gbs; traffic from the committed ncu
             capture (profiles/traffic_scatter.json)
  cpu_baseline  the reference package (oracle/_ref, numba, all host threads)
             on a bounded sample of the same workload
``--impl reference`` times the reference's own CPU implementation instead.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "join input tuples/s (|R|+|S|) and achieved HBM GB/s fraction at 1/2/4/8 B200"

CONFIGS = {
    # name: (n_r, n_s, kind)
    "cfg1": (1_000_000, 4_000_000, "fk"),
    "cfg2": (100_000_000, 400_000_000, "fk"),
    "cfg3m1": (200_000_000, 200_000_000, "fk"),
    "cfg3m4": (200_000_000, 800_000_000, "fk"),
    "cfg3m8": (200_000_000, 1_600_000_000, "fk"),
    "cfg3m16": (200_000_000, 3_200_000_000, "fk"),
    "cfg4": (400_000_000, 1_600_000_000, "negcorr"),
}
# reference results of the seeded inputs (tests/golden/golden.json)
GOLDEN = {
    "cfg1": (4_000_000, 8_587_739_465, 0x7CDED1377072045D),
    "cfg2": (400_000_000, 8_589_753_492, 0xAA48801BE88FA31B),
}
CPU_SAMPLE = (10_000_000, 40_000_000)  # bounded sample of cfg2 for the CPU legs


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def make_inputs(name: str, seed: int = 0):
    from paper_1207_0145_b200 import datagen
    from paper_1207_0145_b200.core import KeyDomain

    n_r, n_s, kind = CONFIGS[name]
    if kind == "fk":
        return datagen.gen_fk(n_r, n_s, seed)
    dom = KeyDomain(1, 1 << 32)
    r, s = datagen.gen_negcorr(n_r, n_s, dom, seed)
    return r, s, dom


# ------------------------------------------------------------ clocks sampler
class Clocks:
    QUERY = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.window = None  # (t0, t1) wall-clock bounds of the timed region
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def start(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.QUERY}",
                                          "--format=csv,noheader,nounits", "-lms", "20"], stdout=self.fh,
                                         stderr=subprocess.DEVNULL)
        except Exception as exc:  # nvidia-smi missing
            log("clock sampling unavailable:", exc)
            self.proc = None

    def mark(self, t0: float, t1: float) -> None:
        """the timed region; samples outside it are dropped"""
        self.window = (t0, t1)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        import datetime

        rows = []
        with open(self.path) as fh:
            for line in fh:
                f = [x.strip() for x in line.split(",")]
                if len(f) < 10:
                    continue
                try:
                    ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                    rows.append((ts, float(f[2]), float(f[3]), f[6:10]))
                except ValueError:
                    continue
        if self.window and rows:
            t0, t1 = self.window
            inside = [r for r in rows if t0 - 0.02 <= r[0] <= t1 + 0.02]
            # a timed region shorter than the sampling period: nearest samples
            rows = inside or sorted(rows, key=lambda r: abs(r[0] - (t0 + t1) / 2))[:2]
        for _, smv, mxv, flags in rows:
            sm.append(smv)
            mx = mxv
            for nm, v in zip(names, flags):
                if v.lower() == "active":
                    reasons.add(nm)
        try:
            os.remove(self.path)
        except OSError:
            pass
        loaded = [x for x in sm if x > 0.5 * (mx or 1)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx,
                "samples": len(sm), "reasons": sorted(reasons)}


# ------------------------------------------------------------- CPU baseline
def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference_sample(reps: int = 2):
    """Time the reference (oracle/_ref, numba) or, if absent, the C oracle
    port on a bounded sample of cfg2.  Returns (tuples/s, kind, cores, sample, result)."""
    from paper_1207_0145_b200 import datagen

    n_r, n_s = CPU_SAMPLE
    r, s, dom = datagen.gen_fk(n_r, n_s, 0)
    t = cpu_threads()
    ref_dir = os.path.join(ROOT, "oracle", "_ref")
    times, res = [], None
    if os.path.isdir(os.path.join(ref_dir, "mpsm")):
        sys.path.insert(0, ref_dir)
        import mpsm  # the reference package, unmodified

        kind = "reference"
        mpsm.warmup()
        rr, ss = mpsm.Relation(r.keys, r.payloads), mpsm.Relation(s.keys, s.payloads)
        cfg = mpsm.JoinConfig(threads=t, algorithm="p-mpsm", key_domain=mpsm.KeyDomain(dom.lower, dom.upper))
        mpsm.run_join(rr, ss, cfg)  # first run: JIT cache / page-in
        for _ in range(reps):
            t0 = time.perf_counter()
            out = mpsm.run_join(rr, ss, cfg)
            times.append(time.perf_counter() - t0)
        res = (out.match_count, out.aggregate_max, None)
    else:
        from oracle import oracle as orc

        kind = "port"
        for _ in range(reps):
            t0 = time.perf_counter()
            out = orc.join(r.keys, r.payloads, s.keys, s.payloads, threads=t, lower=dom.lower, upper=dom.upper,
                           parallel=True)
            times.append(time.perf_counter() - t0)
        res = (out.match_count, out.aggregate_max, out.checksum)
    med = statistics.median(times)
    sample = (f"|R|={n_r:,} |S|={n_s:,} FK (cfg2 generator at 1/10 scale), p-mpsm T={t}, "
              f"median of {reps} wall-clock runs of run_join after warm-up")
    return (n_r + n_s) / med, kind, t, sample, res


def impl_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    steps = []
    val = kind = cores = sample = None
    for i in range(args.warmup + args.steps):
        v, kind, cores, sample, _ = run_reference_sample(reps=1)
        if i >= args.warmup:
            steps.append(v)
    val = statistics.median(steps)
    n = CPU_SAMPLE[0] + CPU_SAMPLE[1]
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "tuples/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * n / val, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic (FK generator, PCG64 seed 0)",
        "config": {"workload": "cfg2 sample: |R|=10M, |S|=40M FK join (CPU-bounded sample of configs[1])",
                   "algorithm": "p-mpsm", "threads": cores},
        "cpu_baseline": {"value": val, "unit": "tuples/s", "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": val, "unit": "tuples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- ours
def impl_ours(args):
    import torch

    ws, rank, local = dist_env()
    # MPSM_BENCH_DIST=1 runs the multi-GPU path at world size 1 (a smoke
    # test of it on a one-GPU box)
    if ws > 1 or (os.environ.get("MPSM_BENCH_DIST") == "1" and "LOCAL_RANK" in os.environ):
        from paper_1207_0145_b200 import distributed

        return distributed.bench_main(args, METRIC, CONFIGS, make_inputs, Clocks, run_reference_sample)

    import paper_1207_0145_b200 as P
    from paper_1207_0145_b200 import _lib
    from paper_1207_0145_b200.core import JoinConfig, Relation

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    P.warmup()
    t_gen = time.perf_counter()
    r, s, dom = make_inputs(args.config)
    n_r, n_s = r.cardinality, s.cardinality
    n_tot = n_r + n_s
    log(f"[bench] generated {args.config}: |R|={n_r:,} |S|={n_s:,} in {time.perf_counter() - t_gen:.1f}s")
    # resident device inputs
    rd = Relation(torch.from_numpy(r.keys).to(dev), torch.from_numpy(r.payloads).to(dev))
    sd = Relation(torch.from_numpy(s.keys).to(dev), torch.from_numpy(s.payloads).to(dev))
    cfg = JoinConfig(threads=1, algorithm="p-mpsm", key_domain=dom)

    clocks = Clocks(local)
    clocks.start()  # sampling runs from before the warm-up; samples are kept for the timed region only
    for _ in range(args.warmup):
        res = P.run_join(rd, sd, cfg)
    torch.cuda.synchronize()
    golden = GOLDEN.get(args.config)
    result = (res.match_count, res.aggregate_max, res.checksum)
    parity = None if golden is None else (result == golden)
    if golden is not None and not parity:
        log(f"[bench] PARITY FAILURE {result} != {golden}")

    _lib.profile_enable(True)
    l0 = _lib.launch_count()
    torch.cuda.synchronize()
    w0 = time.time()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    phase = {"sort_public": 0.0, "partition": 0.0, "sort_private": 0.0, "join": 0.0, "total": 0.0}
    for _ in range(args.steps):
        res = P.run_join(rd, sd, cfg)
        for k in phase:
            phase[k] += res.phase_timings[k]
    ev1.record()
    torch.cuda.synchronize()
    clocks.mark(w0, time.time())
    launches = _lib.launch_count() - l0
    ms = ev0.elapsed_time(ev1) / args.steps
    prof = {k: _lib.profile_read(k) for k in ("seg_scatter", "seg_count", "merge", "merge_partition")}
    _lib.profile_enable(False)
    clk = clocks.stop()
    value = n_tot / (ms / 1e3)

    # roofline of the dominant kernel, the radix scatter pass (seg::k_scatter):
    # algorithmic bytes per tuple = its reads + writes in the layout it runs:
    # pairs 16 + 16; first pass of a packed sort 16 + 8; later packed passes 8 + 8
    wbits = dom.width_bits
    passes = _lib.load().mpsm_sort_pass_count(wbits)
    from paper_1207_0145_b200 import engine as _eng

    packed = _eng.PACK_RECORDS and 1 <= wbits <= 63
    per_tuple = (24 + 16 * (passes - 1)) if packed else 32 * passes
    onesweep_bytes = float(per_tuple) * (n_r + n_s) * args.steps
    os_ms, os_n = prof["seg_scatter"]
    achieved = onesweep_bytes / (os_ms / 1e3) / 1e9 if os_ms > 0 else None
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peaks = json.load(fh)
    except OSError:
        pass
    peak = peaks.get("hbm_gbs", 6650.0)
    # whole-join canonical bytes for context
    canonical = (n_s * (8 + 32 * math.ceil(wbits / 8)) + n_r * (8 + 32 * math.ceil(wbits / 8))
                 + 16 * (n_r + n_s))
    step_gbs = canonical / (ms / 1e3) / 1e9

    # per-phase HBM roofline (the north star asks >= 60 % on the sort and
    # merge-join phases): bytes the phase moves in this layout (count passes
    # 8 B/tuple + scatter passes, merge reads every run once) and SURVEY
    # 8(d)'s canonical bytes, over the phase's CUDA-event time
    n_pub, n_priv = max(n_r, n_s), min(n_r, n_s)
    sort_b = (8 * passes + per_tuple) if packed else (8 * passes + 32 * passes)
    canon_sort = 8 + 32 * math.ceil(wbits / 8)
    rec_b = 8 if packed else 16
    phase_roof = {}
    for name, nb, cb in (("sort_public", n_pub * sort_b, n_pub * canon_sort),
                         ("sort_private", n_priv * sort_b, n_priv * canon_sort),
                         ("join", (n_r + n_s) * rec_b, 16 * (n_r + n_s))):
        t = phase[name] / args.steps
        if t > 0:
            phase_roof[name] = {"gbs": nb / t / 1e9, "frac": nb / t / 1e9 / peak,
                                "canonical_gbs": cb / t / 1e9, "canonical_frac": cb / t / 1e9 / peak}

    e2e = None
    if not args.no_e2e:
        rh = Relation(torch.from_numpy(r.keys).pin_memory(), torch.from_numpy(r.payloads).pin_memory())
        sh = Relation(torch.from_numpy(s.keys).pin_memory(), torch.from_numpy(s.payloads).pin_memory())
        P.run_join(rh, sh, cfg)  # warm the path
        k = max(1, min(args.steps, args.e2e_steps))
        torch.cuda.synchronize()
        _lib.load().mpsm_upload_bytes(1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(k):
            out = P.run_join(rh, sh, cfg)
        e1.record()
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1) / k
        ok = (out.match_count, out.aggregate_max, out.checksum) == result
        up = int(_lib.load().mpsm_upload_bytes(1)) // k  # packed uploads (8-16 B/tuple)
        col = 0 if up else 16 * n_tot  # else: the columns were copied as they are
        e2e = {"value": n_tot / (e_ms / 1e3), "unit": "tuples/s", "ms_per_step": e_ms, "steps": k,
               "h2d_bytes_per_step": up + col, "d2h_bytes_per_step": 8 * _lib.PAIR_FIELDS, "result_ok": ok,
               "host_input_bytes_per_step": 16 * n_tot,
               "input_path": "host-packed records (csrc/upload.cu)" if up else "column copies"}
        del rh, sh

    cpu = None
    if not args.no_cpu_baseline:
        try:
            v, kind, cores, sample, cres = run_reference_sample(reps=2)
            cpu = {"value": v, "unit": "tuples/s", "cores": cores, "kind": kind, "sample": sample}
        except Exception as exc:
            cpu = {"value": None, "unit": "tuples/s", "cores": cpu_threads(), "kind": "reference",
                   "sample": f"failed: {exc!r}"}

    # DRAM bytes per scatter launch from the committed ncu --set full capture
    # (tools/ncu_traffic.py over one bench step's k_scatter launches)
    traffic = traffic_detail = None
    tfile = os.path.join(ROOT, "profiles", "traffic_scatter.json")
    if packed and args.config == "cfg2" and os.path.exists(tfile):
        with open(tfile) as f:
            tj = json.load(f)
        traffic = tj["dram_bytes_per_launch"]
        traffic_detail = {"unit": "bytes per launch (dram read + write)",
                          "algorithmic_bytes_per_launch": tj["algorithmic_bytes_per_launch"],
                          "ratio": tj["traffic_over_algorithmic"], "source": "profiles/traffic_scatter.json"}

    line = {
        "metric": METRIC, "value": value, "unit": "tuples/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic (FK generator SURVEY 8(d), PCG64 seed 0)",
        "config": {"workload": f"{args.config}: |R|={n_r:,} |S|={n_s:,} "
                               + ("FK equi-join" if CONFIGS[args.config][2] == "fk"
                                  else "negatively correlated 80-20 skew join, 32-bit keys")
                               + ", 16-B (u64,u64) tuples",
                   "algorithm": "p-mpsm", "threads": 1, "key_domain": [dom.lower, dom.upper],
                   "l2": f"inputs {16 * (n_r + n_s) / 1e9:.1f} GB >> 126 MB L2 (no flush needed)",
                   "parallelism": "single GPU"},
        "result": {"match_count": result[0], "aggregate_max": result[1], "checksum": hex(result[2]),
                   "matches_golden": parity},
        "phase_ms": {k: 1e3 * v / args.steps for k, v in phase.items()},
        "roofline": {"bound": "hbm", "kernel": "seg::k_scatter (radix scatter pass)", "achieved": achieved,
                     "peak": peak, "unit": "GB/s", "frac": (achieved / peak) if achieved else None,
                     "traffic": traffic, "traffic_detail": traffic_detail,
                     "algorithmic_bytes_per_tuple_per_sort": per_tuple,
                     "layout": "packed 8-B records" if packed else "(key, payload) pairs", "passes_per_sort": passes,
                     "launches": os_n, "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback"},
        "step_canonical_gbs": step_gbs,
        "phase_roofline": phase_roof,
        "kernel_ms_per_step": {k: v[0] / args.steps for k, v in prof.items()},
        "gpu_launches": launches,
        "clocks": clk,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        impl_reference(args)
    else:
        impl_ours(args)


if __name__ == "__main__":
    main()
